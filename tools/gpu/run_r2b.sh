set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r2b_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
tail -3 gpurun_out/r2b_pytest_gpu.txt
cat gpurun_out/r2b_bench.json | head -c 600
