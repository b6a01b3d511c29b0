set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.txt 2>&1
SMART_VERBOSE=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or run_step or every_mode" > gpurun_out/r2c_pytest1.txt 2>&1; echo "rc $?" >> gpurun_out/r2c_pytest1.txt
tail -30 gpurun_out/r2c_pytest1.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2c_pytest2.txt 2>&1; echo "rc $?" >> gpurun_out/r2c_pytest2.txt
tail -30 gpurun_out/r2c_pytest2.txt
timeout 300 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
head -c 700 gpurun_out/r2c_bench.json; tail -5 gpurun_out/r2c_bench.err
