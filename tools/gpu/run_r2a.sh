set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r2a_pytest_gpu.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_steps.py --path layer > gpurun_out/r2a_memcheck.txt 2>&1; echo "rc $?" >> gpurun_out/r2a_memcheck.txt
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_steps.py --path layer > gpurun_out/r2a_synccheck.txt 2>&1; echo "rc $?" >> gpurun_out/r2a_synccheck.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_steps.py --path layer --only toy,cfg2 > gpurun_out/r2a_racecheck.txt 2>&1; echo "rc $?" >> gpurun_out/r2a_racecheck.txt
tail -3 gpurun_out/r2a_pytest_gpu.txt
