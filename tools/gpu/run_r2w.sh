# round-2 re-entry check of HEAD (team merges + tagged lines): GPU parity suite, smoke, cfg2/cfg3 bench
python -m paper_2604_09731_b200._build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r2w_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2w_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r2w_smoke.txt
timeout 600 python bench.py --workload cfg2_llama8b_b1 --steps 100 --no-hbm-regime --no-cpu-baseline > gpurun_out/r2w_bench_cfg2.json 2> gpurun_out/r2w_bench_cfg2.err
timeout 900 python bench.py > gpurun_out/r2w_bench_cfg3.json 2> gpurun_out/r2w_bench_cfg3.err
SMART_PROBES=1 timeout 300 python tools/probes/step_timeline.py > gpurun_out/r2w_timeline_cfg3.txt 2>&1
tail -n 3 gpurun_out/r2w_pytest_gpu.txt
