# team merges + tagged lines (no arrival counter): GPU parity suite, cfg2/cfg3 bench, step timelines
python -m paper_2604_09731_b200._build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r2p_pytest_gpu.txt
timeout 600 python bench.py --workload cfg2_llama8b_b1 --steps 100 --no-hbm-regime --no-cpu-baseline > gpurun_out/r2p_bench_cfg2.json 2> gpurun_out/r2p_bench_cfg2.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2p_bench_cfg3.json 2> gpurun_out/r2p_bench_cfg3.err
SMART_PROBES=1 timeout 300 python tools/probes/step_timeline.py cfg2_llama8b_b1 > gpurun_out/r2p_timeline_cfg2.txt 2>&1
SMART_PROBES=1 timeout 300 python tools/probes/step_timeline.py > gpurun_out/r2p_timeline_cfg3.txt 2>&1
tail -n 3 gpurun_out/r2p_pytest_gpu.txt
