# walk: each node's matching child found in parallel: quick checks, suite, benches, timeline
python -m paper_2604_09731_b200._build > /dev/null
timeout 120 python __graft_entry__.py smoke > gpurun_out/r4c_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r4c_smoke.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or cfg3 or small_selection" > gpurun_out/r4c_quick.txt 2>&1; rc=$?; echo "quick rc $rc" >> gpurun_out/r4c_quick.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4c_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r4c_pytest_gpu.txt
timeout 300 python bench.py --workload cfg2_llama8b_b1 --steps 100 --no-hbm-regime --no-cpu-baseline > gpurun_out/r4c_bench_cfg2.json 2> gpurun_out/r4c_bench_cfg2.err
timeout 400 python bench.py --no-cpu-baseline --no-hbm-regime > gpurun_out/r4c_bench_cfg3.json 2> gpurun_out/r4c_bench_cfg3.err
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r4c_timeline_cfg3.txt 2>&1
tail -n 3 gpurun_out/r4c_pytest_gpu.txt
