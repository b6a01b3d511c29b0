# screened selection for long lists (select_layer): quick parity on the long-list cases, suite, cfg5/cfg3 bench, cfg5 select phases
python -m paper_2604_09731_b200._build > /dev/null
timeout 120 python __graft_entry__.py smoke > gpurun_out/r3z_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r3z_smoke.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "large or b256 or cfg5 or many_above or cfg3" > gpurun_out/r3z_quick.txt 2>&1; rc=$?; echo "quick rc $rc" >> gpurun_out/r3z_quick.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3z_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r3z_pytest_gpu.txt
timeout 400 python bench.py --workload cfg5_r1distill_b256 --steps 50 --no-cpu-baseline --no-hbm-regime > gpurun_out/r3z_bench_cfg5.json 2> gpurun_out/r3z_bench_cfg5.err
timeout 400 python bench.py --no-cpu-baseline --no-hbm-regime > gpurun_out/r3z_bench_cfg3.json 2> gpurun_out/r3z_bench_cfg3.err
SMART_PROBES=1 python -m paper_2604_09731_b200._build > /dev/null
CHEAP=1 SMART_PROBES=1 timeout 300 python tools/probes/probe_cfg5_select.py > gpurun_out/r3z_cfg5_select.txt 2>&1
