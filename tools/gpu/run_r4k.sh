# verify rows published by select_small after the last layer: parity, suite, bench A/B (= off), timelines
python -m paper_2604_09731_b200._build > /dev/null
timeout 120 python __graft_entry__.py smoke > gpurun_out/r4k_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r4k_smoke.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or cfg3 or small_selection" > gpurun_out/r4k_quick.txt 2>&1; rc=$?; echo "quick rc $rc" >> gpurun_out/r4k_quick.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4k_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r4k_pytest_gpu.txt
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r4k_bench_on_$i.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r4k_bench_off_$i.json 2>/dev/null
done
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r4k_timeline_on.txt 2>&1
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r4k_timeline_off.txt 2>&1
