# direct list screening, batched re-polls: quick parity, timeline, bench cfg3
python -m paper_2604_09731_b200._build > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or cfg3 or small_selection" > gpurun_out/r4q_quick.txt 2>&1; rc=$?; echo "quick rc $rc" >> gpurun_out/r4q_quick.txt
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r4q_timeline_cfg3.txt 2>&1
python -m paper_2604_09731_b200._build > /dev/null
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r4q_bench_$i.json 2>/dev/null
done
