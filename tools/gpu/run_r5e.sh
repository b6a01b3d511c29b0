# consume dry chunk at the first slice: parity (quick + sampling + walk tests), bench, timeline
python -m paper_2604_09731_b200._build > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or cfg3 or small_selection" > gpurun_out/r5e_quick.txt 2>&1; rc=$?; echo "quick rc $rc" >> gpurun_out/r5e_quick.txt
if [ $rc -ne 0 ]; then exit 1; fi
for i in 1 2 3; do
timeout 300 python bench.py --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r5e_bench_$i.json 2>/dev/null
done
for w in cfg2_llama8b_b1 cfg4_qwen2vl_b12; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r5e_bench_$w.json 2>/dev/null
done
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r5e_timeline_cfg3.txt 2>&1
