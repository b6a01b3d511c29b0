# select_small reads the slice lists directly (team merge off the critical path): parity, suite, bench, timelines
python -m paper_2604_09731_b200._build > /dev/null
timeout 120 python __graft_entry__.py smoke > gpurun_out/r4m_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r4m_smoke.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or cfg3 or small_selection" > gpurun_out/r4m_quick.txt 2>&1; rc=$?; echo "quick rc $rc" >> gpurun_out/r4m_quick.txt
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r4m_timeline_cfg3.txt 2>&1
if [ $rc -ne 0 ]; then exit 1; fi
python -m paper_2604_09731_b200._build > /dev/null
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r4m_bench_$i.json 2>/dev/null
done
for w in cfg2_llama8b_b1 cfg4_qwen2vl_b12; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --no-hbm-regime --steps-only > gpurun_out/r4m_bench_$w.json 2>/dev/null
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4m_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r4m_pytest_gpu.txt
