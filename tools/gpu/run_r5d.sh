# final evidence of round 2 on HEAD (A8 dry pass, verify_sample at 4 CTAs per SM): every workload, reference arm, ncu launch list + full capture, timelines, smoke, GPU suite
set -x
python -m paper_2604_09731_b200._build > /dev/null
timeout 900 python bench.py > gpurun_out/r5d_bench_cfg3.json 2> gpurun_out/r5d_bench_cfg3.err
for w in cfg2_llama8b_b1 cfg4_qwen2vl_b12 cfg5_r1distill_b256; do
  timeout 600 python bench.py --workload $w --no-hbm-regime > gpurun_out/r5d_bench_$w.json 2> gpurun_out/r5d_bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r5d_bench_reference.json 2> gpurun_out/r5d_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r5d_launches.csv python bench.py --steps 3 --warmup 3 --steps-only > gpurun_out/r5d_launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r5d_full_step python bench.py --steps 2 --warmup 3 --steps-only > gpurun_out/r5d_full.log 2>&1
tail -2 gpurun_out/r5d_full.log
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r5d_timeline_cfg3.txt 2>&1
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py cfg2_llama8b_b1 > gpurun_out/r5d_timeline_cfg2.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r5d_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r5d_smoke.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r5d_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r5d_pytest_gpu.txt
