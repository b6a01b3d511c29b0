# cfg5 (b = 256, per-layer path): ncu launch list of a few steps (per-kernel durations)
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r3v_cfg5_launches.csv python bench.py --workload cfg5_r1distill_b256 --steps 2 --warmup 1 --steps-only > gpurun_out/r3v_cfg5.log 2>&1
tail -2 gpurun_out/r3v_cfg5.log
