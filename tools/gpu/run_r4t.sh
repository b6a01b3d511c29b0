# ncu --set full of one verify_sample (T = 1) launch at cfg3
python -m paper_2604_09731_b200._build > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:verify_kernel -s 45 -c 1 -o gpurun_out/r4t_vsample python bench.py --no-cpu-baseline --no-hbm-regime --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/r4t_ncu.log 2>&1
tail -3 gpurun_out/r4t_ncu.log
