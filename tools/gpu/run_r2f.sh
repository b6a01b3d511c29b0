python -m paper_2604_09731_b200._build > /dev/null
timeout 900 python bench.py > gpurun_out/r2e_bench_cfg3.json 2> gpurun_out/r2e_bench_cfg3.err
timeout 900 python bench.py --workload cfg5_r1distill_b256 --steps 50 --no-hbm-regime > gpurun_out/r2e_bench_cfg5.json 2> gpurun_out/r2e_bench_cfg5.err
tail -n 3 gpurun_out/r2e_bench_cfg3.err gpurun_out/r2e_bench_cfg5.err
