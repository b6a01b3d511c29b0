set -x
python -m paper_2604_09731_b200._build > /dev/null
timeout 900 python bench.py > gpurun_out/r2e_bench_cfg3.json 2> gpurun_out/r2e_bench_cfg3.err
timeout 900 python bench.py --workload cfg5_r1distill_b256 --steps 50 --no-hbm-regime > gpurun_out/r2e_bench_cfg5.json 2> gpurun_out/r2e_bench_cfg5.err
timeout 600 python bench.py --workload cfg2_llama8b_b1 --steps 100 --no-hbm-regime --no-cpu-baseline > gpurun_out/r2e_bench_cfg2.json 2> gpurun_out/r2e_bench_cfg2.err
timeout 600 python bench.py --workload cfg4_qwen2vl_b12 --steps 100 --no-hbm-regime --no-cpu-baseline > gpurun_out/r2e_bench_cfg4.json 2> gpurun_out/r2e_bench_cfg4.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2e_ref.json 2> gpurun_out/r2e_ref.err
tail -3 gpurun_out/r2e_*.err
