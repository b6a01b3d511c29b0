python -m paper_2604_09731_b200._build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r2n_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2n_bench_cfg3.json 2> gpurun_out/r2n_bench_cfg3.err
timeout 900 python bench.py --workload cfg5_r1distill_b256 --steps 50 --no-hbm-regime > gpurun_out/r2n_bench_cfg5.json 2> gpurun_out/r2n_bench_cfg5.err
timeout 600 python bench.py --workload cfg2_llama8b_b1 --steps 100 --no-hbm-regime > gpurun_out/r2n_bench_cfg2.json 2> gpurun_out/r2n_bench_cfg2.err
timeout 600 python bench.py --workload cfg4_qwen2vl_b12 --steps 100 --no-hbm-regime > gpurun_out/r2n_bench_cfg4.json 2> gpurun_out/r2n_bench_cfg4.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2n_ref.json 2> gpurun_out/r2n_ref.err
tail -n 2 gpurun_out/r2n_pytest_gpu.txt gpurun_out/r2n_smoke.txt
