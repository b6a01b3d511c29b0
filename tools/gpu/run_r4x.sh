# final evidence of the session: smoke, full GPU suite, bench cfg3 (full line), reference arm
set -x
python -m paper_2604_09731_b200._build > /dev/null
timeout 300 python __graft_entry__.py smoke > gpurun_out/r4x_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/r4x_smoke.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r4x_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r4x_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r4x_bench_cfg3.json 2> gpurun_out/r4x_bench_cfg3.err
timeout 600 python bench.py --workload cfg5_r1distill_b256 --no-hbm-regime > gpurun_out/r4x_bench_cfg5.json 2> gpurun_out/r4x_bench_cfg5.err
