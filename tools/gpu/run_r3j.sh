# T > 0 verify with Gumbel pruning: sampling parity, then the cfg3 bench (verify_sample_T1_ms)
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 python -m pytest tests/test_gpu_sampling.py -x -q > gpurun_out/r3j_sampling.txt 2>&1; rc=$?; echo "rc $rc" >> gpurun_out/r3j_sampling.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python bench.py --no-cpu-baseline --no-hbm-regime > gpurun_out/r3j_bench_cfg3.json 2> gpurun_out/r3j_bench_cfg3.err
timeout 600 python bench.py --workload cfg5_r1distill_b256 --no-cpu-baseline --no-hbm-regime > gpurun_out/r3j_bench_cfg5.json 2> gpurun_out/r3j_bench_cfg5.err
