# verify_sample: hash before its last xor-shift in the candidate mask: sampling tests, bench (verify_sample_T1_ms)
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 python -m pytest tests/test_gpu_sampling.py -x -q > gpurun_out/r4w_sampling.txt 2>&1; echo "rc $?" >> gpurun_out/r4w_sampling.txt
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r4w_bench_$i.json 2>/dev/null
done
timeout 300 python bench.py --workload cfg5_r1distill_b256 --no-cpu-baseline > gpurun_out/r4w_bench_cfg5.json 2>/dev/null
