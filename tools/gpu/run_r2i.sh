python -m paper_2604_09731_b200._build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_gpu_dflash.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2i_cfg3.json 2>&1
timeout 900 python bench.py --workload cfg5_r1distill_b256 --steps 50 --no-cpu-baseline --e2e-steps 0 --no-hbm-regime > gpurun_out/r2i_cfg5.json 2>&1
