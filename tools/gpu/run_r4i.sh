# full-mantissa fp32 parity + suite
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fp32_full" > gpurun_out/r4i_fp32full.txt 2>&1; echo "rc $?" >> gpurun_out/r4i_fp32full.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4i_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r4i_pytest_gpu.txt
