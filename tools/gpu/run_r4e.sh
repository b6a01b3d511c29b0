# peer exchange (NEXT #4): in-process and two-process (IPC) bit-identity with G = 1, then the suite
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 python -m pytest tests/test_gpu_peer_exchange.py -x -q > gpurun_out/r4e_peer.txt 2>&1; rc=$?; echo "peer rc $rc" >> gpurun_out/r4e_peer.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4e_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r4e_pytest_gpu.txt
tail -n 3 gpurun_out/r4e_pytest_gpu.txt
