# consume ubench: the throughput headroom of a near-oracle top-k bound (CONSUME_EXPERIMENT=4)
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -I paper_2604_09731_b200/csrc"
$NV tools/ubench/consume.cu -o /tmp/consume && timeout 60 /tmp/consume 152064 8 > gpurun_out/r3t.txt 2>&1
$NV -DCONSUME_EXPERIMENT=4 tools/ubench/consume.cu -o /tmp/consume4 && timeout 60 /tmp/consume4 152064 8 >> gpurun_out/r3t.txt 2>&1
$NV -DCONSUME_EXPERIMENT=4 -DCONSUME_COUNTS=1 tools/ubench/consume.cu -o /tmp/consume4c && timeout 60 /tmp/consume4c 152064 8 >> gpurun_out/r3t.txt 2>&1
$NV -DCONSUME_COUNTS=1 tools/ubench/consume.cu -o /tmp/consumec && timeout 60 /tmp/consumec 152064 8 >> gpurun_out/r3t.txt 2>&1
$NV -DCONSUME_EXPERIMENT=2 tools/ubench/consume.cu -o /tmp/consume2 && timeout 60 /tmp/consume2 152064 8 >> gpurun_out/r3t.txt 2>&1
