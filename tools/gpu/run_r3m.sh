# consumer first-chunk phase stamps (CTA 0, warp 0) in the latency mode of the consume ubench
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -I paper_2604_09731_b200/csrc"
$NV -DCONSUME_STAMPS=1 tools/ubench/consume.cu -o /tmp/consume_st && timeout 60 /tmp/consume_st 128256 8 > gpurun_out/r3m_stamps.txt 2>&1
$NV tools/ubench/consume.cu -o /tmp/consume && timeout 60 /tmp/consume 128256 8 >> gpurun_out/r3m_stamps.txt 2>&1
