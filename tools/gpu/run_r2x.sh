# consumer microbenchmark: timing + one ncu --set full capture of a throughput-mode launch (source-level)
set -x
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -I paper_2604_09731_b200/csrc"
$NV tools/ubench/consume.cu -o /tmp/consume || exit 1
$NV -DCONSUME_COUNTS=1 tools/ubench/consume.cu -o /tmp/consume_cnt
$NV -DCONSUME_EXPERIMENT=2 tools/ubench/consume.cu -o /tmp/consume_sm
$NV -DCONSUME_EXPERIMENT=1 tools/ubench/consume.cu -o /tmp/consume_st
for b in consume consume_cnt consume_sm consume_st; do echo "== $b"; timeout 60 /tmp/$b 152064 8; timeout 60 /tmp/$b 128256 8; done > gpurun_out/r2x_consume.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k consume_bench -s 3 -c 1 -o gpurun_out/r2x_consume /tmp/consume 152064 8 > gpurun_out/r2x_ncu.log 2>&1
tail -3 gpurun_out/r2x_ncu.log
