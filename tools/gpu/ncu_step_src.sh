# ncu source-level stall sampling of one cfg3 step kernel launch at the finest sampling interval
set -x
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --warp-sampling-max-passes 20 \
  --warp-sampling-buffer-size 536870912 --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 \
  -o gpurun_out/step_src python tools/probes/step_diag.py > gpurun_out/ncu_step_src.log 2>&1
tail -5 gpurun_out/ncu_step_src.log
