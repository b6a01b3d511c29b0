# ncu --set full capture of one persistent step kernel launch (cfg3), source-level
set -x
python -m paper_2604_09731_b200._build > /dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 \
  -o gpurun_out/step_full python tools/probes/step_diag.py > gpurun_out/ncu_step.log 2>&1
tail -5 gpurun_out/ncu_step.log
