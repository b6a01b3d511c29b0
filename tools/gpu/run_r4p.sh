SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r4p_timeline_cfg3.txt 2>&1
