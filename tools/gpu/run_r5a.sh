# per-CTA timeline of the A8 stream inside the step kernel (probe build, SMART_DEBUG_MODE=9)
SMART_PROBES=1 SMART_DEBUG_MODE=9 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r5a_timeline_a8.txt 2>&1
