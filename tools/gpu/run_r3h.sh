# i-cache experiment: step kernel at occupancy 1 (the selection CTA alone on its SM) vs 2
python -m paper_2604_09731_b200._build > /dev/null
SMART_PROBES=1 SMART_STEP_OCC=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r3h_timeline_occ1.txt 2>&1
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r3h_timeline_occ2.txt 2>&1
