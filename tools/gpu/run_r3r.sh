# team-merge probes: tournament (default) vs parallel ranks (SMART_DEBUG_MODE=8), 3 timelines each
python -m paper_2604_09731_b200._build > /dev/null
for i in 1 2 3; do
SMART_PROBES=1 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r3r_tl_tourn_$i.txt 2>&1
SMART_PROBES=1 SMART_DEBUG_MODE=8 timeout 200 python tools/probes/step_timeline.py > gpurun_out/r3r_tl_rank_$i.txt 2>&1
done
