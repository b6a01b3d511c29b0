SMART_PROBES=1 python -m paper_2604_09731_b200._build > /dev/null
CHEAP=1 SMART_PROBES=1 timeout 300 python tools/probes/probe_cfg5_select.py > gpurun_out/r3zb_cfg5_select.txt 2>&1
CHEAP=1 SMART_PROBES=1 SMART_DEBUG_MODE=9 timeout 300 python tools/probes/probe_cfg5_select.py >> gpurun_out/r3zb_cfg5_select.txt 2>&1
git -C . status > /dev/null 2>&1
