# cfg5 standalone selection phase cycles (SMART_PROBES=1 build), cheap-node cost (trees grow)
SMART_PROBES=1 python -m paper_2604_09731_b200._build --force > /dev/null 2>&1 || SMART_PROBES=1 python -m paper_2604_09731_b200._build > /dev/null
CHEAP=1 SMART_PROBES=1 timeout 300 python tools/probes/probe_cfg5_select.py > gpurun_out/r3w_cfg5_select.txt 2>&1
