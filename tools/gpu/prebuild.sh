#!/bin/bash
# build both library flavours locally; non-zero exit on any compile error (run before gpurun)
cd "$(dirname "$0")/../.." || exit 1
SMART_PROBES=1 python -m paper_2604_09731_b200._build > /tmp/pb1.log 2>&1 || { grep -E "error" /tmp/pb1.log | head; exit 1; }
python -m paper_2604_09731_b200._build > /tmp/pb2.log 2>&1 || { grep -E "error" /tmp/pb2.log | head; exit 1; }
echo prebuild ok
