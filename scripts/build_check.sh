#!/bin/bash
# build the device library; non-zero exit (and the nvcc error) on failure
cd "$(dirname "$0")/.." && python -m paper_2105_01271_b200.build > /tmp/spb_build.log 2>&1 || { grep -B2 -A3 error /tmp/spb_build.log | head -30; exit 1; }
echo "build ok: $(tail -1 /tmp/spb_build.log)"
