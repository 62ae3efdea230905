#!/bin/bash
# rebuild libkkt.so in-tree and report errors / spills
cd "$(dirname "$0")/.." || exit 1
python -c "from paper_2405_14236_b200 import build as b; b.build(force=True)" 2>&1 | grep -iE "error|warning|Traceback" | head -20
grep -B3 "spill" paper_2405_14236_b200/ptxas_report.txt | grep -E "entry|spill" | grep -B1 -E " [1-9][0-9]* bytes spill" | head
echo "DMMA: $(cuobjdump -sass paper_2405_14236_b200/libkkt.so | grep -c DMMA)"
