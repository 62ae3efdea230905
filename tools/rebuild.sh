#!/bin/bash
# rebuild libkkt.so in-tree; exit 1 (and say so) if nvcc fails; report spills and DMMA count
cd "$(dirname "$0")/.." || exit 1
out=$(python -c "from paper_2405_14236_b200 import build as b; b.build(force=True)" 2>&1)
if [ $? -ne 0 ]; then echo "$out" | grep -E "error" | head -20; echo "BUILD FAILED"; exit 1; fi
grep -B3 "spill" paper_2405_14236_b200/ptxas_report.txt | grep -E "entry|spill" | grep -B1 -E " [1-9][0-9]* bytes spill" | head
echo "DMMA: $(cuobjdump -sass paper_2405_14236_b200/libkkt.so | grep -c DMMA)"
