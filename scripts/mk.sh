#!/bin/bash
# Build libapsp_warm.so from the repo root; print errors and fail loudly.
cd "$(dirname "$0")/.." || exit 1
out=$(python paper_2412_15122_b200/build.py 2>&1)
rc=$?
if [ $rc -ne 0 ]; then echo "$out" | grep -iE "error|warning" | head -30; echo "BUILD FAILED"; exit 1; fi
echo "built: $(ls -la --time-style=+%T paper_2412_15122_b200/libapsp_warm.so | awk '{print $6}')"
