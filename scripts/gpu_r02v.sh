#!/bin/bash
# compute-sanitizer memcheck + synccheck over every kernel (incl. the aligned 3-way FULL epilogue)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02v
mkdir -p $O
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize_small.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize run ok" $O/sanitize_$tool.log | head -3
done
