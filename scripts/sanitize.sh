#!/usr/bin/env bash
# compute-sanitizer tier over scripts/sanitize_case.py; summaries to gpurun_out/$TAG/
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for tool in memcheck racecheck synccheck initcheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --kernel-name-exclude regex=2at6native \
        python scripts/sanitize_case.py > "$OUT/sanitize_$tool.log" 2>&1
    echo "$tool rc=$?" >> "$OUT/sanitize_summary.txt"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case ok" "$OUT/sanitize_$tool.log" >> "$OUT/sanitize_summary.txt"
done
cat "$OUT/sanitize_summary.txt"
