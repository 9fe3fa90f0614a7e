#!/usr/bin/env bash
# Run on the GPU box (gpurun): bench line, ncu launch list, ncu --set full captures of the SpMM and tcgen05 GEMM,
# single-GPU per-rank emulation of the m=8 job.  Results land in gpurun_out/$TAG/ (summarised into profiles/ by
# scripts/ncu_summary.py on the CPU side).
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python bench.py --steps 10 --warmup 3 --json-out "$OUT/bench.json" > "$OUT/bench.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# one epoch = layer-1 fwd (3 column tiles), 3 hidden fwd, 3 bwd: skip the warm-up epoch's 7-9 launches
timeout 900 ncu --set full --clock-control none --import-source on -k k_spmm -s 9 -c 5 -o "$OUT/prof_spmm" \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_gemm_tc -s 21 -c 3 -o "$OUT/prof_gemm" \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 python scripts/emulate_rank.py --m 8 --p 1.0 0.1 0.01 0.0 --ranks 0 --partition random \
    > "$OUT/emulate_m8.jsonl" 2> "$OUT/emulate_m8.err"
du -sh "$OUT"/*
