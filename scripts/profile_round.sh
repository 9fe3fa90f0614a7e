#!/usr/bin/env bash
# Run on the GPU box (gpurun): bench line, ncu launch list, ncu --set full captures of one epoch's SpMM launches
# (forward 4 + backward 4 on the Reddit shape) and of the tcgen05 GEMMs, summarised to JSON on the box (the raw
# reports stay under the 64 MiB gpurun_out cap), plus the single-GPU per-rank emulation of the m=8 job.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python bench.py --steps 10 --warmup 3 --json-out "$OUT/bench.json" > "$OUT/bench.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py launches "$OUT/launches.csv" "$OUT/launches.txt" > /dev/null
# one epoch = 8 k_spmm launches (fwd: layer 1 (transform-first), 2, 3, 4 (transform-first); bwd: 4, 3, 2, 1);
# skip the warm-up epoch's 8
for part in fwd:8 bwd:12; do
    name=${part%%:*}; skip=${part##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k k_spmm -s "$skip" -c 4 \
        -o "$OUT/prof_spmm_$name" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
    python scripts/ncu_summary.py full "$OUT/prof_spmm_$name.ncu-rep" "$OUT/spmm_$name.json" > /dev/null
done
timeout 600 ncu --set full --clock-control none --import-source on -k k_gemm_tc -s 16 -c 6 -o "$OUT/prof_gemm" \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py full "$OUT/prof_gemm.ncu-rep" "$OUT/gemm.json" > /dev/null
rm -f "$OUT/prof_spmm_bwd.ncu-rep" "$OUT/prof_gemm.ncu-rep"
timeout 900 python scripts/emulate_rank.py --m 8 --p 1.0 0.1 0.01 0.0 --ranks 0 --partition random \
    > "$OUT/emulate_m8.jsonl" 2> "$OUT/emulate_m8.err"
du -sh "$OUT"/*
