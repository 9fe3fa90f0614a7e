#!/usr/bin/env bash
# Round-2 measurement pass on one B200 (bash scripts/profile_r02.sh <tag>) (gpurun): bench lines (Reddit bf16 / fp32, products bf16 = DRAM-resident
# gathers), the gather ceilings, single-GPU emulation of the m = 8 job (every rank, ldg2 and random partitions),
# ncu launch lists (bench and emulation) and ncu --set full captures of the SpMM / GEMM launches.
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python bench.py --steps 20 --warmup 5 --json-out "$OUT/bench_bf16.json" > "$OUT/bench_bf16.log" 2>&1
python bench.py --steps 10 --warmup 3 --prec fp32 --no-cpu-baseline --json-out "$OUT/bench_fp32.json" > "$OUT/bench_fp32.log" 2>&1
python bench.py --steps 10 --warmup 3 --config products --no-cpu-baseline --json-out "$OUT/bench_products.json" > "$OUT/bench_products.log" 2>&1
# A/B: TMA tile::gather4 staged SpMM (bf16 256-wide rows) on the L2-resident (Reddit) and DRAM-resident shapes
BNS_SPMM_TMA=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --json-out "$OUT/bench_bf16_tma.json" > "$OUT/bench_bf16_tma.log" 2>&1
BNS_SPMM_TMA=1 python bench.py --steps 10 --warmup 3 --config yelp --no-cpu-baseline --no-e2e --json-out "$OUT/bench_yelp_tma.json" > "$OUT/bench_yelp_tma.log" 2>&1
python bench.py --steps 10 --warmup 3 --config yelp --no-cpu-baseline --no-e2e --json-out "$OUT/bench_yelp.json" > "$OUT/bench_yelp.log" 2>&1
./build/gather_ceiling 20 > "$OUT/gather_ceiling.jsonl" 2>&1
python scripts/ceiling_rmat.py > "$OUT/ceiling_rmat.jsonl" 2>&1
for part in ldg2 random; do
  timeout 1500 python scripts/emulate_rank.py --m 8 --p 0.1 --ranks all --partition $part --cache-x0 --no-timing \
      >> "$OUT/emulate_m8_all.jsonl" 2>> "$OUT/emulate.err"
done
timeout 900 python scripts/emulate_rank.py --m 8 --p 1.0 0.1 0.01 0.0 --ranks 0 --partition ldg2 --cache-x0 \
    > "$OUT/emulate_m8_rank0_phases.jsonl" 2>> "$OUT/emulate.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py launches "$OUT/launches.csv" "$OUT/launches.txt" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/emu_launches.csv" \
    python scripts/emulate_rank.py --m 8 --p 0.1 --ranks 0 --partition ldg2 --cache-x0 --no-timing --steps 2 --warmup 1 \
    > /dev/null 2>&1
python scripts/ncu_summary.py launches "$OUT/emu_launches.csv" "$OUT/emu_launches.txt" > /dev/null
# the 8 k_spmm launches of one whole epoch (the second): their DRAM bytes are the step's SpMM traffic
timeout 1200 ncu --set full --clock-control none -k k_spmm -s 8 -c 8 \
    -o "$OUT/prof_spmm" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py full "$OUT/prof_spmm.ncu-rep" "$OUT/spmm.json" k_spmm > /dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_tc -s 16 -c 6 -o "$OUT/prof_gemm" \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py full "$OUT/prof_gemm.ncu-rep" "$OUT/gemm.json" > /dev/null
timeout 600 ncu --set full --clock-control none -k regex:"k_induce_count|k_induce_scatter|k_sample_fused|k_segs_fused" -s 4 -c 4 \
    -o "$OUT/prof_induce" python scripts/emulate_rank.py --m 8 --p 0.1 --ranks 0 --partition ldg2 --cache-x0 \
    --steps 2 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py full "$OUT/prof_induce.ncu-rep" "$OUT/induce.json" > /dev/null
rm -f "$OUT"/*.ncu-rep "$OUT"/*.csv
du -sh "$OUT"/*
