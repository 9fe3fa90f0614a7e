#!/usr/bin/env bash
# Run on the GPU box: profile_round.sh (bench line, ncu launch list, ncu full SpMM / GEMM captures, m=8 rank-0
# emulation) and the emulation sweep over every rank of m = 2 / 4 / 8 at p in {1, 0.1, 0.01, 0} (input-halo cache on).
set -u
TAG=${1:-r01d}
bash scripts/profile_round.sh "$TAG"
for m in 2 4 8; do
    timeout 1200 python scripts/emulate_rank.py --m $m --p 1.0 0.1 0.01 0.0 --ranks all --partition random --cache-x0 \
        >> gpurun_out/$TAG/emulate_sweep.jsonl 2>> gpurun_out/$TAG/emulate_sweep.err
done
