mkdir -p gpurun_out/v7
for cfg in "2500 70000 37" "50000 2000000 128" "232965 30000000 602" "232965 114600000 602"; do
  set -- $cfg
  J="{\"wl\": {\"N\": $1, \"nnz\": $2, \"m\": 2, \"d0\": $3, \"C\": 41, \"seed\": 71}, \"dims\": [$3, 256, 41], \"layer\": 0, \"prec\": 1, \"draws\": [[\"bns\", 0.1]], \"out\": \"/tmp/ipcp\"}"
  echo "== $cfg" >> gpurun_out/v7/probe.log
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tests/ipc_worker.py "$J" >> gpurun_out/v7/probe.log 2>&1
  echo "rc=$?" >> gpurun_out/v7/probe.log
done
