#!/bin/bash
# randomised multi-process runs of the product All-Scan path (ZecoRank + AllScanP2P over CUDA IPC, all ranks on
# one GPU): every output / gradient against the f64 oracle and the single-process list form
i=0
for cfg in "2 2 512 1" "3 4 320 1" "4 2 1024 2" "2 6 768 2" "3 1 2048 1" "4 8 256 2" "2 3 4096 1" "5 2 640 1"; do
  set -- $cfg; P=$1; H=$2; L=$3; G=$4
  out=$(python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
        --master-port $((29801 + i)) scripts/spmd_ipc_check.py --same-device --rounds 2 --seq $L --heads $H \
        --overlap-groups $G --oracle 2>&1)
  ok=$(echo "$out" | grep -c "SPMD IPC check OK")
  errs=$(echo "$out" | grep "oracle " | sed 's/.*oracle \([a-z]*\): rel err \(.*\)/\1=\2/' | tr '\n' ' ')
  echo "{\"P\": $P, \"heads\": $H, \"tokens_per_rank\": $L, \"overlap_groups\": $G, \"ok\": $ok, \"oracle\": \"$errs\"}"
  i=$((i + 1))
done
