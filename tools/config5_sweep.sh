#!/bin/bash
# BASELINE config 5: the synthetic random-strategy sweep, 10^4 .. 10^9 candidates
# in total (strong scaling: n / N per GPU), at 1/2/4 GPUs of one box, through
# bench.py's fused step (1.6T@2048). One JSON line per (total, N) on stdout.
#   tools/config5_sweep.sh "1 2 4" > profiles/r02_config5.jsonl
GPUS=${1:-"1 2 4"}
for N in $GPUS; do
  for total in 10000 100000 1000000 10000000 100000000 1000000000; do
    n=$((total / N))
    if [ $total -le 10000000 ]; then S="--steps 200 --warmup 20"; elif [ $total -le 100000000 ]; then S="--steps 20 --warmup 5"; else S="--steps 5 --warmup 3"; fi
    B="--candidates-per-gpu $n $S --no-search --no-pyref --no-cpu --no-e2e --no-parity"
    if [ $N = 1 ]; then
      timeout 900 python bench.py $B 2>/dev/null | tail -1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29600 + N)) bench.py --gpus $N $B 2>/dev/null | grep "^{" | tail -1
    fi
  done
done
