#!/bin/bash
# A/B of librgnn.so build variants (variants/*.so) on the bench's phase times.
#   bash tools/variants.sh <config> ...      (BENCH_ARGS="--model hgt" for extra bench flags)
cp paper_2301_06284_b200/librgnn.so /tmp/librgnn_base.so
for f in /tmp/librgnn_base.so variants/*.so; do
  cp $f paper_2301_06284_b200/librgnn.so
  for c in "$@"; do
    r=$(timeout 600 python bench.py --config $c $BENCH_ARGS --steps 20 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
    echo "$(basename $f) $c $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: v for k, v in d["phases_ms_per_step"].items() if k in ("aggregate","bwd_fused","bwd_tm","dst_term","gemm_fwd","hgt_bwd_walk","hgt_bwd_src","hgt_bwd_dw_rel")})' 2>&1)"
  done
done
cp /tmp/librgnn_base.so paper_2301_06284_b200/librgnn.so
