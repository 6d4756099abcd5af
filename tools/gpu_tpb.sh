#!/bin/bash
# Threads per CTA of the block-pair kernels (KG_PAIR_TPB builds under build/tpb/) with texture loads.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-tpb}; mkdir -p $O
for rep in 1 2; do
  for T in 512 384 640 768; do
    L=paper_1305_3345_b200/libkgpu.so; [ $T != 512 ] && L=build/tpb/libkgpu_$T.so
    for w in c2 ecb_dec; do
      KG_LIBKGPU=$L timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/${w}_${T}_${rep}.json 2>/dev/null
    done
  done
done
