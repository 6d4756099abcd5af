#!/bin/bash
# Threads per CTA of the CBC-encrypt chain kernel (KG_CHAIN_TPB builds under build/tpb/).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-chain_tpb}; mkdir -p $O
for rep in 1 2; do for T in 1024 512 768; do
  L=paper_1305_3345_b200/libkgpu.so; [ $T != 1024 ] && L=build/tpb/libkgpu_c$T.so
  KG_LIBKGPU=$L timeout 300 python bench.py --workload c3 --no-cpu-baseline --no-e2e > $O/c3_${T}_${rep}.json 2>/dev/null
done; done
