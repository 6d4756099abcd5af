#!/bin/bash
# Out-of-place tail-pool claims: one 32-group warp unit (default) vs whole pages (KG_POOL_PAGES=1 build).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-pool_pages}; mkdir -p $O
for rep in 1 2; do for v in base pp; do
  L=paper_1305_3345_b200/libkgpu.so; [ $v = pp ] && L=build/tpb/libkgpu_pp.so
  for w in c2 ecb_dec c2_keyed; do
    KG_LIBKGPU=$L timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-check > $O/${w}_${v}_${rep}.json 2>/dev/null
  done
done; done
KG_LIBKGPU=build/tpb/libkgpu_pp.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q > $O/pytest_pp.log 2>&1; echo rc=$? >> $O/pytest_pp.log
