#!/bin/bash
# CBC vs ECB decrypt, in place vs out of place, at the C2 size.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-inplace}; mkdir -p $O
for rep in 1 2; do for w in c2 c2_inplace ecb_dec ecb_dec_inplace; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-check > $O/${w}_${rep}.json 2>/dev/null
done; done
