#!/bin/bash
# ncu --set full of the mixed-key and ECB kernels (traffic + pipe evidence).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-ncu_more}; mkdir -p $O
run() {  # name regex workload
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $O/prof_$1 \
    python bench.py --workload $3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$1.log 2>&1
}
run c2_keyed kg_keyed_pair c2_keyed
run c3_keyed kg_keyed_chain c3_keyed
run ecb_dec kg_blockpar ecb_dec
run ecb_enc kg_blockpar ecb_enc
echo done > $O/done.txt
