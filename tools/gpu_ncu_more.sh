#!/bin/bash
# ncu --set full of the mixed-key and ECB kernels (traffic + pipe evidence).
# usage: tools/gpu_ncu_more.sh OUT [keyed|modes]   (two reports per call: gpurun copies back <= 64 MiB)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-ncu_more}; mkdir -p $O
run() {  # name regex workload
  timeout 900 ncu --set full --clock-control none -k regex:$2 -s 3 -c 1 -o $O/prof_$1 \
    python bench.py --workload $3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$1.log 2>&1
}
if [ "${2:-keyed}" = keyed ]; then
  run c2_keyed kg_keyed_pair c2_keyed
  run c3_keyed kg_keyed_chain c3_keyed
else
  run ecb_dec kg_blockpar ecb_dec
  run ecb_enc kg_blockpar ecb_enc
fi
echo done > $O/done.txt
