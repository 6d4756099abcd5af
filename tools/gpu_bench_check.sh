#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-bcheck}; mkdir -p $O
for w in c2 c3 ecb_enc c2_keyed c3_keyed; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/$w.json 2> $O/$w.err
done
timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.json 2> $O/c5.err
KG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/n2.json 2> $O/n2.err
