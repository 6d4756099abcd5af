#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-tex_ab2}; mkdir -p $O
cat > /tmp/props.cu <<'EOC'
#include <cstdio>
#include <cuda_runtime.h>
int main(){cudaDeviceProp p; cudaGetDeviceProperties(&p,0); printf("{\"maxTexture1DLinear\": %d, \"textureAlignment\": %zu}\n", p.maxTexture1DLinear, p.textureAlignment);}
EOC
nvcc -o /tmp/props /tmp/props.cu && /tmp/props > $O/props.json
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for t in 1 0; do
  KG_TEXIN=$t timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5_tex$t.json 2>$O/bench_c5_tex$t.err
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c2.json 2>$O/bench_c2.err
