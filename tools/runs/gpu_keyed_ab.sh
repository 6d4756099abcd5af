cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/keyed1; mkdir -p $O
timeout 900 python -m pytest tests/test_keyed_gpu.py -x -q > $O/pytest_keyed.log 2>&1; echo "rc=$?" >> $O/pytest_keyed.log
for v in 0 1 2; do
  for w in c2_keyed c3_keyed; do
    KG_KEYED=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_${w}_v$v.json 2> $O/bench_${w}_v$v.err
  done
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c2.json 2>&1
