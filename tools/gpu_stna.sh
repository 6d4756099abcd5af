cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
# (historical: the KG_STNA variant was reverted after this A/B; profiles/r1_tex/README.md)
O=gpurun_out/stna; mkdir -p $O
for rep in 1 2; do for t in 1 0; do
  KG_STNA=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/c2_stna${t}_$rep.json 2>/dev/null
done; done
KG_STNA=1 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "cbc_device" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
