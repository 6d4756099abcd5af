"""Mixed-key batches (row f1 extension): page p under key
key_ids[p].  Every page is compared with the oracle under its own key."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu


def expected(direction, mode, keys, ids, data, n, pb, ivs):
    out = np.empty_like(data)
    for p in range(n):
        sl = slice(p * pb, (p + 1) * pb)
        iv = None if ivs is None else ivs[16 * p:16 * p + 16]
        out[sl] = oracle_pages(direction, mode, keys[int(ids[p])], data[sl], 1, pb, iv)
    return out


@pytest.mark.parametrize("key_bytes", [16, 24, 32])
@pytest.mark.parametrize("direction,mode", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("n,pb", [(37, 4096), (300, 512), (5, 48), (300, 256), (1500, 4096)])
def test_keyed_parity(key_bytes, direction, mode, n, pb):
    kg, torch = kg_ready()
    key_set = [10, 11, 200, 255, 0]
    keys = {}
    for i, kid in enumerate(key_set):
        keys[kid] = synth.make_key(key_bytes, seed=1000 + 7 * i + key_bytes)
        kg.set_key(kid, keys[kid])
    rng = np.random.default_rng(n + pb + key_bytes)
    ids = np.array(key_set, dtype=np.uint16)[rng.integers(0, len(key_set), n)]
    data = synth.make_pages(n, pb, seed=n * 3 + pb)
    ivs = synth.make_ivs(n, seed=n * 5) if mode == 0 else None
    exp = expected(direction, mode, keys, ids, data, n, pb, ivs)
    x = torch.from_numpy(data).cuda()
    out = torch.empty_like(x)
    tid = torch.from_numpy(ids.astype(np.int16)).cuda()
    tiv = None if ivs is None else torch.from_numpy(ivs).cuda()
    kg.wait(kg.submit_pages_keyed(direction, mode, x, out, n, pb, tiv, tid, key_bytes))
    torch.cuda.synchronize()
    assert first_mismatch(out.cpu().numpy(), exp) is None
    # in place, ids + ivs in pinned host memory
    y = x.clone()
    hid = tid.cpu().pin_memory()
    hiv = None if tiv is None else tiv.cpu().pin_memory()
    kg.wait(kg.submit_pages_keyed(direction, mode, y, y, n, pb, hiv, hid, key_bytes))
    torch.cuda.synchronize()
    assert first_mismatch(y.cpu().numpy(), exp) is None


def test_keyed_errors_and_snapshot():
    kg, torch = kg_ready()
    n, pb = 8, 4096
    k_a, k_b = synth.make_key(16, seed=1), synth.make_key(16, seed=2)
    kg.set_key(20, k_a)
    kg.set_key(21, synth.make_key(32, seed=3))
    x = torch.from_numpy(synth.make_pages(n, pb)).cuda()
    iv = torch.from_numpy(synth.make_ivs(n)).cuda()
    out = torch.empty_like(x)
    ids = torch.full((n,), 20, dtype=torch.int16, device="cuda")
    t = kg.submit_pages_keyed(1, 0, x, out, n, pb, iv, ids, 16)
    kg.set_key(20, k_b)                       # re-key after submit: the batch keeps k_a
    kg.wait(t)
    exp = oracle_pages(1, 0, k_a, x.cpu().numpy(), n, pb, iv.cpu().numpy())
    assert first_mismatch(out.cpu().numpy(), exp) is None
    ids[3] = 21                               # a key of another size
    assert kg.wait_raw(kg.submit_pages_keyed(1, 0, x, out, n, pb, iv, ids, 16)) == kg.ENOKEY
    ids[3] = 99                               # an unset key
    kg.raw_lib()
    assert kg.wait_raw(kg.submit_pages_keyed(1, 0, x, out, n, pb, iv, ids, 16)) == kg.ENOKEY
    ids[3] = 20
    kg.wait(kg.submit_pages_keyed(1, 0, x, out, n, pb, iv, ids, 16))   # ok again
    lib = kg.raw_lib()
    assert lib.kg_submit_pages_keyed(1, 0, x.data_ptr(), out.data_ptr(), n, pb, iv.data_ptr(),
                                     ids.data_ptr() + 1, 16, None) == kg.EINVAL    # misaligned ids
    assert lib.kg_submit_pages_keyed(1, 0, x.data_ptr(), out.data_ptr(), n, pb, iv.data_ptr(),
                                     ids.data_ptr(), 20, None) == kg.EINVAL        # bad key size


def test_keyed_const_keys_cross_stream():
    """The constant-bank key copy (KG_KEYED=2) is refilled when the snapshot
    or the direction changes; the refill on one stream must wait for a launch
    still reading the old copy on another stream."""
    kg, torch = kg_ready()
    n, pb = 4096, 4096                         # 16 MiB: long enough to still run when the refill is queued
    k_a, k_b = synth.make_key(16, seed=31), synth.make_key(16, seed=32)
    kg.set_key(40, k_a)
    data = synth.make_pages(n, pb, seed=77)
    ivs = synth.make_ivs(n, seed=78)
    x = torch.from_numpy(data).cuda()
    iv = torch.from_numpy(ivs).cuda()
    ids = torch.full((n,), 40, dtype=torch.int16, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2, o3 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    torch.cuda.synchronize()
    t1 = kg.submit_pages_keyed(1, 0, x, o1, n, pb, iv, ids, 16, s1)      # dec, key A (copy: A/dec)
    kg.set_key(40, k_b)
    t2 = kg.submit_pages_keyed(1, 0, x, o2, n, pb, iv, ids, 16, s2)      # dec, key B (refill on s2)
    t3 = kg.submit_pages_keyed(0, 1, x, o3, n, pb, None, ids, 16, s1)    # ECB enc, key B (refill on s1)
    for t in (t1, t2, t3):
        kg.wait(t)
    torch.cuda.synchronize()
    assert first_mismatch(o1.cpu().numpy(), oracle_pages(1, 0, k_a, data, n, pb, ivs)) is None
    assert first_mismatch(o2.cpu().numpy(), oracle_pages(1, 0, k_b, data, n, pb, ivs)) is None
    assert first_mismatch(o3.cpu().numpy(), oracle_pages(0, 1, k_b, data, n, pb, None)) is None


@pytest.mark.parametrize("variant", ["0", "1"])
def test_keyed_other_variants(variant):
    """The A/B alternatives behind KG_KEYED (read once per process) stay
    correct: run a slice of the parity matrix in a child process."""
    import os
    import subprocess
    import sys
    kg_ready()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KG_KEYED=variant)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_keyed_gpu.py"), "-k", "test_keyed_parity and (37 or 1500)"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("direction,mode", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("path", ["staged", "auto"])
def test_keyed_host_batches(direction, mode, path):
    """Mixed-key batches with pinned host pages (rows f1 x f4): through the
    staging pipeline (chunk launches each read their slice of the ids) or,
    under AUTO, zero-copy below the threshold and staged above it."""
    kg, torch = kg_ready()
    key_set = [3, 77, 254]
    keys = {}
    for i, kid in enumerate(key_set):
        keys[kid] = synth.make_key(16, seed=900 + i)
        kg.set_key(kid, keys[kid])
    n, pb = (9000, 4096) if path == "auto" else (1500, 4096)   # auto: 35 MiB > the 32 MiB zero-copy cap
    rng = np.random.default_rng(n + direction * 2 + mode)
    ids = np.array(key_set, dtype=np.uint16)[rng.integers(0, len(key_set), n)]
    data = synth.make_pages(n, pb, seed=n + 11)
    ivs = synth.make_ivs(n, seed=n + 12) if mode == 0 else None
    exp = expected(direction, mode, keys, ids, data, n, pb, ivs)
    hin = torch.from_numpy(data).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    hid = torch.from_numpy(ids.astype(np.int16)).pin_memory()
    hiv = None if ivs is None else torch.from_numpy(ivs).pin_memory()
    if path == "staged":
        kg.set_host_path(kg.HOST_STAGED)
        kg.set_pipeline(64 * 4096, 3)           # many chunks, slots wrap
    try:
        kg.wait(kg.submit_pages_keyed(direction, mode, hin, hout, n, pb, hiv, hid, 16))
        assert first_mismatch(hout.numpy(), exp) is None
        # in place, ids in device memory
        y = hin.clone().pin_memory()
        did = hid.cuda()
        kg.wait(kg.submit_pages_keyed(direction, mode, y, y, n, pb, hiv, did, 16))
        assert first_mismatch(y.numpy(), exp) is None
    finally:
        kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
