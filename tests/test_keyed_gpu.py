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
