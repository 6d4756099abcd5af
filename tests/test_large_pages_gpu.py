"""Pages far larger than the workloads' 4 KiB (the ABI takes any positive
multiple of 16 up to 2^32-16 bytes): 64 KiB .. 4 MiB pages, even and odd
block counts, every kernel family (block pairs, one block per lane, chains,
mixed keys), device / pinned / in place, against the oracle on every byte.
Chains of 262,144 blocks exercise the per-thread page loop; the block-pair
kernels' 32-bit group index within a page and the per-page pool units."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, gpu_pages, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu

SHAPES = [(8, 1 << 20), (3, (1 << 20) + 16), (2, 4 << 20), (40, 65536), (5, 65536 + 48)]


@pytest.mark.parametrize("n,pb", SHAPES)
@pytest.mark.parametrize("direction,mode", [(1, 0), (0, 0), (1, 1), (0, 1)])
def test_large_pages_device(n, pb, direction, mode):
    key = synth.make_key(16, seed=n + pb)
    data = synth.make_pages(n, pb, seed=pb + 1)
    ivs = synth.make_ivs(n, seed=n + 2) if mode == 0 else None
    exp = oracle_pages(direction, mode, key, data, n, pb, ivs)
    got = gpu_pages(direction, mode, key, data, n, pb, ivs, where="device")
    assert first_mismatch(got, exp) is None
    got = gpu_pages(direction, mode, key, data, n, pb, ivs, where="device", inplace=True)
    assert first_mismatch(got, exp) is None


@pytest.mark.parametrize("n,pb", [(8, 1 << 20), (3, (1 << 20) + 16)])
@pytest.mark.parametrize("direction", [0, 1])
def test_large_pages_pinned(n, pb, direction):
    key = synth.make_key(32, seed=n * 3 + pb)
    data = synth.make_pages(n, pb, seed=pb + 5)
    ivs = synth.make_ivs(n, seed=n + 6)
    exp = oracle_pages(direction, 0, key, data, n, pb, ivs)
    got = gpu_pages(direction, 0, key, data, n, pb, ivs, where="pinned")
    assert first_mismatch(got, exp) is None


@pytest.mark.parametrize("direction,mode", [(1, 0), (0, 0), (0, 1)])
def test_large_pages_keyed(direction, mode):
    kg, torch = kg_ready()
    n, pb = 6, 1 << 20
    keys = {k: synth.make_key(16, seed=700 + k) for k in (1, 2, 3)}
    for k, v in keys.items():
        kg.set_key(k, v)
    ids = np.array([1, 2, 3, 3, 2, 1], dtype=np.uint16)
    data = synth.make_pages(n, pb, seed=701)
    ivs = synth.make_ivs(n, seed=702) if mode == 0 else None
    exp = np.empty_like(data)
    for p in range(n):
        sl = slice(p * pb, (p + 1) * pb)
        exp[sl] = oracle_pages(direction, mode, keys[int(ids[p])], data[sl], 1, pb,
                               None if ivs is None else ivs[16 * p:16 * p + 16])
    x = torch.from_numpy(data).cuda()
    out = torch.empty_like(x)
    tid = torch.from_numpy(ids.astype(np.int16)).cuda()
    tiv = None if ivs is None else torch.from_numpy(ivs).cuda()
    kg.wait(kg.submit_pages_keyed(direction, mode, x, out, n, pb, tiv, tid, 16))
    torch.cuda.synchronize()
    assert first_mismatch(out.cpu().numpy(), exp) is None
