"""Element-by-element parity of the CUDA path (through the C ABI) with the
oracle on seeded inputs.  Bit-exact: AES is integer work.
Sizes span several warp units / CTAs with ragged tails; page sizes include
the degenerate 16-byte page and sizes that are not multiples of 512 B."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, gpu_pages, oracle_pages

pytestmark = pytest.mark.gpu

SHAPES = [(1, 16), (1, 4096), (2, 32), (3, 48), (16, 4096), (31, 4096), (33, 512), (149, 4096),
          (300, 4096), (97, 8192), (5, 65536), (1000, 16), (257, 496), (4096, 1024), (1500, 4096)]


@pytest.mark.parametrize("n,pb", SHAPES)
@pytest.mark.parametrize("key_bytes", [16, 24, 32])
@pytest.mark.parametrize("direction", [0, 1])
def test_cbc_device(direction, key_bytes, n, pb):
    seed = 1000 * n + pb + key_bytes + direction
    key = synth.make_key(key_bytes, seed=seed)
    data = synth.make_pages(n, pb, seed=seed + 1)
    ivs = synth.make_ivs(n, seed=seed + 2)
    exp = oracle_pages(direction, 0, key, data, n, pb, ivs)
    got = gpu_pages(direction, 0, key, data, n, pb, ivs, where="device")
    assert first_mismatch(got, exp) is None, f"first mismatch at byte {first_mismatch(got, exp)}"


@pytest.mark.parametrize("n,pb", [(1, 4096), (33, 512), (149, 4096), (300, 8192), (1000, 16), (257, 496)])
@pytest.mark.parametrize("direction", [0, 1])
def test_cbc_device_in_place(direction, n, pb):
    key = synth.make_key(16, seed=n + pb)
    data = synth.make_pages(n, pb, seed=n + pb + 1)
    ivs = synth.make_ivs(n, seed=n + pb + 2)
    exp = oracle_pages(direction, 0, key, data, n, pb, ivs)
    got = gpu_pages(direction, 0, key, data, n, pb, ivs, where="device", inplace=True)
    assert first_mismatch(got, exp) is None


@pytest.fixture(params=["staged", "auto"])
def host_path(request):
    from gpu_util import kg_ready
    kg, _ = kg_ready()
    kg.set_host_path(kg.HOST_STAGED if request.param == "staged" else kg.HOST_AUTO, 32 << 20)
    yield request.param
    kg.set_host_path(kg.HOST_AUTO, 32 << 20)


@pytest.mark.parametrize("n,pb", [(1, 16), (16, 4096), (149, 4096), (1000, 512), (3000, 4096)])
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("inplace", [False, True])
def test_cbc_pinned(direction, n, pb, inplace, host_path):
    key = synth.make_key(32, seed=7 * n + pb)
    data = synth.make_pages(n, pb, seed=n)
    ivs = synth.make_ivs(n, seed=n + 9)
    exp = oracle_pages(direction, 0, key, data, n, pb, ivs)
    got = gpu_pages(direction, 0, key, data, n, pb, ivs, where="pinned", inplace=inplace)
    assert first_mismatch(got, exp) is None


@pytest.mark.parametrize("in_where,out_where,iv_where", [("device", "pinned", "device"), ("pinned", "device", "pinned"),
                                                         ("pinned", "pinned", "device"), ("device", "device", "pinned")])
@pytest.mark.parametrize("direction", [0, 1])
def test_cbc_mixed_residency(direction, in_where, out_where, iv_where, host_path):
    n, pb = 700, 4096
    key = synth.make_key(16, seed=77)
    data = synth.make_pages(n, pb, seed=78)
    ivs = synth.make_ivs(n, seed=79)
    exp = oracle_pages(direction, 0, key, data, n, pb, ivs)
    got = gpu_pages(direction, 0, key, data, n, pb, ivs, where=in_where, out_where=out_where, iv_where=iv_where)
    assert first_mismatch(got, exp) is None


@pytest.mark.parametrize("n,pb", [(1, 16), (3, 4096), (149, 4096), (1000, 48)])
@pytest.mark.parametrize("key_bytes", [16, 32])
@pytest.mark.parametrize("direction", [0, 1])
def test_ecb(direction, key_bytes, n, pb):
    key = synth.make_key(key_bytes, seed=n * 3 + pb)
    data = synth.make_pages(n, pb, seed=n * 5 + pb)
    exp = oracle_pages(direction, 1, key, data, n, pb, None)
    got = gpu_pages(direction, 1, key, data, n, pb, None, where="device")
    assert first_mismatch(got, exp) is None
    got = gpu_pages(direction, 1, key, data, n, pb, None, where="pinned", inplace=True)
    assert first_mismatch(got, exp) is None


def test_small_staging_chunks_many_slots():
    """Pinned path with chunks much smaller than the batch: the 3-slot ring
    wraps many times."""
    from gpu_util import kg_ready
    kg, torch = kg_ready()
    n, pb = 1001, 4096
    key = synth.make_key(16, seed=5)
    data = synth.make_pages(n, pb, seed=6)
    ivs = synth.make_ivs(n, seed=7)
    exp = oracle_pages(1, 0, key, data, n, pb, ivs)
    kg.set_host_path(kg.HOST_STAGED)
    for chunk, slots in [(4096, 2), (3 * 4096, 3), (64 * 1024, 8), (10 * 4096 + 16, 3), (0, 4), (0, 2)]:
        kg.set_pipeline(chunk, slots)
        try:
            got = gpu_pages(1, 0, key, data, n, pb, ivs, where="pinned")
        finally:
            kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
            kg.set_host_path(kg.HOST_AUTO, 32 << 20)
        assert first_mismatch(got, exp) is None, (chunk, slots)


@pytest.mark.parametrize("n,pb", [(1, 16), (16, 4096), (149, 4096), (1000, 512), (3000, 4096)])
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("mode", ["zerocopy", "auto"])
def test_cbc_host_zero_copy(direction, n, pb, mode):
    """Row f4: kernels reading/writing pinned host pages directly (no staging)."""
    from gpu_util import kg_ready
    kg, torch = kg_ready()
    key = synth.make_key(16, seed=3 * n + pb)
    data = synth.make_pages(n, pb, seed=n + 1)
    ivs = synth.make_ivs(n, seed=n + 2)
    exp = oracle_pages(direction, 0, key, data, n, pb, ivs)
    kg.set_host_path(kg.HOST_ZEROCOPY if mode == "zerocopy" else kg.HOST_AUTO, 64 << 10)
    try:
        got = gpu_pages(direction, 0, key, data, n, pb, ivs, where="pinned")
        got_ip = gpu_pages(direction, 0, key, data, n, pb, ivs, where="pinned", inplace=True)
        got_mixed = gpu_pages(direction, 0, key, data, n, pb, ivs, where="pinned", out_where="device")
    finally:
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
    assert first_mismatch(got, exp) is None
    assert first_mismatch(got_ip, exp) is None
    assert first_mismatch(got_mixed, exp) is None


def test_alloc_pinned_numa_buffers():
    """Row f4: library-allocated NUMA-local pinned buffers work as batch memory
    on both host paths and round-trip through free."""
    from gpu_util import kg_ready
    kg, torch = kg_ready()
    n, pb = 2048, 4096
    key = synth.make_key(16, seed=91)
    kg.set_key(0, key)
    data = synth.make_pages(n, pb, seed=92)
    ivs = synth.make_ivs(n, seed=93)
    exp = oracle_pages(1, 0, key, data, n, pb, ivs)
    hin = kg.alloc_pinned(n * pb)
    hout = kg.alloc_pinned(n * pb)
    hiv = kg.alloc_pinned(16 * n)
    try:
        hin.copy_(torch.from_numpy(data))
        hiv.copy_(torch.from_numpy(ivs))
        for hp in (kg.HOST_STAGED, kg.HOST_ZEROCOPY):
            kg.set_host_path(hp)
            hout.zero_()
            kg.wait(kg.submit_pages(1, 0, hin, hout, n, pb, hiv, 0))
            assert first_mismatch(hout.numpy(), exp) is None, hp
    finally:
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
        for t in (hin, hout, hiv):
            kg.free_pinned(t)
    assert kg.raw_lib().kg_free_pinned(12345) == kg.EINVAL


def test_staged_batches_back_to_back():
    """Several host batches in flight at once through the staging ring (no wait
    between submits): slots and the double-buffered IV stage must not be
    reused before their previous users are done."""
    from gpu_util import kg_ready
    kg, torch = kg_ready()
    kg.set_host_path(kg.HOST_STAGED)
    kg.set_pipeline(64 * 4096, 3)
    try:
        n, pb = 700, 4096
        key = synth.make_key(16, seed=501)
        kg.set_key(0, key)
        jobs = []
        for b in range(6):
            data = synth.make_pages(n, pb, seed=600 + b)
            ivs = synth.make_ivs(n, seed=700 + b)
            d = b % 2
            hin = torch.from_numpy(data).pin_memory()
            hiv = torch.from_numpy(ivs).pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            t = kg.submit_pages(d, 0, hin, hout, n, pb, hiv, 0)
            jobs.append((t, d, data, ivs, hout, hin, hiv))
        for t, d, data, ivs, hout, *_ in jobs:
            kg.wait(t)
            exp = oracle_pages(d, 0, key, data, n, pb, ivs)
            assert first_mismatch(hout.numpy(), exp) is None
    finally:
        kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)


def test_staged_auto_chunks_warm_and_cold():
    """Auto chunking: a batch submitted while earlier batches' copies are still
    queued runs warm (16 MiB chunks, no ramps), one submitted to idle copy
    engines cold (8 MiB chunks, ramped ends); slots are sized for the warm
    chunk from the start.  Batches of 9,000 x 4 KiB pages (ragged against both
    chunk sizes) on separate streams, both directions, every byte vs the oracle."""
    from gpu_util import kg_ready
    kg, torch = kg_ready()
    kg.set_host_path(kg.HOST_STAGED)
    kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
    try:
        n, pb = 9000, 4096
        key = synth.make_key(32, seed=811)
        kg.set_key(0, key)
        streams = [torch.cuda.Stream() for _ in range(3)]
        jobs = []
        for b in range(5):
            data = synth.make_pages(n, pb, seed=820 + b)
            ivs = synth.make_ivs(n, seed=830 + b)
            d = (b + 1) % 2
            hin = torch.from_numpy(data).pin_memory()
            hiv = torch.from_numpy(ivs).pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            t = kg.submit_pages(d, 0, hin, hout, n, pb, hiv, 0, streams[b % 3])
            jobs.append((t, d, data, ivs, hout, hin, hiv))
            if b == 3:  # let the pipeline go idle: the last batch is cold again
                kg.wait(t)
        for t, d, data, ivs, hout, *_ in jobs:
            if t != jobs[3][0]:
                kg.wait(t)
            exp = oracle_pages(d, 0, key, data, n, pb, ivs)
            assert first_mismatch(hout.numpy(), exp) is None
    finally:
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)


@pytest.mark.parametrize("pb", [1056, 4096, 2080])
@pytest.mark.parametrize("inplace", [False, True])
def test_tail_pool_large_batches(pb, inplace):
    """Batches large enough for the block-pair kernel's tail-balancing pool
    (>= 64 pages per CTA), incl. pair counts per page that are not multiples of
    32 (pool units then straddle page boundaries)."""
    n = 64 * 148 + 37
    key = synth.make_key(16, seed=pb + inplace)
    data = synth.make_pages(n, pb, seed=pb)
    ivs = synth.make_ivs(n, seed=pb + 1)
    exp = oracle_pages(1, 0, key, data, n, pb, ivs)
    got = gpu_pages(1, 0, key, data, n, pb, ivs, where="device", inplace=inplace)
    assert first_mismatch(got, exp) is None
    exp_e = oracle_pages(1, 1, key, data, n, pb, None)
    got_e = gpu_pages(1, 1, key, data, n, pb, None, where="device", inplace=inplace)
    assert first_mismatch(got_e, exp_e) is None


@pytest.mark.parametrize("lag", ["0", "2"])
def test_staged_d2h_lag_modes(lag):
    """The staged pipeline's D2H lag modes other than the default (KG_D2H_LAG,
    read once per process): the staged parity cases in a child process."""
    import os
    import subprocess
    import sys
    from gpu_util import kg_ready
    kg_ready()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KG_D2H_LAG=lag, KG_RAMP_DOWN="0" if lag == "2" else "1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_parity_gpu.py"),
                        "-k", "(staged_batches or small_staging or cbc_pinned or mixed_residency) and not lag_modes"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("env", [{"KG_TEXIN": "0"}, {"KG_TEX_MAX_ELEMS": "4096"}])
def test_texture_path_variants(env):
    """Device-batch parity with plain LDG page loads (KG_TEXIN=0) and with
    64 KiB texture windows (KG_TEX_MAX_ELEMS=4096: every batch above 16 pages
    runs as several windowed launches, in place and out of place, with IV
    offsets), in a child process (both are read once per process)."""
    import os
    import subprocess
    import sys
    from gpu_util import kg_ready
    kg_ready()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_parity_gpu.py"),
                        "-k", "(cbc_device or ecb or tail_pool or mixed_residency or one_batch_texture) and not texture_path"],
                       cwd=root, env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_texture_cache_eviction_many_buffers_and_streams():
    """More distinct input buffers (80) than the texture cache holds (64) and
    more streams (70) than a use set tracks (64): entries are evicted only
    after their launches finish, and every batch still matches the oracle."""
    from gpu_util import kg_ready
    kg, torch = kg_ready()
    n, pb = 3, 4096
    key = synth.make_key(16, seed=808)
    kg.set_key(0, key)
    streams = [torch.cuda.Stream() for _ in range(70)]
    jobs = []
    for b in range(80):
        data = synth.make_pages(n, pb, seed=900 + b)
        ivs = synth.make_ivs(n, seed=1000 + b)
        x = torch.from_numpy(data).cuda()
        iv = torch.from_numpy(ivs).cuda()
        out = torch.empty_like(x)
        torch.cuda.synchronize()
        s = streams[b % len(streams)]
        jobs.append((kg.submit_pages(1, 0, x, out, n, pb, iv, 0, s), data, ivs, x, iv, out))
        if b % 7 == 6:                      # some buffers freed and reallocated while others are in flight
            t, d, v, *_ = jobs.pop(0)
            kg.wait(t)
    for t, data, ivs, x, iv, out in jobs:
        kg.wait(t)
        torch.cuda.synchronize()
        exp = oracle_pages(1, 0, key, data, n, pb, ivs)
        assert first_mismatch(out.cpu().numpy(), exp) is None


@pytest.mark.parametrize("direction,mode", [(1, 0), (0, 0), (1, 1), (0, 1)])
def test_staged_device_input_one_batch_texture(direction, mode):
    """Device input, pinned output, staged in many small chunks: every chunk's
    launch reads its slice of ONE texture over the whole batch input
    (a texture per chunk missed the cache every chunk); in
    KG_TEX_MAX_ELEMS runs (test_texture_path_variants) the batch exceeds one
    texture and the chunks fall back to their own textures."""
    from gpu_util import kg_ready, put
    kg, torch = kg_ready()
    n, pb = 300, 4096
    key = synth.make_key(16, seed=515)
    kg.set_key(0, key)
    data = synth.make_pages(n, pb, seed=516)
    ivs = synth.make_ivs(n, seed=517) if mode == 0 else None
    exp = oracle_pages(direction, mode, key, data, n, pb, ivs)
    x = put(torch, data, "device")
    iv = None if ivs is None else put(torch, ivs, "device")
    out = torch.empty(n * pb, dtype=torch.uint8).pin_memory()
    kg.set_host_path(kg.HOST_STAGED, 0)
    kg.set_pipeline(16 * pb, 3)          # 19 chunks
    try:
        kg.wait(kg.submit_pages(direction, mode, x, out, n, pb, iv, 0))
    finally:
        kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
    torch.cuda.synchronize()
    assert first_mismatch(out.numpy(), exp) is None


@pytest.mark.parametrize("n", [4, 7, 591, 592, 593, 595, 599, 1183, 4733])
@pytest.mark.parametrize("inplace", [False, True])
def test_cbc_encrypt_chain_units(n, inplace):
    """CBC-encrypt chain kernels deal pages to CTAs in 4-page units (kChainAlign):
    batch sizes around 148 x 4 pages and odd remainders, every byte vs the oracle."""
    key = synth.make_key(32, seed=900 + n)
    data = synth.make_pages(n, 4096, seed=901 + n)
    ivs = synth.make_ivs(n, seed=902 + n)
    exp = oracle_pages(0, 0, key, data, n, 4096, ivs)
    got = gpu_pages(0, 0, key, data, n, 4096, ivs, where="device", inplace=inplace)
    assert first_mismatch(got, exp) is None
