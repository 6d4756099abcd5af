"""Small-config workload for compute-sanitizer (memcheck/racecheck/synccheck/
initcheck): every kernel variant once, device + pinned + in-place + NSK."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402

kg.init(0)
for kb in (16, 24, 32):
    kg.set_key(kb, synth.make_key(kb))
for n, pb in [(3, 4096), (5, 48), (40, 512)]:
    data = torch.from_numpy(synth.make_pages(n, pb)).cuda()
    ivs = torch.from_numpy(synth.make_ivs(n)).cuda()
    hdata = data.cpu().pin_memory()
    hivs = ivs.cpu().pin_memory()
    for kb in (16, 24, 32):
        for d in (0, 1):
            for mode in (0, 1):
                out = torch.empty_like(data)
                kg.wait(kg.submit_pages(d, mode, data, out, n, pb, ivs if mode == 0 else None, kb))
                x = data.clone()
                kg.wait(kg.submit_pages(d, mode, x, x, n, pb, ivs if mode == 0 else None, kb))
                assert torch.equal(x, out)
                for hp in (kg.HOST_STAGED, kg.HOST_ZEROCOPY):
                    kg.set_host_path(hp)
                    hout = torch.empty_like(hdata).pin_memory()
                    kg.wait(kg.submit_pages(d, mode, hdata, hout, n, pb, hivs if mode == 0 else None, kb))
                    assert torch.equal(hout.cuda(), out)
                kg.set_host_path(kg.HOST_AUTO)
# mixed-key batches: block pairs with constant-bank keys, register-key chains, odd-m kernel
for i, kid in enumerate((3, 7, 9)):
    kg.set_key(kid, synth.make_key(16, seed=50 + i))
for n, pb in [(3, 4096), (5, 48), (40, 512)]:
    data = torch.from_numpy(synth.make_pages(n, pb)).cuda()
    ivs = torch.from_numpy(synth.make_ivs(n)).cuda()
    ids = torch.tensor([(3, 7, 9)[p % 3] for p in range(n)], dtype=torch.int16, device="cuda")
    for d in (0, 1):
        for mode in (0, 1):
            out = torch.empty_like(data)
            kg.wait(kg.submit_pages_keyed(d, mode, data, out, n, pb, ivs if mode == 0 else None, ids, 16))
            x = data.clone()
            kg.wait(kg.submit_pages_keyed(d, mode, x, x, n, pb, ivs if mode == 0 else None, ids, 16))
            assert torch.equal(x, out)
# staged batches back to back (warm schedule: no ramps, the slot rotation
# continuing across batches), small chunks so every batch spans several slots
kg.set_host_path(kg.HOST_STAGED)
kg.set_pipeline(4 * 4096, 3)
n, pb = 37, 4096
hdata = torch.from_numpy(synth.make_pages(n, pb)).pin_memory()
hivs = torch.from_numpy(synth.make_ivs(n)).pin_memory()
streams = [torch.cuda.Stream() for _ in range(3)]
outs = [torch.empty_like(hdata).pin_memory() for _ in range(4)]
ts = [kg.submit_pages(b % 2, 0, hdata, outs[b], n, pb, hivs, 16, streams[b % 3]) for b in range(4)]
for t in ts:
    kg.wait(t)
ref = torch.empty_like(hdata).pin_memory()
kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
kg.set_host_path(kg.HOST_AUTO)
kg.wait(kg.submit_pages(0, 0, hdata, ref, n, pb, hivs, 16))
assert torch.equal(outs[0], ref) and torch.equal(outs[2], ref)
kg.nsk_start(2, kg.NSK_DIRECT | kg.NSK_NOCAL, 2000)
n, pb = 4, 4096
data = torch.from_numpy(synth.make_pages(n, pb)).cuda()
ivs = torch.from_numpy(synth.make_ivs(n)).cuda()
out = torch.empty_like(data)
for d in (0, 1):
    kg.wait(kg.submit_pages(d, 0, data, out, n, pb, ivs, 16))
kg.nsk_stop()
print("sanitize workload ok")
