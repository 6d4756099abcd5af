"""Concurrency soak (SPEC.md:64, 489 idea): several host threads submit and
wait concurrently; every ticket completes exactly once and every output is
correct (compared against a GPU-computed reference of the same batch)."""
import threading

import numpy as np
import pytest

import synth
from gpu_util import gpu_pages, kg_ready

pytestmark = pytest.mark.gpu


def test_threads_submit_wait():
    kg, torch = kg_ready()
    n, pb = 64, 4096
    key = synth.make_key(16, seed=99)
    kg.set_key(9, key)
    p = synth.make_pages(n, pb, seed=100)
    iv = synth.make_ivs(n, seed=101)
    expect = gpu_pages(0, 0, key, p, n, pb, iv, key_id=8)
    src = torch.from_numpy(p).cuda()
    tiv = torch.from_numpy(iv).cuda()
    errors, seen = [], []
    lock = threading.Lock()

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            outs = [torch.empty_like(src) for _ in range(4)]
            for i in range(600):
                o = outs[i % 4]
                t = kg.submit_pages(0, 0, src, o, n, pb, tiv, 9, stream=s)
                with lock:
                    seen.append(t)
                kg.wait(t)
                if i % 97 == 0:
                    s.synchronize()
                    if not np.array_equal(o.cpu().numpy(), expect):
                        errors.append((tid, i))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors[:5]
    assert len(seen) == len(set(seen)) == 2400
