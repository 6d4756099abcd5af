"""Helpers for the -m gpu tests: run the CUDA path through the C ABI on
seeded inputs and compare with the oracle.  Imported only by gpu tests."""
import os

import numpy as np

CORES = len(os.sched_getaffinity(0))


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        import pytest
        pytest.skip("no CUDA device")
    return torch


def kg_ready(device=0):
    torch = torch_cuda()
    import paper_1305_3345_b200 as kg
    torch.cuda.set_device(device)
    torch.cuda.init()
    kg.init(device)
    return kg, torch


def put(torch, arr: np.ndarray, where: str):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if where == "device":
        return t.cuda()
    if where == "pinned":
        return t.pin_memory()
    raise ValueError(where)


def gpu_pages(direction, mode, key, data, n, pb, ivs, where="device", inplace=False, key_id=0,
              out_where=None, iv_where=None, stream=None):
    """Run one batch through kg_submit_pages/kg_wait; return the output as numpy."""
    kg, torch = kg_ready()
    kg.set_key(key_id, key)
    out_where = out_where or where
    iv_where = iv_where or where
    tin = put(torch, data, where)
    tout = tin if inplace else (torch.empty(n * pb, dtype=torch.uint8, device="cuda") if out_where == "device"
                                else torch.empty(n * pb, dtype=torch.uint8).pin_memory())
    tiv = None if ivs is None else put(torch, ivs, iv_where)
    t = kg.submit_pages(direction, mode, tin, tout, n, pb, tiv, key_id, stream)
    kg.wait(t)
    torch.cuda.synchronize()
    return tout.cpu().numpy()


def oracle_pages(direction, mode, key, data, n, pb, ivs):
    import oracle
    return oracle.pages(direction, mode, key, data, n, pb, ivs, threads=CORES)


def first_mismatch(a: np.ndarray, b: np.ndarray):
    d = np.nonzero(a != b)[0]
    return None if d.size == 0 else int(d[0])
