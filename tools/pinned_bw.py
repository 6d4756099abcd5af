"""Duplex host-link bandwidth on different pinned allocations (1 GiB)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1305_3345_b200 as kg  # noqa: E402

kg.init(0)
n = 1 << 30
a = torch.empty(n, dtype=torch.uint8).pin_memory()
b = torch.empty(n, dtype=torch.uint8).pin_memory()
print(json.dumps({"alloc": "torch pin_memory", "duplex_gbs": bench.duplex_link_gbs(torch, a, b, 256 << 20)}))
a2, b2 = kg.alloc_pinned(n), kg.alloc_pinned(n)
print(json.dumps({"alloc": "kg_alloc_pinned " + os.environ.get("KG_PINNED_MODE", "hostalloc"),
                  "duplex_gbs": bench.duplex_link_gbs(torch, a2, b2, 256 << 20)}))
kg.free_pinned(a2)
kg.free_pinned(b2)
