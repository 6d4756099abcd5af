import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1305_3345_b200 as kg
import synth
kg.init(0)
kg.set_key(0, synth.make_key(16))
x = torch.from_numpy(synth.make_pages(4, 4096)).cuda()
iv = torch.from_numpy(synth.make_ivs(4)).cuda()
y = torch.empty_like(x)
kg.nsk_start(2, kg.NSK_DIRECT | kg.NSK_NOCAL, 3000)
print("started", flush=True)
t = kg.submit_pages(1, 0, x, y, 4, 4096, iv, 0)
print("submitted", t, flush=True)
print("wait rc", kg.wait_raw(t), flush=True)
print("stop rc", kg.raw_lib().kg_nsk_stop(), flush=True)
