import os, sys, json
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
import torch, paper_1305_3345_b200 as kg, synth
PB=4096; n=int(sys.argv[1]); chunk=int(sys.argv[2])
kg.init(0); kg.set_key(0, synth.make_key(16)); kg.set_pipeline(chunk<<20, 3)
hx=torch.from_numpy(synth.make_pages(n,PB)).pin_memory(); hiv=torch.from_numpy(synth.make_ivs(n)).pin_memory(); ho=torch.empty_like(hx).pin_memory()
for i in range(3): kg.wait(kg.submit_pages(1,0,hx,ho,n,PB,hiv,0))
