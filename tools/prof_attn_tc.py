"""One ReuseViT embed (tcgen05 attention, the default) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2506_14107_b200 import ReuseViT
cfg = synth.CONFIGS["l14"]
x, c = synth.make_video(cfg, 1440, 0.2, seed=2000)
m = ReuseViT(cfg, 0)
m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg)))
m.load_gates(synth.pack_gates(cfg, synth.make_gates(cfg)))
Z, M, _, st = m.embed(torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda(), graph=False, attn_tc=True)
torch.cuda.synchronize()
print(st["reuse_all"])
