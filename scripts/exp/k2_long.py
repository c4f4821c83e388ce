"""One long K2 (B=1, T=4000, U=50 -> kC=2 single-warp instance; U=100 -> multi-warp) for ncu source sampling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import workloads
import paper_2303_10384_b200 as rb
U = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cfg = workloads.Config("k2long", B=1, Tmax=4000, Umax=U, V=16, logit_seed=3)
pb = workloads.problem(cfg, device="cuda")
for _ in range(3):
    rb.rnnt_loss(pb["logits"], pb["targets"], pb["logit_lens"], pb["target_lens"], 0, grads=False)
torch.cuda.synchronize()
print("ok")
