"""Small driver for profiling K2 alone: c3 shapes, a few utterances, loss only."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2303_10384_b200 as rb
cfg = dataclasses.replace(workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"], B=int(os.environ.get("PROF_B", "2")))
variant = sys.argv[2] if len(sys.argv) > 2 else "rnnt"
pb = workloads.problem(cfg, device="cuda")
for _ in range(3):
    l, _ = rb.loss(pb["logits"], pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank, variant, grads=False)
torch.cuda.synchronize()
print(l.tolist())
