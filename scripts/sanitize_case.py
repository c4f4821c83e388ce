"""Small cases for compute-sanitizer: every entry point, all variants, fp32/bf16, scalar + vector paths."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2303_10384_b200 as rb
from paper_2303_10384_b200 import lattice as rlat
import workloads

for shape in [(3, 9, 4, 8, 0), (2, 33, 40, 130, 129), (2, 20, 70, 256, 3), (2, 12, 5, 1024, 7)]:
    B, T, U, V, blank = shape
    for variant in ("rnnt", "force_final", "allow_ignore"):
        cfg = workloads.random_config(B, T, U, V, seed=sum(shape), blank=blank, variant=variant)
        pb = workloads.problem(cfg)
        z = pb["logits"].cuda()
        rb.loss(z, pb["targets"], pb["logit_lens"], pb["target_lens"], blank, variant)
        rb.loss(z.to(torch.bfloat16), pb["targets"], pb["logit_lens"], pb["target_lens"], blank, variant,
                grads="inplace")
        rb.rnnt_viterbi(z, pb["targets"], pb["logit_lens"], pb["target_lens"], blank, variant)
        L = rlat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], blank, variant)
        rb.rnnt_lattice_loss(z, L, pb["logit_lens"], pb["target_lens"])
# the fused joint: forward, alignment, training step (K6, K6<grad>, K7); V % 128 != 0 tail; compose lattices
from paper_2303_10384_b200 import compose as rcmp
for (B, T, U, H, V) in [(2, 9, 4, 128, 128), (2, 21, 7, 256, 500), (2, 11, 5, 384, 200), (3, 7, 3, 512, 130)]:
    cfg = workloads.random_config(B, T, U, V, seed=T + U)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, bias = (x.cuda() for x in workloads.joint_inputs(B, T, U, H, V, seed=T + U))
    rb.rnnt_joint_loss(enc, pred, W, bias, y, T_b, U_b, 0, "allow_ignore")
    rb.rnnt_joint_viterbi(enc, pred, W, bias, y, T_b, U_b, 0, "force_final")
    rb.rnnt_joint_loss_grad(enc, pred, W, bias, y, T_b, U_b, 0, "rnnt")          # K6<grad>, K8, K9, K7
    rb.rnnt_joint_loss_grad(enc, pred, W, bias, y, torch.from_numpy(T_b).cuda(), torch.from_numpy(U_b).cuda(), 0,
                            "rnnt")                                                  # padded rows, zeroed tail
    pb = workloads.problem(cfg)
    Lc = rcmp.compose_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], V, 0, "force_final")
    rb.rnnt_lattice_loss(pb["logits"].cuda(), Lc, pb["logit_lens"], pb["target_lens"])
# the chunked / overlapped path (>= 2^24 elements)
cfg = workloads.random_config(4, 120, 40, 1024, seed=15, variable=True)
pb = workloads.problem(cfg)
rb.rnnt_loss(pb["logits"].cuda(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0)
# the host-buffer ring path (fp32 and bf16)
cfg = workloads.random_config(5, 17, 6, 64, seed=21)
pb = workloads.problem(cfg)
for dt in (torch.float32, torch.bfloat16):
    zh = pb["logits"].to(dt).pin_memory()
    rb.rnnt_loss_host(zh, torch.from_numpy(pb["targets"]), torch.from_numpy(pb["logit_lens"]),
                      torch.from_numpy(pb["target_lens"]), 0, "rnnt", grads_host=torch.empty_like(zh))
torch.cuda.synchronize()
print("sanitize cases done")
