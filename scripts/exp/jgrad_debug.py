"""Debug: the fused joint training step's gradients, tensor by tensor, vs the oracle (rounding="forward") and
vs a torch fp32 chain rule on the GPU (from the oracle-free inputs), printing max |err| / max |ref|."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_2303_10384_b200 as rb
import workloads
from oracle import joint as oj

for (B, T, U, H, V) in [(2, 9, 4, 128, 128), (2, 40, 16, 512, 1024), (3, 30, 10, 256, 500), (2, 11, 5, 384, 200)]:
    cfg = workloads.random_config(B, T, U, V, seed=5, variant="rnnt")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=5)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt")
    torch.cuda.synchronize()
    args = [x.double().numpy() for x in (enc, pred, W, b)]
    ref = oj.joint_loss_and_grads(*args, y, T_b, U_b, 0, "rnnt")
    bnd = oj.r23_bounds(*args, y, T_b, U_b, 0, "rnnt")
    print(f"B{B} T{T} U{U} H{H} V{V}: loss rel {np.abs(out[0].cpu().numpy() - ref[0]).max() / np.abs(ref[0]).max():.2e}")
    for name, k, mine, r in zip(("d_enc", "d_pred", "d_W", "d_bias"), ("d_f", "d_g", "d_W", "d_bias"), out[1:], ref[1:]):
        m = mine.cpu().numpy().astype(np.float64)
        err = np.abs(m - r)
        print(f"   {name:7s} max|err|/max|ref| {err.max() / max(np.abs(r).max(), 1e-30):.3e}  "
              f"err/bound {np.max(err / np.maximum(bnd[k], 1e-300)):.3f}  nan {np.isnan(m).sum()}")
