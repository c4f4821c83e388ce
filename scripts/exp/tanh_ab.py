"""K6 forward at p124 / c3: tanh.approx (RNNT_K6_DEBUG=8) vs the 2-MUFU tanh: time and loss deviation vs the
oracle-exact losses (run twice with the env var set or not)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import workloads
import paper_2303_10384_b200 as rb
from oracle import joint as oj
out = {}
for cfg_name in ("p124", "c3"):
    base = {**workloads.CONFIGS, **workloads.EXTRA_CONFIGS}[cfg_name]
    T_np, U_np = workloads.lengths(base)
    y = workloads.targets(base, U_np)
    enc, pred, W, b = workloads.joint_inputs(base.B, base.Tmax, base.Umax, 512, base.V, seed=base.logit_seed % 1000 + 1)
    e, p_, w_, b_ = enc.cuda(), pred.cuda(), W.cuda(), b.cuda()
    yt, Tt, Ut = (torch.from_numpy(x).cuda() for x in (y, T_np, U_np))
    ws = torch.empty(rb.rnnt_workspace_bytes(base.B, base.Tmax, base.Umax), dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for x in ev: x.record()
    times = []
    for i in range(12):
        l = rb.rnnt_joint_loss(e, p_, w_, b_, yt, Tt, Ut, 0, "rnnt", workspace=ws, events=ev)
        torch.cuda.synchronize()
        if i >= 2: times.append(ev[0].elapsed_time(ev[1]))
    ref = oj.joint_loss(enc[:2].double().numpy(), pred[:2].double().numpy(), W.double().numpy(), b.double().numpy(),
                        y[:2], T_np[:2], U_np[:2], 0, "rnnt")
    rel = np.abs(l[:2].cpu().numpy() - ref) / np.abs(ref)
    out[cfg_name] = {"k6_ms": float(np.median(times)), "loss_rel_err_utt01": rel.tolist()}
print(json.dumps({"dbg": os.environ.get("RNNT_K6_DEBUG", "0"), **out}))
