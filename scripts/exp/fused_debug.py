"""Debug the fused small-call schedule at c2: time to failure and which phase."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, workloads
import paper_2303_10384_b200 as rb
cfg = workloads.CONFIGS["c2"]
pb = workloads.problem(cfg, device="cuda")
z = pb["logits"]
y = torch.as_tensor(pb["targets"]).cuda(); T = torch.as_tensor(pb["logit_lens"]).cuda(); U = torch.as_tensor(pb["target_lens"]).cuda()
for grads in (False, True):
    t0 = time.time()
    try:
        l, g = rb.loss(z, y, T, U, cfg.blank, "rnnt", grads=grads)
        torch.cuda.synchronize()
        print("grads", grads, "ok", time.time() - t0, float(l.sum()), flush=True)
    except Exception as e:
        print("grads", grads, "FAIL after", time.time() - t0, repr(e)[:200], flush=True)
        break
