"""Debug helper: one dsde_verify call on a cfg3-sized batch (prints kernel output)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_01083_b200 as m
import synth

B, V = int(os.environ.get("B", 256)), 128256
w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=("code",), seed=3)
k = synth.random_k(B, 8, 3)
s = synth.generate_step(w, 0, k, device="cuda")
st = m.State(m.Config.default(), B)
step = m.Step(st, B, V, torch.bfloat16)
for it in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step.verify(s.cu_sl, s.draft_tokens, s.target, s.draft, s.seeds, int(k.sum()))
    e1.record()
    torch.cuda.synchronize()
    print("verify ms", e0.elapsed_time(e1), flush=True)
print("err", st.device_error())
