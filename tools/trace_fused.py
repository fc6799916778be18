"""One fused dsde_step on cfg3-like inputs (debug: build with -DDSDE_FUSED_TRACE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_01083_b200 as m, synth
B, V = 256, 128256
w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=("code",), seed=3)
k = synth.random_k(B, 8, 5)
inp = synth.generate_step(w, 0, k, device="cuda")
st = m.State(m.Config.default(), B)
step = m.Step(st, B, V, torch.bfloat16)
for it in range(2):
    out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, int(k.sum()))
    torch.cuda.synchronize()
    print("---- iteration", it, "err", st.device_error(), flush=True)
