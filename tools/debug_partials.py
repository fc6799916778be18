"""Debug helper: run dsde_verify on a tiny batch and print the chunk partials."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_01083_b200 as m
import synth
from tests.gpu_util import gpu_verify, to_device_inputs, make_host_batch

for dtype in (torch.float32, torch.bfloat16):
    V = 32000
    host = make_host_batch(V, [1], seed=3, dtype=dtype)
    st = m.State(m.Config.default(), 4)
    dev = to_device_inputs(host, dtype)
    n = 1; B = 1
    ws = torch.zeros(m.workspace_size(B, n, V, dtype) + 256, dtype=torch.uint8, device="cuda")
    ws = ws[(-ws.data_ptr()) % 256:]
    acc = torch.zeros(B, dtype=torch.int32, device="cuda"); em = torch.zeros(n + B, dtype=torch.int32, device="cuda")
    kl = torch.zeros(n, dtype=torch.float32, device="cuda")
    m.dsde_verify(st, V, n, dev["cu_sl"], dev["draft_tokens"], dev["target"], dev["draft"], dev["seeds"], acc, em, kl, None, ws)
    torch.cuda.synchronize()
    nc = (V + (8192 if dtype == torch.bfloat16 else 4096) - 1) // (8192 if dtype == torch.bfloat16 else 4096)
    raw = ws[: 48 * nc].cpu().numpy()
    for c in range(nc):
        rec = raw[48 * c: 48 * (c + 1)]
        S, A, D = np.frombuffer(rec[:24].tobytes(), np.float64)
        M, C = np.frombuffer(rec[24:32].tobytes(), np.float32)
        idx, flags = np.frombuffer(rec[32:40].tobytes(), np.int32)
        maxd = np.frombuffer(rec[40:44].tobytes(), np.float32)[0]
        print(dtype, c, S, A, D, M, C, idx, flags, maxd)
    print("acc", acc.cpu().numpy(), "kl", kl.cpu().numpy(), "err", st.device_error())
