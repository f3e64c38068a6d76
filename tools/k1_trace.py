"""Phase timeline of the fused memo build (k1_memo): per-CTA globaltimer stamps via FZ_K1_TRACE.

    python tools/k1_trace.py C2 [C3t3 ...]        (FZ_SCAN_LG=k in the environment forces the lanes per x)

Prints, per phase, the latest start (barrier release) and the earliest / median / latest end of the
phase's work over the CTAs, relative to the earliest phase-0 start (microseconds)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_20474_b200 import fz  # noqa: E402
from tools.quick_time import CFG  # noqa: E402

fz.set_memo_cap(64 << 30)
buf = torch.zeros(1024 * 32, dtype=torch.int64, device="cuda")
for name in sys.argv[1:] or ["C2"]:
    g, n, t, mode, *pct = CFG[name]
    lay = fz.Layout(g, t, n + 1, entries=(mode != "count"))
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
    for rep in range(4):
        buf.zero_()
        os.environ["FZ_K1_TRACE"] = str(buf.data_ptr())
        fz.Memo(layout=lay, workspace=ws)
        torch.cuda.synchronize()
        os.environ["FZ_K1_TRACE"] = ""
    tr = buf.view(1024, 16, 2).cpu()
    used = (tr[:, 0, 0] != 0)
    tr = tr[used]
    t0 = int(tr[:, 0, 0].min())
    print(f"{name}: {tr.shape[0]} CTAs, fill mode {lay.info['fill_mode']}, lg env {os.environ.get('FZ_SCAN_LG', '-')}")
    for p in range(16):
        st, en = tr[:, p, 0], tr[:, p, 1]
        if int(st.max()) == 0:
            break
        s = (st - t0).double() / 1e3
        e = (en - t0).double() / 1e3
        print(f"  phase {p}: start max {float(s.max()):7.2f}  end min {float(e.min()):7.2f} "
              f"med {float(e.median()):7.2f} max {float(e.max()):7.2f}  (work max {float((e - s).max()):6.2f})")
        if os.environ.get("FZ_TRACE_CTAS"):
            w = (e - s)
            print("     work by CTA:", " ".join(f"{i}:{float(w[i]):.1f}" for i in range(min(32, w.numel()))),
                  "...", f"{w.numel() - 1}:{float(w[-1]):.1f}")
