"""Per-slice cost profile of one walk launch (diagnostic build with -DFZ_SLICE_TRACE=1, selected by FZ_LIB_PATH):
unrank vs walk cycles, the walk cost along the slice order (deciles), and how the slices' end times spread.
Usage: FZ_LIB_PATH=ab/libfz_trace.so python tools/slice_trace.py T1 T95 ..."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_20474_b200 import fz  # noqa: E402
from tools.quick_time import CFG  # noqa: E402


def main():
    lib = ctypes.CDLL(fz.LIB_PATH)
    lib.fz_debug_slice_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    for name in sys.argv[1:]:
        g, n, t, mode, *pct = CFG[name]
        lay = fz.Layout(g, t, n + 1, entries=(mode != "count"))
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
        memo = fz.Memo(layout=lay, workspace=ws)
        pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
        out = None
        for _ in range(3):
            plan = fz.Plan(memo, n, mode, workspace=pws)
            if out is None and mode == "materialize":
                out = torch.empty((plan.rows, len(g)), dtype=torch.int32, device="cuda")
            plan.launch(out)
            torch.cuda.synchronize()
        ns = plan.nslices
        buf = np.zeros((min(ns, 1 << 20), 4), dtype=np.uint32)
        assert lib.fz_debug_slice_trace(buf.ctypes.data, buf.shape[0]) == 0
        un, wk, te = buf[:, 0].astype(np.float64), buf[:, 1].astype(np.float64), buf[:, 2].astype(np.float64) * 64
        te -= te.min()
        print(f"{name}: {ns} slices; unrank cycles sum {un.sum():.3e} (mean {un.mean():.0f}), walk cycles sum "
              f"{wk.sum():.3e} (mean {wk.mean():.0f}); unrank share {un.sum() / (un.sum() + wk.sum()):.3f}")
        dec = np.array_split(np.arange(len(wk)), 10)
        print("  walk cycles per slice by decile of the slice order: " +
              " ".join(f"{wk[d].mean():.0f}" for d in dec))
        print("  max slice (unrank + walk) cycles %.0f, p99 %.0f, p50 %.0f" %
              ((un + wk).max(), np.percentile(un + wk, 99), np.percentile(un + wk, 50)))
        q = np.percentile(te, [50, 90, 99, 100])
        print("  slice end times (us after the first end): p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(q / 1e3))
        del out


if __name__ == "__main__":
    main()
