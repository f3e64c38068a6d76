"""Thin ctypes binding of libfz.so (include/fz.h).  Argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C ABI; PyTorch is
used here only to own device memory (workspaces, output buffers) and to hand
over the current CUDA stream.  There is no CPU fallback: importing this module
fails loudly when the extension is missing.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FZ_LIB_PATH") or os.path.join(_HERE, "libfz.so")   # override: A/B builds (tools)

MATERIALIZE, COUNT, HASH = 0, 1, 2
_MODES = {"materialize": MATERIALIZE, "count": COUNT, "hash": HASH}

FZ_MAX_D = 10


class FzError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"fz status {status}: {message}")
        self.status = status


class _MemoInfo(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("t", ctypes.c_int), ("top", ctypes.c_uint64), ("entries", ctypes.c_uint64),
                ("max_card", ctypes.c_uint64), ("batches", ctypes.c_uint64), ("batch", ctypes.c_uint32),
                ("fill_mode", ctypes.c_int), ("window_rows", ctypes.c_uint64), ("memo_top", ctypes.c_uint64)]

MEMO_TOP_AUTO = 0                 # fz_layout_create_partial: largest memo_top whose rows fit the cap
MEMO_TOP_FULL = (1 << 64) - 1     # memo_top = top


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    u32p, u64p, vp = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p
    c_int, u64 = ctypes.c_int, ctypes.c_uint64
    sig = {
        "fz_memo_workspace_bytes": [u32p, c_int, c_int, u64, c_int, u64p],
        "fz_memo_build": [u32p, c_int, c_int, u64, c_int, vp, u64, vp, ctypes.POINTER(vp)],
        "fz_memo_get_info": [vp, ctypes.POINTER(_MemoInfo)],
        "fz_memo_device_views": [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)],
        "fz_count": [vp, u64, vp, u64p],
        "fz_shard_rows": [vp, u64, c_int, c_int, u64p, u64p],
        "fz_plan_workspace_bytes": [vp, u64p],
        "fz_plan_create": [vp, u64, c_int, c_int, c_int, vp, u64, vp, ctypes.POINTER(vp)],
        "fz_plan_shard": [vp, vp, u64p, u64p, u64p],
        "fz_plan_walk": [vp, ctypes.POINTER(c_int), ctypes.POINTER(c_int)],
        "fz_layout_create": [u32p, c_int, c_int, u64, c_int, ctypes.POINTER(vp)],
        "fz_layout_create_partial": [u32p, c_int, c_int, u64, u64, c_int, ctypes.POINTER(vp)],
        "fz_layout_workspace_bytes": [vp, u64p],
        "fz_layout_get_info": [vp, ctypes.POINTER(_MemoInfo)],
        "fz_memo_build_layout": [vp, vp, u64, vp, ctypes.POINTER(vp)],
        "fz_layout_shard_rows": [vp, u64, c_int, c_int, u64p, u64p],
        "fz_recommend_t": [u32p, c_int, u64, c_int, ctypes.POINTER(c_int), ctypes.POINTER(ctypes.c_double)],
        "fz_enumerate_launch": [vp, vp, u64, u64, vp],
        "fz_plan_result": [vp, vp, u64p, u64p],
        "fz_plan_result_ptr": [vp, ctypes.POINTER(vp)],
        "fz_enumerate": [vp, u64, c_int, c_int, c_int, u64, vp, u64, vp, u64, vp, u64p, u64p],
        "fz_run_workspace_bytes": [u32p, c_int, c_int, u64, c_int, u64, u64p],
        "fz_run_host": [u32p, c_int, c_int, u64, c_int, vp, u64, vp, u64, vp, u64p, u64p],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.fz_free.argtypes = [vp]
    L.fz_free.restype = None
    L.fz_plan_free.argtypes = [vp]
    L.fz_plan_free.restype = None
    L.fz_layout_free.argtypes = [vp]
    L.fz_layout_free.restype = None
    L.fz_last_error.restype = ctypes.c_char_p
    L.fz_launch_count.restype = ctypes.c_uint64
    L.fz_set_memo_cap.argtypes = [u64]
    L.fz_set_memo_cap.restype = None
    L.fz_set_fill_mode.argtypes = [c_int]
    L.fz_set_fill_mode.restype = None
    return L


_L = _load()


def _check(st: int) -> None:
    if st != 0:
        raise FzError(st, _L.fz_last_error().decode())


def _gens(gens):
    arr = (ctypes.c_uint32 * len(gens))(*[int(g) for g in gens])
    return arr


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _mode(mode) -> int:
    return _MODES[mode] if isinstance(mode, str) else int(mode)


def launch_count() -> int:
    """Kernel launches issued by this thread through libfz so far."""
    return int(_L.fz_launch_count())


def set_memo_cap(nbytes: int) -> None:
    _L.fz_set_memo_cap(nbytes)


def recommend_t(gens, n: int, mode="materialize"):
    """Memo dimension with the lowest predicted time (host cost model, fz_recommend_t).
    Returns (t, {t: predicted seconds})."""
    d = len(gens)
    tb = ctypes.c_int()
    cost = (ctypes.c_double * (d + 1))()
    _check(_L.fz_recommend_t(_gens(gens), d, int(n), _mode(mode), ctypes.byref(tb), cost))
    return tb.value, {t: cost[t] for t in range(d + 1) if cost[t] < 1e299}


def set_fill_mode(mode: int) -> None:
    """Force the memo copy-increment schedule (1 ring, 2 L2, 3 grid, 4 chains, 5 chain scan; 0 = automatic)."""
    _L.fz_set_fill_mode(int(mode))


class Layout:
    """A1 host object (fz_layout): validation, sizing and host tables for (gens, t, top).
    memo_top (partial memo, fz_layout_create_partial): memo rows only for x < memo_top; None = full,
    MEMO_TOP_AUTO = the largest that fits the memo cap."""

    def __init__(self, gens, t: int, top: int, entries: bool = True, memo_top: int | None = None):
        self.gens = tuple(int(g) for g in gens)
        self.d, self.t, self.top, self.entries = len(self.gens), int(t), int(top), bool(entries)
        h = ctypes.c_void_p()
        if memo_top is None:
            _check(_L.fz_layout_create(_gens(self.gens), self.d, self.t, self.top, int(entries), ctypes.byref(h)))
        else:
            _check(_L.fz_layout_create_partial(_gens(self.gens), self.d, self.t, self.top, int(memo_top),
                                               int(entries), ctypes.byref(h)))
        self.h = h
        nbytes = ctypes.c_uint64()
        _check(_L.fz_layout_workspace_bytes(self.h, ctypes.byref(nbytes)))
        self.workspace_bytes = nbytes.value
        info = _MemoInfo()
        _check(_L.fz_layout_get_info(self.h, ctypes.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in _MemoInfo._fields_}

    def shard_rows(self, n: int, mode, nshards: int):
        """Host-side shard cut (same as the device planner K4): (row_begin list, rows list)."""
        rb = (ctypes.c_uint64 * nshards)()
        rl = (ctypes.c_uint64 * nshards)()
        _check(_L.fz_layout_shard_rows(self.h, int(n), _mode(mode), nshards, rb, rl))
        return list(rb), list(rl)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _L is not None:
            _L.fz_layout_free(h)
            self.h = None


class Memo:
    """A memo built on the GPU (fz_memo_build_layout); owns (or borrows) its device workspace."""

    def __init__(self, gens=None, t: int = 0, top: int = 0, entries: bool = True, device=None, stream=None,
                 layout: Layout | None = None, workspace: torch.Tensor | None = None):
        self.layout = layout if layout is not None else Layout(gens, t, top, entries)
        lay = self.layout
        self.gens, self.d, self.t, self.top = lay.gens, lay.d, lay.t, lay.top
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        need = max(lay.workspace_bytes, 256)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=device)
        self.ws = workspace
        h = ctypes.c_void_p()
        with torch.cuda.device(self.ws.device):
            _check(_L.fz_memo_build_layout(lay.h, ctypes.c_void_p(self.ws.data_ptr()), need, _stream(stream),
                                           ctypes.byref(h)))
        self.h = h
        self.info = lay.info

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _L is not None:
            _L.fz_free(h)
            self.h = None

    def views(self):
        """(rows u32 [entries, t], off u64 [top+1], S u64 [d+1, top]) as tensors aliasing the workspace."""
        r, o, s = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(_L.fz_memo_device_views(self.h, ctypes.byref(r), ctypes.byref(o), ctypes.byref(s)))
        base = self.ws.data_ptr()

        def sl(ptr, nbytes):
            off = ptr - base
            return self.ws[off:off + nbytes]

        E = self.info["entries"]
        rows = sl(r.value, 4 * E * self.t).view(torch.int32).view(E, self.t) if self.t and E and self.info["fill_mode"] else None
        off = sl(o.value, 8 * (self.top + 1)).view(torch.int64)
        S = sl(s.value, 8 * (self.d + 1) * self.top).view(torch.int64).view(self.d + 1, self.top)
        return rows, off, S


def memo_build(gens, t: int, top: int, *, entries: bool = True, device=None, stream=None,
               memo_top: int | None = None) -> Memo:
    lay = Layout(gens, t, top, entries, memo_top=memo_top)
    return Memo(layout=lay, device=device, stream=stream)


def count(memo: Memo, n: int, stream=None) -> int:
    out = ctypes.c_uint64()
    _check(_L.fz_count(memo.h, n, _stream(stream), ctypes.byref(out)))
    return out.value


def shard_rows(memo: Memo, n: int, mode, nshards: int):
    rb = (ctypes.c_uint64 * nshards)()
    rl = (ctypes.c_uint64 * nshards)()
    _check(_L.fz_shard_rows(memo.h, n, _mode(mode), nshards, rb, rl))
    return list(rb), list(rl)


def plan_workspace_bytes(memo: Memo) -> int:
    nbytes = ctypes.c_uint64()
    _check(_L.fz_plan_workspace_bytes(memo.h, ctypes.byref(nbytes)))
    return nbytes.value


class Plan:
    """A shard plan (K4 output) in a device workspace tensor."""

    def __init__(self, memo: Memo, n: int, mode, shard: int = 0, nshards: int = 1, stream=None,
                 workspace: torch.Tensor | None = None):
        self.memo, self.n, self.mode = memo, int(n), _mode(mode)
        self.stream = stream          # the stream K4 runs on: shard() / result() synchronise it by default
        need = plan_workspace_bytes(memo)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=memo.ws.device)
        self.ws = workspace
        h = ctypes.c_void_p()
        _check(_L.fz_plan_create(memo.h, self.n, self.mode, shard, nshards, ctypes.c_void_p(self.ws.data_ptr()),
                                 need, _stream(stream), ctypes.byref(h)))
        self.h = h
        self._shard = None

    def shard(self, stream=None):
        """(row_begin, rows, nslices) as computed by K4 on the device (synchronises the plan's stream)."""
        if self._shard is None:
            rb, rl, ns = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
            s = stream if stream is not None else self.stream
            _check(_L.fz_plan_shard(self.h, _stream(s), ctypes.byref(rb), ctypes.byref(rl), ctypes.byref(ns)))
            self._shard = (rb.value, rl.value, ns.value)
        return self._shard

    WALKS = {0: "rows", 1: "deep", 2: "table", 3: "count_pairs", 4: "count_runs", 5: "count_staged"}

    def walk(self):
        """(kernel kind, bytes per card lookup) of this plan's enumeration (fz_plan_walk)."""
        k, cb = ctypes.c_int(), ctypes.c_int()
        _check(_L.fz_plan_walk(self.h, ctypes.byref(k), ctypes.byref(cb)))
        return self.WALKS[k.value], cb.value

    @property
    def row_begin(self):
        return self.shard()[0]

    @property
    def rows(self):
        return self.shard()[1]

    @property
    def nslices(self):
        return self.shard()[2]

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _L is not None:
            _L.fz_plan_free(h)
            self.h = None

    def launch(self, out: torch.Tensor | None = None, row_base: int | None = None, stream=None) -> None:
        """Asynchronous K5 launch.  `out` (MATERIALIZE) is an int32 tensor [>= rows, d]; row_base None
        keys the hash from the shard's first global row (read on the device)."""
        rb = (1 << 64) - 1 if row_base is None else int(row_base)
        ptr, cap = None, 0
        if out is not None:
            assert out.dtype in (torch.int32, torch.uint32) and out.is_contiguous()
            ptr, cap = out.data_ptr(), out.numel() // self.memo.d
        _check(_L.fz_enumerate_launch(self.h, ctypes.c_void_p(ptr), cap, rb,
                                      _stream(stream if stream is not None else self.stream)))

    def result(self, stream=None):
        """(rows, hash) of this shard after its enumeration (synchronises the plan's stream)."""
        r, h = ctypes.c_uint64(), ctypes.c_uint64()
        s = stream if stream is not None else self.stream
        _check(_L.fz_plan_result(self.h, _stream(s), ctypes.byref(r), ctypes.byref(h)))
        return r.value, h.value

    def result_tensor(self) -> torch.Tensor:
        """The plan's {rows, hash} u64 accumulators as an int64[2] device tensor view."""
        p = ctypes.c_void_p()
        _check(_L.fz_plan_result_ptr(self.h, ctypes.byref(p)))
        off = p.value - self.ws.data_ptr()
        return self.ws[off:off + 16].view(torch.int64)


def enumerate(memo: Memo, n: int, mode="materialize", *, out=None, shard: int = 0, nshards: int = 1,
              row_base: int | None = None, stream=None):
    """Plan + enumerate shard `shard` of Z(n).  Returns (rows tensor | None, row count, hash)."""
    plan = Plan(memo, n, mode, shard, nshards, stream=stream)
    m = plan.mode
    if m == MATERIALIZE and out is None:   # plan.rows synchronises `stream`, the one K4 ran on
        out = torch.empty((max(plan.rows, 1), memo.d), dtype=torch.int32, device=memo.ws.device)
    plan.launch(out if m == MATERIALIZE else None, row_base, stream=stream)
    rows, h = plan.result(stream=stream)
    if m == MATERIALIZE:
        return out[:plan.rows], rows, h
    return None, rows, h


def run_host(gens, t: int, n: int, mode="materialize", h_out: torch.Tensor | None = None, device=None, stream=None,
             workspace: torch.Tensor | None = None, ring_bytes: int = 0):
    """Whole path from host buffers (fz_run_host).  For MATERIALIZE, h_out is a (pinned) CPU int32
    tensor [>= |Z(n)|, d] that receives the rows, streamed through a device output ring: the part of
    `workspace` beyond the memo (allocated here with `ring_bytes` of ring, 0 = default, when None).
    Returns (rows, hash)."""
    garr = _gens(gens)
    d, m = len(gens), _mode(mode)
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if workspace is None:
        workspace = torch.empty(run_workspace_bytes(gens, t, n, mode, ring_bytes), dtype=torch.uint8, device=device)
    ptr, cap = None, 0
    if h_out is not None:
        ptr, cap = h_out.data_ptr(), h_out.numel() // d
    r, h = ctypes.c_uint64(), ctypes.c_uint64()
    _check(_L.fz_run_host(garr, d, int(t), int(n), m, ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                          ctypes.c_void_p(ptr), cap, _stream(stream), ctypes.byref(r), ctypes.byref(h)))
    return r.value, h.value


def run_workspace_bytes(gens, t: int, n: int, mode="materialize", ring_bytes: int = 0) -> int:
    """Device bytes fz_run_host needs: the memo, plan headers and (MATERIALIZE) an output ring of
    `ring_bytes` (0 = the default: what the output needs, at most 64 MB)."""
    nbytes = ctypes.c_uint64()
    _check(_L.fz_run_workspace_bytes(_gens(gens), len(gens), int(t), int(n), _mode(mode), int(ring_bytes),
                                     ctypes.byref(nbytes)))
    return nbytes.value
