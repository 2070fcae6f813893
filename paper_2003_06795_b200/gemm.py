"""Matmul-with-config: the Python face of the kernel families.

This is the call north_star asks for beside the reference's config ->
performance function (synthetic.analytic_perf, reference
pkg/src/kernelprune/synthetic.py:65): run *this* KernelConfig on *this*
problem, on the B200, through the C-ABI (include/kp_abi.h). PyTorch is used
only for device memory and the current CUDA stream; the arithmetic is in
libkp.so. There is no CPU fallback: without the library or a GPU every entry
point raises.

Operands are logical: ``a`` is op(A) with shape (m, k) or (batch, m, k) and
``b`` is op(B) with shape (k, n) or (batch, k, n). A transposed view (e.g.
``x.t()``) is passed to the kernel as a trans_a / trans_b layout without a
copy; a 2-D operand next to a 3-D one is broadcast with batch stride 0.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .dataset import KernelConfig


def _torch():
    import torch
    return torch


def _family_dtype(family: int):
    torch = _torch()
    return torch.bfloat16 if family == nat.BF16_TC else torch.float32


def _operand_layout(t, rows: int, cols: int):
    """(transposed, ld) for a logical rows x cols operand view, or None."""
    s_r, s_c = t.stride(-2), t.stride(-1)
    if s_c == 1 or cols == 1:
        ld = s_r if rows > 1 else cols
        if ld >= cols:
            return False, ld
    if s_r == 1 or rows == 1:
        ld = s_c if cols > 1 else rows
        if ld >= rows:
            return True, ld
    return None


def _prep(t, rows, cols):
    lay = _operand_layout(t, rows, cols)
    if lay is None:
        t = t.contiguous()
        lay = (False, cols)
    return t, lay


def describe(a, b, out=None, alpha: float = 1.0, beta: float = 0.0, family="f32"):
    """Validate operands and build (desc, a, b, out) for the C-ABI."""
    torch = _torch()
    fam = nat.family_id(family)
    want = _family_dtype(fam)
    if a.dim() not in (2, 3) or b.dim() not in (2, 3):
        raise nat.BadProblemShape("operands must be 2-D or 3-D (batched)")
    if a.dtype != want or b.dtype != want:
        raise nat.BadProblemShape(f"family {family!r} expects {want} operands, "
                                  f"got {a.dtype} and {b.dtype}")
    check_device(a, b, out)
    m, k = a.shape[-2], a.shape[-1]
    k2, n = b.shape[-2], b.shape[-1]
    if k != k2:
        raise nat.BadProblemShape(f"inner dims differ: a is {tuple(a.shape)}, b is {tuple(b.shape)}")
    batch_a = a.shape[0] if a.dim() == 3 else 1
    batch_b = b.shape[0] if b.dim() == 3 else 1
    if batch_a != batch_b and 1 not in (batch_a, batch_b):
        raise nat.BadProblemShape("batch sizes differ")
    batch = max(batch_a, batch_b)
    a, (ta, lda) = _prep(a, m, k)
    b, (tb, ldb) = _prep(b, k, n)
    sa = a.stride(0) if a.dim() == 3 and batch_a > 1 else 0
    sb = b.stride(0) if b.dim() == 3 and batch_b > 1 else 0
    shape = (batch, m, n) if (a.dim() == 3 or b.dim() == 3) else (m, n)
    if out is None:
        if beta != 0.0:
            raise nat.BadProblemShape("beta != 0 needs an `out` tensor")
        out = torch.empty(shape, dtype=torch.float32, device=a.device)
    else:
        if out.dtype != torch.float32 or tuple(out.shape) != shape or out.stride(-1) != 1:
            raise nat.BadProblemShape(f"out must be float32 {shape} with unit column stride")
    ldc = out.stride(-2) if m > 1 else n
    sc = out.stride(0) if out.dim() == 3 else m * ldc
    desc = nat.KpGemmDesc(batch, m, k, n, int(ta), int(tb), lda, ldb, ldc, sa, sb, sc,
                          float(alpha), float(beta))
    return desc, a, b, out


def check_device(*tensors):
    """All tensors (None skipped) are CUDA tensors on one device; returns it.
    A CPU tensor or a second device would otherwise reach the kernels as a
    foreign pointer and fault the context instead of raising."""
    devs = {t.device for t in tensors if t is not None}
    if any(d.type != "cuda" for d in devs):
        raise nat.KernelLibraryError("operands must be CUDA tensors (no CPU fallback)")
    if len(devs) != 1:
        raise nat.BadProblemShape(f"operands live on different devices: {sorted(map(str, devs))}")
    return devs.pop()


def _stream_handle(device=None):
    """The current stream of `device` (default: the current device)."""
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def on_device(t):
    """Context making t's device current, so the library launches there."""
    return _torch().cuda.device(t.device)


def matmul(a, b, config=None, *, family="f32", out=None, alpha: float = 1.0,
           beta: float = 0.0):
    """C = alpha * a @ b + beta * out on the GPU with one kernel config.

    ``config=None`` uses the runtime selector compiled into the library (the
    generated decision-tree header, codegen.emit_selector_source).
    """
    fam = nat.family_id(family)
    desc, a, b, out = describe(a, b, out, alpha, beta, family)
    lib = nat.lib()
    with on_device(a):
        if config is None:
            chosen = nat.KpConfig()
            nat.check(lib.kp_gemm_auto(fam, ctypes.byref(desc), a.data_ptr(), b.data_ptr(),
                                       out.data_ptr(), _stream_handle(a.device),
                                       ctypes.byref(chosen)), "kp_gemm_auto")
        else:
            nat.check(lib.kp_gemm(fam, nat.to_kp_config(config), ctypes.byref(desc),
                                  a.data_ptr(), b.data_ptr(), out.data_ptr(),
                                  _stream_handle(a.device)), "kp_gemm")
    return out


def matmul_host(a: np.ndarray, b: np.ndarray, config=None, *, family="f32", device=0):
    """Host-buffer entry point (numpy in, numpy out): pinned H2D copies, the
    kernel, and the D2H copy, all stream-ordered. Used for the e2e figure."""
    torch = _torch()
    fam = nat.family_id(family)
    want = _family_dtype(fam)
    ta = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).pin_memory()
    tb = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float32)).pin_memory()
    dev = torch.device("cuda", device)
    da = ta.to(dev, non_blocking=True).to(want)
    db = tb.to(dev, non_blocking=True).to(want)
    dc = matmul(da, db, config, family=family)
    host = torch.empty(dc.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(dc, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy()


def matmul_pinned(a_host, b_host, out_host, config=None, *, family="f32"):
    """End-to-end call on pinned host tensors: H2D copies, the kernel (runtime
    selector when config is None), D2H copy, stream synchronise."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    want = _family_dtype(nat.family_id(family))
    da = a_host.to(dev, non_blocking=True)
    db = b_host.to(dev, non_blocking=True)
    if da.dtype != want:
        da, db = da.to(want), db.to(want)
    dc = matmul(da, db, config, family=family)
    out_host.copy_(dc, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out_host


class PinnedPipeline:
    """End-to-end GEMMs on pinned host buffers with the copies overlapped.

    Three streams ordered by events: copy-in (H2D), compute, copy-out (D2H).
    Problems are issued largest first; a large FP32 problem is split into
    row blocks of A / C (B copied once, first), so the kernel of block j and
    the D2H of block j-1 run under the H2D of block j+1 and the host link
    stays busy from the first byte to the last (rows of C are independent
    and every K1 config accumulates each element in the same k order, so the
    blocks give exactly the unsplit result).  Device buffers are cached per
    shape.

    ``graph=True`` captures one step per distinct problem list (same host
    buffers) into a CUDA graph on first use and replays it afterwards: the
    whole H2D / kernel / D2H schedule then costs one launch of host work.
    Replays read whatever the host buffers hold at replay time."""

    CHUNK_BYTES = 4 << 20   # A bytes per row block of a split problem (tools/e2e_probe.py)
    MIN_ROWS = 256

    def __init__(self, family="f32", graph: bool = False):
        torch = _torch()
        self.family = family
        self.graph = graph
        self._graphs = {}
        self.want = _family_dtype(nat.family_id(family))
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_run = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self._bufs = {}

    def _buffers(self, i, a_host, b_host, out_host):
        torch = _torch()
        key = (i, tuple(a_host.shape), tuple(b_host.shape))
        if key not in self._bufs:
            self._bufs[key] = (torch.empty(a_host.shape, dtype=a_host.dtype, device=self.dev),
                               torch.empty(b_host.shape, dtype=b_host.dtype, device=self.dev),
                               torch.empty(out_host.shape, dtype=torch.float32, device=self.dev))
        return self._bufs[key]

    def _blocks(self, a_host):
        """Row blocks [(r0, r1)] of one problem (one block unless it is a
        large 2-D FP32 problem)."""
        m = a_host.shape[0]
        if (self.family != "f32" or a_host.dim() != 2 or not a_host.is_contiguous()):
            return [(0, m)]
        nbytes = a_host.numel() * a_host.element_size()
        nblk = min(max(1, -(-nbytes // self.CHUNK_BYTES)), max(1, m // self.MIN_ROWS))
        step = -(-m // nblk)
        return [(r, min(m, r + step)) for r in range(0, m, step)]

    def run(self, problems, configs=None):
        """problems: [(a_host, b_host, out_host)] pinned; returns when all
        results are in the host buffers."""
        torch = _torch()
        if not self.graph:
            self._enqueue(problems, configs)
            self.s_out.synchronize()
            return [hc for _, _, hc in problems]
        key = tuple((a.data_ptr(), b.data_ptr(), c.data_ptr(), tuple(a.shape), tuple(b.shape),
                     tuple(c.shape)) for a, b, c in problems)
        key += (None if configs is None else tuple(tuple(_cfg_tuple(c)) for c in configs),)
        entry = self._graphs.get(key)
        if entry is None:
            self._enqueue(problems, configs)   # buffers, selectors, kernel attributes
            self.s_out.synchronize()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.dev)
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=cap):
                for st in (self.s_in, self.s_run, self.s_out):
                    st.wait_stream(cap)
                self._enqueue(problems, configs)
                for st in (self.s_in, self.s_run, self.s_out):
                    cap.wait_stream(st)
            entry = self._graphs[key] = g
        entry.replay()
        torch.cuda.current_stream().synchronize()
        return [hc for _, _, hc in problems]

    def _enqueue(self, problems, configs):
        torch = _torch()
        order = sorted(range(len(problems)),
                       key=lambda i: -problems[i][0].numel() * problems[i][1].shape[-1])
        items = []  # (problem, r0, r1, h2d event)
        with torch.cuda.stream(self.s_in):
            for i in order:
                ha, hb, hc = problems[i]
                da, db, dc = self._buffers(i, ha, hb, hc)
                db.copy_(hb, non_blocking=True)
                for r0, r1 in self._blocks(ha):
                    da[r0:r1].copy_(ha[r0:r1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self.s_in)
                    items.append((i, r0, r1, ev))
        for i, r0, r1, ev_in in items:
            ha, hb, hc = problems[i]
            da, db, dc = self._buffers(i, ha, hb, hc)
            whole = r0 == 0 and r1 == ha.shape[0]
            with torch.cuda.stream(self.s_run):
                self.s_run.wait_event(ev_in)
                xa, xb = (da, db) if da.dtype == self.want else (da.to(self.want), db.to(self.want))
                cfg = None if configs is None else configs[i]
                if whole:
                    matmul(xa, xb, cfg, family=self.family, out=dc)
                else:
                    matmul(xa[r0:r1], xb, cfg, family=self.family, out=dc[r0:r1])
                ev = torch.cuda.Event()
                ev.record(self.s_run)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev)
                if whole:
                    hc.copy_(dc, non_blocking=True)
                else:
                    hc[r0:r1].copy_(dc[r0:r1], non_blocking=True)


def _cfg_tuple(cfg):
    return cfg.as_tuple() if hasattr(cfg, "as_tuple") else tuple(cfg)


def time_config(a, b, config, *, family="f32", out=None, warmup: int = 3, reps: int = 10,
                min_sample_ns: float = 50_000.0, max_cell_ns: float = 0.0) -> float:
    """Median per-launch device time (ns) of one config on one problem."""
    fam = nat.family_id(family)
    desc, a, b, out = describe(a, b, out, 1.0, 0.0, family)
    res = ctypes.c_double()
    with on_device(a):
        nat.check(nat.lib().kp_gemm_time(fam, nat.to_kp_config(config), ctypes.byref(desc),
                                         a.data_ptr(), b.data_ptr(), out.data_ptr(), warmup,
                                         reps, min_sample_ns, max_cell_ns, ctypes.byref(res),
                                         _stream_handle(a.device)),
                  "kp_gemm_time")
    return res.value


def sweep_problem(a, b, configs, *, family="f32", out=None, warmup: int = 2, reps: int = 5,
                  min_sample_ns: float = 50_000.0, max_cell_ns: float = 0.0,
                  early_exit: bool = True) -> list[float]:
    """Median runtime (ns) of every config on one problem (C++ timing loop,
    kp_sweep_problem_ex). ``early_exit=False`` gives every config the full
    statistic (config-range tasks of a split problem)."""
    fam = nat.family_id(family)
    desc, a, b, out = describe(a, b, out, 1.0, 0.0, family)
    cfgs = (nat.KpConfig * len(configs))(*[nat.to_kp_config(c) for c in configs])
    res = (ctypes.c_double * len(configs))()
    with on_device(a):
        nat.check(nat.lib().kp_sweep_problem_ex(fam, cfgs, len(configs), ctypes.byref(desc),
                                                a.data_ptr(), b.data_ptr(), out.data_ptr(),
                                                warmup, reps, min_sample_ns, max_cell_ns,
                                                1 if early_exit else 0, res,
                                                _stream_handle(a.device)),
                  "kp_sweep_problem_ex")
    return list(res)


def family_configs(family="f32") -> tuple[KernelConfig, ...]:
    """The family's config list in canonical order (kp_config_at)."""
    fam = nat.family_id(family)
    lib = nat.lib()
    out = []
    cfg = nat.KpConfig()
    for i in range(lib.kp_num_configs(fam)):
        nat.check(lib.kp_config_at(fam, i, ctypes.byref(cfg)), "kp_config_at")
        out.append(KernelConfig(*cfg.as_tuple()))
    return tuple(out)


def select(m: int, k: int, n: int, *, family="f32", trans_a=False, trans_b=False,
           batch: int = 1) -> KernelConfig:
    """The config the compiled runtime selector returns for (m, k, n) (the
    strided-batched selector when batch > 1, kp_select_ex)."""
    cfg = nat.KpConfig()
    nat.check(nat.lib().kp_select_ex(nat.family_id(family), int(trans_a), int(trans_b), batch,
                                     m, k, n, ctypes.byref(cfg)), "kp_select_ex")
    return KernelConfig(*cfg.as_tuple())


def auto_config(m: int, k: int, n: int, *, family="f32", trans_a=False, trans_b=False,
                batch: int = 1):
    """What kp_gemm_auto runs for (m, k, n): the selector's KernelConfig, or
    "skinny" when the small-M path (m <= 16) takes the problem."""
    cfg = nat.KpConfig()
    nat.check(nat.lib().kp_auto_config(nat.family_id(family), int(trans_a), int(trans_b), batch,
                                       m, k, n, ctypes.byref(cfg)), "kp_auto_config")
    t = cfg.as_tuple()
    return nat.SKINNY if t == (0, 0, 0, 0, 0) else KernelConfig(*t)


def set_skinny(mode: int) -> int:
    """kp_set_skinny: 0 never, 1 auto (default), 2 every m <= 16 problem."""
    prev = int(nat.lib().kp_set_skinny(int(mode)))
    if prev < 0:
        raise ValueError(f"invalid skinny mode {mode}")
    return prev


def launch_count() -> int:
    return int(nat.lib().kp_launch_count())


_OP = None


def torch_op():
    """Register (once) and return ``torch.ops.kernelprune.matmul(a, b, family)``:
    the runtime-selected GEMM (kp_gemm_auto) as a PyTorch custom operator, so
    the deployed library is callable from torch code, torch.compile graphs and
    TorchScript-free C++ callers of the dispatcher alike. A fake (meta)
    implementation gives shape/dtype propagation without a launch."""
    global _OP
    if _OP is not None:
        return _OP
    torch = _torch()

    @torch.library.custom_op("kernelprune::matmul", mutates_args=(),
                             schema="(Tensor a, Tensor b, str family) -> Tensor")
    def _matmul(a, b, family):
        return matmul(a, b, None, family=family)

    @_matmul.register_fake
    def _(a, b, family):
        return a.new_empty(a.shape[:-1] + b.shape[-1:], dtype=torch.float32)

    _OP = torch.ops.kernelprune.matmul
    return _OP
