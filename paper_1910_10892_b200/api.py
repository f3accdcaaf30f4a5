"""Python front end over the C-ABI (device tensors in, device tensors out).

Mirrors the reference's operator surface for the hot path
(/root/reference/proj/include/mp): ``isgmr_forward`` / ``trwp_forward``
(isgmr.hpp:145-152, trwp.hpp:148-156), ``isgmr_backward`` / ``trwp_backward``
(autodiff.hpp:63-197), the engine ``step()`` / ``aggregate()`` pair
(isgmr.hpp:49-59, trwp.hpp:47-61) and ``GridTopology`` (grid.hpp:73-96), with
a leading batch dimension. Argument meaning follows the reference; invalid
arguments raise ``MrfInvalidArgument`` (a ``ValueError``) where the reference
throws ``std::invalid_argument``.

PyTorch is only the device-memory / stream plumbing here: every computation
runs in libmrf_cuda.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ENGINE_ISGMR, ENGINE_TRWP, check, lib


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class GridTopology:
    """Scanline geometry for an H x W grid with 4/8/16 connectivity
    (mp::GridTopology, grid.hpp:73-96; identical scanline order and edge ids)."""

    def __init__(self, height: int, width: int, connectivity: int):
        h = C.c_void_p()
        check(lib().mrf_topology_create(height, width, connectivity, C.byref(h)))
        self._h = h
        self.height, self.width, self.connectivity = height, width, connectivity
        nd = C.c_int()
        te = C.c_int64()
        self.edge_count = np.zeros(connectivity, np.int64)
        self.dir_offset = np.zeros(connectivity, np.int64)
        check(lib().mrf_topology_info(h, C.byref(nd), C.byref(te),
                                      self.edge_count.ctypes.data_as(C.POINTER(C.c_int64)),
                                      self.dir_offset.ctypes.data_as(C.POINTER(C.c_int64))))
        self.num_dirs = nd.value
        self.total_edges = te.value

    @property
    def handle(self):
        return self._h

    @property
    def nodes(self):
        return self.height * self.width

    def edge_index(self) -> np.ndarray:
        out = np.zeros((self.num_dirs, self.nodes), np.int32)
        check(lib().mrf_topology_edge_index(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def scanlines(self, r: int):
        cnt = C.c_int32()
        check(lib().mrf_topology_scanlines(self._h, r, None, None, C.byref(cnt), 0))
        first = np.zeros(cnt.value, np.int32)
        length = np.zeros(cnt.value, np.int32)
        check(lib().mrf_topology_scanlines(self._h, r, first.ctypes.data_as(C.c_void_p),
                                           length.ctypes.data_as(C.c_void_p), C.byref(cnt), cnt.value))
        return first, length

    def index_bytes(self, labels: int, iterations: int) -> int:
        """IndexStore::bytes() == K * sum_r |E^r| * (L + 1) (index_store.hpp:11-15)."""
        return iterations * self.total_edges * (labels + 1)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().mrf_topology_destroy(h)
            except Exception:
                pass
            self._h = None


@dataclass
class MRF:
    """A batch of MRF instances sharing one topology and one pairwise table.

    unary   [B, N, L] float32 cuda       (UnaryVolume::values)
    V       [L, L]    float32 cuda       (PairwiseFunction::table)
    weight  float, or [B, R/2, N] tensor (EdgeWeights constant / planes)
    rho     float, or [B, R/2, N] tensor (TreeCoefficients, TRWP only)
    assume_finite  skip the forward's non-finite unary scan (the reference
                   engines throw on non-finite unaries; default: scan)
    """

    topo: GridTopology
    unary: torch.Tensor
    V: torch.Tensor
    weight: float | torch.Tensor = 1.0
    rho: float | torch.Tensor = 0.5
    assume_finite: bool = False

    def __post_init__(self):
        t = self.topo
        if self.unary.dim() == 2:
            self.unary = self.unary.unsqueeze(0)
        if self.unary.dim() != 3 or self.unary.shape[1] != t.nodes:
            raise ValueError("unary must be [B, H*W, L]")
        for name in ("unary", "V"):
            x = getattr(self, name)
            if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
        L = self.labels
        if tuple(self.V.shape) != (L, L):
            raise ValueError("V must be [L, L]")
        for name in ("weight", "rho"):
            x = getattr(self, name)
            if isinstance(x, torch.Tensor):
                if x.dim() == 2:
                    x = x.unsqueeze(0)
                    setattr(self, name, x)
                if tuple(x.shape) != (self.batch, t.num_dirs // 2, t.nodes) or x.dtype != torch.float32 \
                        or not x.is_cuda or not x.is_contiguous():
                    raise ValueError(f"{name} planes must be contiguous float32 CUDA [B, R/2, N]")

    @property
    def batch(self):
        return self.unary.shape[0]

    @property
    def labels(self):
        return self.unary.shape[2]

    def c_problem(self, diag_gap: torch.Tensor | None = None) -> _lib.Problem:
        t = self.topo
        wt = self.weight if isinstance(self.weight, torch.Tensor) else None
        rt = self.rho if isinstance(self.rho, torch.Tensor) else None
        return _lib.Problem(self.batch, t.height, t.width, self.labels, self.unary.data_ptr(), self.V.data_ptr(),
                            0.0 if wt is not None else float(self.weight), None if wt is None else wt.data_ptr(),
                            0.5 if rt is not None else float(self.rho), None if rt is None else rt.data_ptr(),
                            int(self.assume_finite), None if diag_gap is None else diag_gap.data_ptr())


@dataclass
class ForwardResult:
    """mp::ForwardResult (inference.hpp:62-68) for a batch: cost [B,N,L],
    labels [B,N] (int32 view of uint16), messages [B,R,N,L], p [B,K,E,L],
    q [B,K,E]."""

    cost: torch.Tensor
    labels: torch.Tensor
    messages: torch.Tensor
    p: torch.Tensor
    q: torch.Tensor
    iterations: int
    # [B] (diagnostic=True) or None: the reference's min_argmin_gap (+inf when untracked)
    min_argmin_gap: torch.Tensor | None = None


@dataclass
class GradientSet:
    """mp::GradientSet (autodiff.hpp:17-29): unary [B,N,L], pairwise [B,L,L],
    edge_weights [B,R/2,N]."""

    unary: torch.Tensor
    pairwise: torch.Tensor
    edge_weights: torch.Tensor

    def edge_weight_total(self):
        return self.edge_weights.sum(dim=(1, 2))


def _alloc_forward(mrf: MRF, K: int):
    t, B, L = mrf.topo, mrf.batch, mrf.labels
    dev = mrf.unary.device
    return ForwardResult(
        cost=torch.empty((B, t.nodes, L), dtype=torch.float32, device=dev),
        labels=torch.empty((B, t.nodes), dtype=torch.int16, device=dev),
        messages=torch.empty((B, t.num_dirs, t.nodes, L), dtype=torch.float32, device=dev),
        p=torch.empty((B, K, t.total_edges, L), dtype=torch.uint8, device=dev),
        q=torch.empty((B, K, t.total_edges), dtype=torch.uint8, device=dev),
        iterations=K)


_WS: dict = {}


def _workspace(kind: str, nbytes: int, device, stream):
    """Per-(device, stream, kind) workspace reused across calls. Calls on one
    stream are ordered, so reuse is safe; it grows when a larger one is
    needed (the old buffer is released only after the stream drains it)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (str(device), s.cuda_stream, kind)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            buf.record_stream(s)
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _forward(engine: int, mrf: MRF, K: int, out: ForwardResult | None, stream, diagnostic: bool = False):
    if K < 1:
        raise _lib.MrfInvalidArgument(1, "iterations must be >= 1")
    out = out or _alloc_forward(mrf, K)
    gap = None
    if diagnostic:
        gap = torch.full((mrf.batch,), float("inf"), dtype=torch.float32, device=mrf.unary.device)
    out.min_argmin_gap = gap
    pr = mrf.c_problem(gap)
    wsb = lib().mrf_forward_workspace_bytes(mrf.topo.handle, C.byref(pr), engine, K)
    ws = _workspace("fwd", wsb, mrf.unary.device, stream)
    fo = _lib.ForwardOut(_ptr(out.cost), _ptr(out.labels), _ptr(out.messages), _ptr(out.p), _ptr(out.q))
    fn = lib().mrf_isgmr_forward_f32 if engine == ENGINE_ISGMR else lib().mrf_trwp_forward_f32
    check(fn(mrf.topo.handle, C.byref(pr), K, C.byref(fo), _ptr(ws), wsb, _stream(stream)))
    return out


def isgmr_forward(mrf: MRF, iterations: int, out: ForwardResult | None = None, stream=None,
                  diagnostic: bool = False) -> ForwardResult:
    """mp::isgmr_forward<float> (isgmr.hpp:145-152) for a batch. diagnostic=True
    also tracks min_argmin_gap (dense kernel: same results, slower)."""
    return _forward(ENGINE_ISGMR, mrf, iterations, out, stream, diagnostic)


def trwp_forward(mrf: MRF, iterations: int, out: ForwardResult | None = None, stream=None,
                 diagnostic: bool = False) -> ForwardResult:
    """mp::trwp_forward<float> (trwp.hpp:148-156) for a batch; rho from mrf.rho."""
    return _forward(ENGINE_TRWP, mrf, iterations, out, stream, diagnostic)


def _backward(engine: int, mrf: MRF, fwd_p, fwd_q, K: int, grad_cost, out: GradientSet | None, stream):
    t, B, L = mrf.topo, mrf.batch, mrf.labels
    dev = mrf.unary.device
    if grad_cost.shape != mrf.unary.shape:
        raise _lib.MrfInvalidArgument(1, "backward: cost gradient size mismatch")
    grad_cost = grad_cost.contiguous()
    out = out or GradientSet(torch.empty_like(mrf.unary), torch.empty((B, L, L), dtype=torch.float32, device=dev),
                             torch.empty((B, t.num_dirs // 2, t.nodes), dtype=torch.float32, device=dev))
    pr = mrf.c_problem()
    wsb = lib().mrf_backward_workspace_bytes(t.handle, C.byref(pr), engine, K)
    ws = _workspace("bwd", wsb, dev, stream)
    g = _lib.Grads(_ptr(out.unary), _ptr(out.pairwise), _ptr(out.edge_weights))
    fn = lib().mrf_isgmr_backward_f32 if engine == ENGINE_ISGMR else lib().mrf_trwp_backward_f32
    check(fn(t.handle, C.byref(pr), K, _ptr(fwd_p), _ptr(fwd_q), _ptr(grad_cost), C.byref(g), _ptr(ws), wsb,
             _stream(stream)))
    return out


def isgmr_backward(mrf: MRF, fwd: ForwardResult, grad_cost, out=None, stream=None) -> GradientSet:
    """mp::isgmr_backward<float> (autodiff.hpp:63-126) for a batch."""
    return _backward(ENGINE_ISGMR, mrf, fwd.p, fwd.q, fwd.iterations, grad_cost, out, stream)


def trwp_backward(mrf: MRF, fwd: ForwardResult, grad_cost, out=None, stream=None) -> GradientSet:
    """mp::trwp_backward<float> (autodiff.hpp:133-197) for a batch."""
    return _backward(ENGINE_TRWP, mrf, fwd.p, fwd.q, fwd.iterations, grad_cost, out, stream)


def aggregate(mrf: MRF, messages, cost=None, labels=None, stream=None):
    """aggregate_costs + argmin_labels (inference.hpp:25-57)."""
    t = mrf.topo
    cost = cost if cost is not None else torch.empty_like(mrf.unary)
    labels = labels if labels is not None else torch.empty((mrf.batch, t.nodes), dtype=torch.int16,
                                                           device=mrf.unary.device)
    pr = mrf.c_problem()
    check(lib().mrf_aggregate_f32(t.handle, C.byref(pr), _ptr(messages), _ptr(cost), _ptr(labels), _stream(stream)))
    return cost, labels


class _Engine:
    """Shared state of the engine classes: messages on the device, indices
    in a [B, K_cap, E, L] / [B, K_cap, E] store that grows by doubling when
    step() runs past its capacity (the reference regrows on every
    append_iteration, index_store.hpp:21-25)."""

    def __init__(self, mrf: MRF, max_iterations: int, diagnostic: bool):
        if mrf.labels > 256:
            raise _lib.MrfInvalidArgument(1, "engine: more than 256 labels")
        if not mrf.assume_finite and not check_finite(mrf.unary):
            raise _lib.MrfInvalidArgument(1, "engine: non-finite unary potential")
        t, dev = mrf.topo, mrf.unary.device
        self.mrf, self.k = mrf, 0
        self.K_cap = max(1, max_iterations)
        self.p = torch.empty((mrf.batch, self.K_cap, t.total_edges, mrf.labels), dtype=torch.uint8, device=dev)
        self.q = torch.empty((mrf.batch, self.K_cap, t.total_edges), dtype=torch.uint8, device=dev)
        self.gap = torch.full((mrf.batch,), float("inf"), dtype=torch.float32, device=dev) if diagnostic else None

    def _reserve(self):
        if self.k < self.K_cap:
            return
        cap = 2 * self.K_cap
        p = torch.empty((self.p.shape[0], cap) + tuple(self.p.shape[2:]), dtype=torch.uint8, device=self.p.device)
        q = torch.empty((self.q.shape[0], cap, self.q.shape[2]), dtype=torch.uint8, device=self.q.device)
        p[:, :self.K_cap].copy_(self.p)
        q[:, :self.K_cap].copy_(self.q)
        self.p, self.q, self.K_cap = p, q, cap

    def iterations(self):
        return self.k

    def indices(self):
        """(p, q) of the iterations run so far: [B, k, E, L], [B, k, E]."""
        return self.p[:, :self.k], self.q[:, :self.k]

    def aggregate(self, stream=None):
        return aggregate(self.mrf, self.messages(), stream=stream)

    def min_argmin_gap(self):
        """[B] floats in diagnostic mode, else +inf (not tracked)."""
        if self.gap is None:
            return torch.full((self.mrf.batch,), float("inf"))
        return self.gap.cpu()


class IsgmrEngine(_Engine):
    """mp::IsgmrEngine (isgmr.hpp:26-143): step() runs one iteration,
    aggregate() returns (cost, labels)."""

    def __init__(self, mrf: MRF, max_iterations: int = 1, diagnostic: bool = False):
        super().__init__(mrf, max_iterations, diagnostic)
        t = mrf.topo
        shape = (mrf.batch, t.num_dirs, t.nodes, mrf.labels)
        self.m = torch.zeros(shape, dtype=torch.float32, device=mrf.unary.device)
        self.mhat = torch.zeros(shape, dtype=torch.float32, device=mrf.unary.device)

    def step(self, stream=None):
        self._reserve()
        pr = self.mrf.c_problem(self.gap)
        check(lib().mrf_isgmr_step_f32(self.mrf.topo.handle, C.byref(pr), self.k, self.K_cap, _ptr(self.m),
                                       _ptr(self.mhat), _ptr(self.p), _ptr(self.q), _stream(stream)))
        self.m, self.mhat = self.mhat, self.m  # publish m <- mhat (isgmr.hpp:55)
        self.k += 1

    def messages(self):
        return self.m


class TrwpEngine(_Engine):
    """mp::TrwpEngine (trwp.hpp:25-146)."""

    def __init__(self, mrf: MRF, max_iterations: int = 1, diagnostic: bool = False):
        super().__init__(mrf, max_iterations, diagnostic)
        t = mrf.topo
        if not isinstance(mrf.rho, torch.Tensor) and not (0.0 < float(mrf.rho) <= 1.0):
            raise _lib.MrfInvalidArgument(1, "rho must be in (0, 1]")
        self.m = torch.zeros((mrf.batch, t.num_dirs, t.nodes, mrf.labels), dtype=torch.float32,
                             device=mrf.unary.device)

    def step(self, stream=None):
        self._reserve()
        pr = self.mrf.c_problem(self.gap)
        check(lib().mrf_trwp_step_f32(self.mrf.topo.handle, C.byref(pr), self.k, self.K_cap, _ptr(self.m),
                                      _ptr(self.p), _ptr(self.q), _stream(stream)))
        self.k += 1

    def messages(self):
        return self.m


def check_finite(x: torch.Tensor, stream=None) -> bool:
    flag = C.c_int()
    check(lib().mrf_check_finite_f32(_ptr(x), x.numel(), C.byref(flag), _stream(stream)))
    return bool(flag.value)


def pack_shared_grads(mrf: MRF, grads: GradientSet, out=None, stream=None):
    """[sum_b dV_b (L*L), sum of dw planes] -- the buffer one all-reduce sums."""
    L = mrf.labels
    out = out if out is not None else torch.empty(L * L + 1, dtype=torch.float32, device=mrf.unary.device)
    pr = mrf.c_problem()
    g = _lib.Grads(_ptr(grads.unary), _ptr(grads.pairwise), _ptr(grads.edge_weights))
    check(lib().mrf_pack_shared_grads_f32(C.byref(pr), mrf.topo.num_dirs, C.byref(g), _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ readout and evaluation

@dataclass
class SoftHeadResult:
    """mp::SoftHeadResult (softhead.hpp:15-20), batched; grad_cost is the
    soft_head_backward output (softhead.hpp:58-74), produced in the same pass."""
    confidence: torch.Tensor | None  # [B, N, L]
    disparity: torch.Tensor          # [B, N]
    loss: torch.Tensor               # [B] mean |disparity - target|
    grad_cost: torch.Tensor | None   # [B, N, L] d loss / d cost


def soft_head(cost: torch.Tensor, target: torch.Tensor, confidence: bool = False, grad: bool = True,
              stream=None) -> SoftHeadResult:
    """soft_head_forward + soft_head_backward (softhead.hpp:22-74) fused:
    cost [B, N, L] (aggregate output), target [B, N]."""
    if cost.dim() == 2:
        cost = cost.unsqueeze(0)
    if target.dim() == 1:
        target = target.unsqueeze(0)
    B, N, L = cost.shape
    if tuple(target.shape) != (B, N):
        raise _lib.MrfInvalidArgument(1, "soft_head_forward: target size mismatch")
    cost, target = cost.contiguous(), target.contiguous()
    conf = torch.empty_like(cost) if confidence else None
    disp = torch.empty((B, N), dtype=torch.float32, device=cost.device)
    g = torch.empty_like(cost) if grad else None
    loss = torch.empty(B, dtype=torch.float32, device=cost.device)
    check(lib().mrf_soft_head_f32(B, N, L, _ptr(cost), _ptr(target), _ptr(conf) if conf is not None else None,
                                  _ptr(disp), _ptr(g) if g is not None else None, _ptr(loss), _stream(stream)))
    return SoftHeadResult(conf, disp, loss, g)


def energy(mrf: MRF, labels: torch.Tensor, topo: GridTopology | None = None, stream=None):
    """mp::energy (potentials.hpp:175-199) of a labelling per image (float64
    numpy [B]); `topo` may be a separate evaluation topology of the same grid
    (the 4-connected protocol, mrfmp.cpp:91-94)."""
    t = topo or mrf.topo
    if labels.dim() == 1:
        labels = labels.unsqueeze(0)
    labels = labels.contiguous()
    if labels.dtype not in (torch.int16, torch.uint16) or tuple(labels.shape) != (mrf.batch, t.nodes):
        raise _lib.MrfInvalidArgument(1, "energy: labelling size mismatch")
    m = mrf
    if t is not mrf.topo:
        if (t.height, t.width) != (mrf.topo.height, mrf.topo.width) or t.num_dirs > mrf.topo.num_dirs:
            raise _lib.MrfInvalidArgument(1, "energy: evaluation topology must be the same grid with <= directions")
        w = mrf.weight
        if isinstance(w, torch.Tensor):  # families of the evaluation directions (same order)
            w = w[:, : t.num_dirs // 2].contiguous()
        m = MRF(t, mrf.unary, mrf.V, w, 0.5)
    pr = m.c_problem()
    out = (C.c_double * mrf.batch)()
    check(lib().mrf_energy_f32(t.handle, C.byref(pr), _ptr(labels), out, _stream(stream)))
    import numpy as np

    return np.array(out[:], dtype=np.float64)


def iterate_energy(engine: str, mrf: MRF, iterations: int, eval_topo: GridTopology | None = None, stream=None):
    """isgmr_iterate_energy / trwp_iterate_energy (isgmr.hpp:156-169,
    trwp.hpp:158-171): energy of the aggregated labelling after each
    iteration, on eval_topo when given."""
    eng = (IsgmrEngine if engine == "isgmr" else TrwpEngine)(mrf, iterations)
    out = []
    for _ in range(iterations):
        eng.step(stream)
        _, labels = eng.aggregate(stream)
        out.append(energy(mrf, labels, eval_topo, stream))
    return out


def sgm_iterative(mrf: MRF, iterations: int, variant: str = "standard", stream=None):
    """mp::sgm_iterative (baselines.hpp:108-161): `iterations` SGM rounds,
    each on the previous round's normalised message sum as its unary volume.
    Returns [(cost [B,N,L], labels [B,N] int16)] per round."""
    if iterations < 1:
        raise _lib.MrfInvalidArgument(1, "sgm_iterative: iterations must be >= 1")
    cur = MRF(mrf.topo, mrf.unary, mrf.V, mrf.weight, mrf.rho, mrf.assume_finite)
    out = []
    for k in range(iterations):
        cost, labels, msgs = sgm_forward(cur, variant, stream)
        out.append((cost, labels))
        if k + 1 < iterations:
            nxt = torch.empty_like(mrf.unary)
            pr = cur.c_problem()
            check(lib().mrf_sgm_next_unary_f32(cur.topo.handle, C.byref(pr), _ptr(msgs), _ptr(nxt), _stream(stream)))
            cur = MRF(mrf.topo, nxt, mrf.V, mrf.weight, mrf.rho, True)
    return out


def sgm_forward(mrf: MRF, variant: str = "standard", stream=None):
    """mp::sgm_forward (baselines.hpp:31-98): returns (cost [B,N,L], labels
    [B,N] int16, messages [B,R,N,L]). 'revised' is one ISGMR iteration."""
    t = mrf.topo
    v = {"standard": 0, "revised": 1}[variant]
    msgs = torch.empty((mrf.batch, t.num_dirs, t.nodes, mrf.labels), dtype=torch.float32, device=mrf.unary.device)
    cost = torch.empty_like(mrf.unary)
    labels = torch.empty((mrf.batch, t.nodes), dtype=torch.int16, device=mrf.unary.device)
    pr = mrf.c_problem()
    check(lib().mrf_sgm_f32(t.handle, C.byref(pr), v, _ptr(msgs), _ptr(cost), _ptr(labels), _stream(stream)))
    return cost, labels, msgs


# ------------------------------------------------------------------ MPCV1 I/O

_MPCV1 = b"MPCV1"


def save_cost_volume(path: str, volume) -> None:
    """Write an [H, W, L] float32 cost volume as MPCV1 (the reference's
    on-disk format, io.hpp:29-35 / io.cpp:118-131): magic, H, W, L as
    little-endian uint32, then the values row-major with label fastest."""
    import numpy as np

    v = volume.detach().cpu().numpy() if isinstance(volume, torch.Tensor) else np.asarray(volume)
    if v.ndim != 3:
        raise _lib.MrfInvalidArgument(1, "cost volume: expected [H, W, L]")
    H, W, L = v.shape
    with open(path, "wb") as f:
        f.write(_MPCV1 + np.array([H, W, L], "<u4").tobytes() + np.ascontiguousarray(v, "<f4").tobytes())


def load_cost_volume(path: str):
    """Read an MPCV1 cost volume as a float32 numpy [H, W, L] array, with the
    reference reader's checks (io.cpp:133-152): magic, non-zero sizes,
    L <= 256, complete payload, finite values."""
    import numpy as np

    with open(path, "rb") as f:
        raw = f.read()
    if raw[:5] != _MPCV1:
        raise ValueError(f"cost volume: bad magic in {path}")
    if len(raw) < 17:
        raise ValueError("cost volume: truncated header")
    H, W, L = (int(x) for x in np.frombuffer(raw[5:17], "<u4"))
    if not (H and W and L) or L > 256:
        raise ValueError("cost volume: invalid dimensions")
    n = H * W * L
    if len(raw) < 17 + 4 * n:
        raise ValueError("cost volume: truncated payload")
    v = np.frombuffer(raw[17:17 + 4 * n], "<f4").astype(np.float32).reshape(H, W, L)
    if not np.isfinite(v).all():
        raise ValueError("cost volume: non-finite value")
    return v
