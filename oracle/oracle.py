"""TEST INFRASTRUCTURE ONLY: numpy/ctypes front end for the CPU checkers.

Two checkers live under oracle/:
  * ``lib/libmrf_oracle.so`` -- the plain-C restatement (mrf_oracle.c);
  * ``_ref/libmrf_ref.so``   -- the unmodified reference library compiled from
    /root/reference/proj sources plus the ref_capi.cpp shim (present wherever it
    was built; it travels to the GPU box with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference arm
may import this module. The product package never does.

Array conventions follow the reference layouts:
  unary [N][L] f32, V [L][L] f32 (V(a,b)=V[a*L+b]), weight/rho planes [R/2][N],
  messages [R][N][L], p [K][E][L] u8, q [K][E] u8, cost [N][L], labels [N] u16.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "libmrf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmrf_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build(quiet: bool = True) -> None:
    """Compile the restatement (always) and the reference shim (when the
    reference tree exists)."""
    import subprocess

    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


_libs: dict = {}


def _load(path):
    if path not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        _libs[path] = C.CDLL(path)
    return _libs[path]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def _orc():
    lib = _load(ORACLE_SO)
    if not getattr(lib, "_typed", False):
        lib.orc_topo_create.restype = _vp
        lib.orc_topo_create.argtypes = [C.c_int, C.c_int, C.c_int]
        lib.orc_topo_free.argtypes = [_vp]
        lib.orc_total_edges.restype = C.c_int64
        lib.orc_total_edges.argtypes = [_vp]
        lib.orc_topo_dump.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int]
        for f in ("orc_isgmr_forward", "orc_trwp_forward"):
            getattr(lib, f).argtypes = [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp, _vp]
        for f in ("orc_isgmr_backward", "orc_trwp_backward"):
            getattr(lib, f).argtypes = [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.orc_soft_head.restype = C.c_float
        lib.orc_soft_head.argtypes = [C.c_int, C.c_int, _vp, _vp, _vp, _vp]
        lib._typed = True
    return lib


def _ref():
    lib = _load(REF_SO)
    if not getattr(lib, "_typed", False):
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_topology.argtypes = [C.c_int] * 3 + [_vp] * 7 + [C.c_int]
        lib.ref_scanline_nodes.argtypes = [C.c_int] * 4 + [_vp]
        lib.ref_isgmr_forward_f32.argtypes = [C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, C.c_int, C.c_int] + [_vp] * 6
        lib.ref_trwp_forward_f32.argtypes = ([C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, C.c_float, _vp,
                                             C.c_int, C.c_int] + [_vp] * 6)
        lib.ref_isgmr_backward_f32.argtypes = ([C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, C.c_int, _vp, _vp, _vp,
                                               C.c_int, _vp, _vp, _vp])
        lib.ref_trwp_backward_f32.argtypes = ([C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, C.c_float, _vp, C.c_int,
                                              _vp, _vp, _vp, C.c_int, _vp, _vp, _vp])
        lib.ref_soft_head_f32.argtypes = [C.c_int] * 3 + [_vp] * 5
        lib.ref_sgm_revised_f32.argtypes = [C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, _vp, _vp]
        lib.ref_energy_f32.argtypes = [C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, _vp, _vp]
        lib.ref_sgm_standard_f32.argtypes = [C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, _vp, _vp, _vp]
        lib.ref_sgm_iterative_f32.argtypes = [C.c_int] * 4 + [_vp, _vp, C.c_float, _vp, C.c_int, C.c_int, _vp, _vp]
        lib.ref_gradient_check.argtypes = [C.c_int] * 7 + [C.c_uint64, _vp, _vp, _vp]
        lib._typed = True
    return lib


def _check_ref(rc):
    if rc != 0:
        raise ValueError(_ref().ref_last_error().decode())


# --------------------------------------------------------------------------- problems

@dataclass
class Problem:
    """One MRF instance in reference layout (float32 unless noted)."""

    H: int
    W: int
    L: int
    conn: int
    unary: np.ndarray                 # [N*L]
    V: np.ndarray                     # [L*L]
    w_const: float = 1.0
    w_planes: np.ndarray | None = None   # [R/2 * N]
    rho_const: float = 0.5
    rho_planes: np.ndarray | None = None  # [R/2 * N]

    @property
    def N(self):
        return self.H * self.W

    def c_struct(self):
        return _OrcProblem(self.H, self.W, self.L, _ptr(self.unary), _ptr(self.V), self.w_const,
                           _ptr(self.w_planes), self.rho_const, _ptr(self.rho_planes))


class _OrcProblem(C.Structure):
    _fields_ = [("H", C.c_int), ("W", C.c_int), ("L", C.c_int), ("unary", C.c_void_p),
                ("pairwise", C.c_void_p), ("w_const", C.c_float), ("w_planes", C.c_void_p),
                ("rho_const", C.c_float), ("rho_planes", C.c_void_p)]


@dataclass
class Topology:
    total_edges: int
    edge_count: np.ndarray   # [R] int64
    dir_offset: np.ndarray   # [R] int64
    edge_index: np.ndarray   # [R][N] int32
    nlines: np.ndarray       # [R] int32
    line_first: list         # R arrays
    line_len: list           # R arrays


def _topo_arrays(H, W, conn):
    R, N = conn, H * W
    cap = W + (H - 1) * 2 + (W - 1) * 2 + H + 4
    return (np.zeros(R, np.int64), np.zeros(R, np.int64), np.zeros(R * N, np.int32), np.zeros(R, np.int32),
            np.zeros(R * cap, np.int32), np.zeros(R * cap, np.int32), cap)


def _topo_pack(total, ec, do, ei, nl, lf, ll, cap, H, W, conn):
    R, N = conn, H * W
    return Topology(int(total), ec, do, ei.reshape(R, N), nl,
                    [lf[r * cap:r * cap + nl[r]].copy() for r in range(R)],
                    [ll[r * cap:r * cap + nl[r]].copy() for r in range(R)])


def oracle_topology(H, W, conn) -> Topology:
    lib = _orc()
    t = lib.orc_topo_create(H, W, conn)
    if not t:
        raise ValueError("invalid topology")
    try:
        ec, do, ei, nl, lf, ll, cap = _topo_arrays(H, W, conn)
        lib.orc_topo_dump(t, _ptr(ec), _ptr(do), _ptr(ei), _ptr(nl), _ptr(lf), _ptr(ll), cap)
        return _topo_pack(lib.orc_total_edges(t), ec, do, ei, nl, lf, ll, cap, H, W, conn)
    finally:
        lib.orc_topo_free(t)


def ref_topology(H, W, conn) -> Topology:
    lib = _ref()
    ec, do, ei, nl, lf, ll, cap = _topo_arrays(H, W, conn)
    tot = np.zeros(1, np.int64)
    _check_ref(lib.ref_topology(H, W, conn, _ptr(tot), _ptr(ec), _ptr(do), _ptr(ei), _ptr(nl), _ptr(lf),
                                _ptr(ll), cap))
    return _topo_pack(tot[0], ec, do, ei, nl, lf, ll, cap, H, W, conn)


def total_edges(H, W, conn) -> int:
    lib = _orc()
    t = lib.orc_topo_create(H, W, conn)
    try:
        return int(lib.orc_total_edges(t))
    finally:
        lib.orc_topo_free(t)


# --------------------------------------------------------------------------- engines

@dataclass
class Forward:
    cost: np.ndarray
    labels: np.ndarray
    messages: np.ndarray
    p: np.ndarray
    q: np.ndarray
    gap: float = float("inf")  # ForwardResult::min_argmin_gap (impl="ref" only)


@dataclass
class Grads:
    unary: np.ndarray
    pairwise: np.ndarray
    wplanes: np.ndarray


def _fwd_buffers(pr: Problem, K: int):
    E = total_edges(pr.H, pr.W, pr.conn)
    N, L, R = pr.N, pr.L, pr.conn
    return Forward(np.zeros(N * L, np.float32), np.zeros(N, np.uint16), np.zeros(R * N * L, np.float32),
                   np.zeros(K * E * L, np.uint8), np.zeros(K * E, np.uint8))


def _grad_buffers(pr: Problem):
    return Grads(np.zeros(pr.N * pr.L, np.float32), np.zeros(pr.L * pr.L, np.float32),
                 np.zeros((pr.conn // 2) * pr.N, np.float32))


def forward(engine: str, pr: Problem, K: int, impl: str = "oracle", threads: int = 1) -> Forward:
    """engine in {"isgmr","trwp"}; impl in {"oracle","ref"}."""
    out = _fwd_buffers(pr, K)
    if impl == "oracle":
        lib = _orc()
        t = lib.orc_topo_create(pr.H, pr.W, pr.conn)
        st = pr.c_struct()
        try:
            fn = lib.orc_isgmr_forward if engine == "isgmr" else lib.orc_trwp_forward
            rc = fn(t, C.byref(st), K, _ptr(out.cost), _ptr(out.labels), _ptr(out.messages), _ptr(out.p),
                    _ptr(out.q))
        finally:
            lib.orc_topo_free(t)
        if rc != 0:
            raise ValueError("oracle forward: invalid argument")
    else:
        lib = _ref()
        gap = np.zeros(1, np.float32)
        if engine == "isgmr":
            _check_ref(lib.ref_isgmr_forward_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                                 _ptr(pr.w_planes), K, threads, _ptr(out.cost), _ptr(out.labels),
                                                 _ptr(out.messages), _ptr(out.p), _ptr(out.q), _ptr(gap)))
        else:
            _check_ref(lib.ref_trwp_forward_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                                _ptr(pr.w_planes), pr.rho_const, _ptr(pr.rho_planes), K, threads,
                                                _ptr(out.cost), _ptr(out.labels), _ptr(out.messages), _ptr(out.p),
                                                _ptr(out.q), _ptr(gap)))
        out.gap = float(gap[0])
    return out


def backward(engine: str, pr: Problem, K: int, p, q, grad_cost, impl: str = "oracle", threads: int = 1) -> Grads:
    g = _grad_buffers(pr)
    grad_cost = np.ascontiguousarray(grad_cost, np.float32)
    if impl == "oracle":
        lib = _orc()
        t = lib.orc_topo_create(pr.H, pr.W, pr.conn)
        st = pr.c_struct()
        try:
            fn = lib.orc_isgmr_backward if engine == "isgmr" else lib.orc_trwp_backward
            rc = fn(t, C.byref(st), K, _ptr(p), _ptr(q), _ptr(grad_cost), _ptr(g.unary), _ptr(g.pairwise),
                    _ptr(g.wplanes))
        finally:
            lib.orc_topo_free(t)
        if rc != 0:
            raise ValueError("oracle backward: invalid argument")
    else:
        lib = _ref()
        if engine == "isgmr":
            _check_ref(lib.ref_isgmr_backward_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                                  _ptr(pr.w_planes), K, _ptr(p), _ptr(q), _ptr(grad_cost), threads,
                                                  _ptr(g.unary), _ptr(g.pairwise), _ptr(g.wplanes)))
        else:
            _check_ref(lib.ref_trwp_backward_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                                 _ptr(pr.w_planes), pr.rho_const, _ptr(pr.rho_planes), K, _ptr(p),
                                                 _ptr(q), _ptr(grad_cost), threads, _ptr(g.unary),
                                                 _ptr(g.pairwise), _ptr(g.wplanes)))
    return g


def soft_head(cost, target, L, impl: str = "oracle"):
    cost = np.ascontiguousarray(cost, np.float32)
    target = np.ascontiguousarray(target, np.float32)
    N = target.size
    disp = np.zeros(N, np.float32)
    grad = np.zeros(N * L, np.float32)
    if impl == "oracle":
        loss = _orc().orc_soft_head(N, L, _ptr(cost), _ptr(target), _ptr(disp), _ptr(grad))
    else:
        lossb = np.zeros(1, np.float32)
        _check_ref(_ref().ref_soft_head_f32(1, N, L, _ptr(cost), _ptr(target), _ptr(lossb), _ptr(disp), _ptr(grad)))
        loss = float(lossb[0])
    return float(loss), disp, grad


def ref_sgm_revised(pr: Problem):
    cost = np.zeros(pr.N * pr.L, np.float32)
    msg = np.zeros(pr.conn * pr.N * pr.L, np.float32)
    _check_ref(_ref().ref_sgm_revised_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                          _ptr(pr.w_planes), _ptr(cost), _ptr(msg)))
    return cost, msg


def ref_sgm_standard(pr: Problem):
    cost = np.zeros(pr.N * pr.L, np.float32)
    labels = np.zeros(pr.N, np.uint16)
    msg = np.zeros(pr.conn * pr.N * pr.L, np.float32)
    _check_ref(_ref().ref_sgm_standard_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                           _ptr(pr.w_planes), _ptr(cost), _ptr(labels), _ptr(msg)))
    return cost, labels, msg


def ref_sgm_iterative(pr: Problem, K: int, variant: str = "standard"):
    """mp::sgm_iterative of the reference: [(cost, labels)] per round."""
    costs = np.zeros((K, pr.N * pr.L), np.float32)
    labels = np.zeros((K, pr.N), np.uint16)
    _check_ref(_ref().ref_sgm_iterative_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                            _ptr(pr.w_planes), K, int(variant == "revised"), _ptr(costs),
                                            _ptr(labels)))
    return [(costs[k], labels[k]) for k in range(K)]


def ref_energy(pr: Problem, labels) -> float:
    out = np.zeros(1, np.float64)
    labels = np.ascontiguousarray(labels, np.uint16)
    _check_ref(_ref().ref_energy_f32(pr.H, pr.W, pr.L, pr.conn, _ptr(pr.unary), _ptr(pr.V), pr.w_const,
                                     _ptr(pr.w_planes), _ptr(labels), _ptr(out)))
    return float(out[0])


def ref_gradient_check(H, W, L, conn, K, trwp, per_edge, seed):
    e = np.zeros(1, np.float64)
    comp = np.zeros(1, np.uint64)
    sk = np.zeros(1, np.uint64)
    _check_ref(_ref().ref_gradient_check(H, W, L, conn, K, int(trwp), int(per_edge), seed, _ptr(e), _ptr(comp),
                                         _ptr(sk)))
    return float(e[0]), int(comp[0]), int(sk[0])
