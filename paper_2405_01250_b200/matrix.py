"""Device-resident DiaQ matrices and their kernels (drop-in for diaqsim.matrix).

Reference: /root/reference/pkg/src/diaqsim/matrix.py.  Conventions are
unchanged: d = column - row, diagonal d holds n-|d| values, element (r, r+d)
sits at storage position k = r + min(d, 0), iteration is ascending in d, and
kernels take immutable inputs and return fresh matrices (matrix.py:1-14).

Storage (B200 layout): one device complex128 arena per matrix
(interleaved re/im: one 16-byte load per element) plus a host table of
ascending offsets and row-aligned element starts (diaq_layout).  Host
`Diagonal(index, re, im)` views are materialised lazily, so code written
against the reference (`a.get(d).re.tolist()`, `np.array_equal`) still works.

Hot-path operations run as sm_100a kernels through the C-ABI:
from_dense, to_dense, kron_identity, matmul (spgemm), spmv,
multiply_diagonals.  transpose/adjoint/add/scale/kron/nnz/sparsity and the
JSON wire form are O(stored) host metadata operations kept for API
completeness ("not on the hot path").
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .alloc import DEFAULT_ALIGNMENT
from .errors import ShapeError, UnsupportedFeatureError

# diagonals whose values all fall below this after a matmul are dropped
PRUNE_EPS = 1e-15

DTYPES = {"single": np.float32, "double": np.float64}


def diag_len(d: int, n_dim: int) -> int:
    """Length of diagonal d of an n_dim x n_dim matrix (matrix.py:31-35)."""
    if abs(d) > n_dim - 1:
        raise ValueError(f"diagonal {d} out of range for n_dim={n_dim}")
    return n_dim - abs(d)


@dataclass
class Diagonal:
    """One stored diagonal as host planar real/imaginary arrays."""

    index: int
    re: np.ndarray
    im: np.ndarray

    def __len__(self) -> int:
        return len(self.re)


class _Dev:
    """Device arena + host offset/start tables."""

    __slots__ = ("offs", "starts", "vals", "st")

    def __init__(self, offs: np.ndarray, starts: np.ndarray, vals):
        self.offs = offs
        self.starts = starts
        self.vals = vals
        self.st = None  # diaq_matrix_t, built once (the arena never moves)


class DiaqMatrix:
    """Square complex matrix stored as ascending full diagonals on the device.

    Absent diagonals are all-zero; stored zeros are kept.  The matrix is
    either device-authoritative (built by a kernel) or host-authoritative
    (after set_diag/drop); each side is materialised from the other on demand.
    """

    def __init__(self, n_dim: int, dtype=np.float64, align: int = DEFAULT_ALIGNMENT):
        if n_dim < 1:
            raise ShapeError(f"n_dim must be >= 1, got {n_dim}")
        self.n_dim = int(n_dim)
        self.dtype = np.dtype(dtype)
        self.align = align
        self._host: dict[int, Diagonal] | None = {}
        self._dev: _Dev | None = None

    # -- construction from a device arena -----------------------------------

    @classmethod
    def _from_device(cls, n_dim: int, offs, starts, vals, dtype=np.float64) -> "DiaqMatrix":
        out = cls(n_dim, dtype)
        out._host = None
        out._dev = _Dev(np.ascontiguousarray(offs, dtype=np.int64),
                        np.ascontiguousarray(starts, dtype=np.int64), vals)
        return out

    @classmethod
    def _empty_device(cls, n_dim: int, offs, dtype=np.float64) -> "DiaqMatrix":
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        starts, total = L.layout(n_dim, offs)
        vals = L.empty_c128(max(total, 1))
        return cls._from_device(n_dim, offs, starts, vals, dtype)

    # -- host <-> device -----------------------------------------------------

    def _device(self) -> _Dev:
        """Device representation (uploads host diagonals once if needed)."""
        if self._dev is None:
            offs = np.array(sorted(self._host), dtype=np.int64)
            starts, total = L.layout(self.n_dim, offs)
            buf = np.zeros(max(total, 1), dtype=np.complex128)
            for i, d in enumerate(offs.tolist()):
                dg = self._host[d]
                s = int(starts[i])
                buf[s:s + len(dg)].real = dg.re
                buf[s:s + len(dg)].imag = dg.im
            self._dev = _Dev(offs, starts, L.to_device_c128(buf))
        return self._dev

    def _hostmap(self) -> dict[int, Diagonal]:
        """Host representation (downloads the arena once if needed)."""
        if self._host is None:
            dv = self._dev
            arena = dv.vals.cpu().numpy() if len(dv.offs) else np.zeros(0, np.complex128)
            host = {}
            for i, d in enumerate(dv.offs.tolist()):
                s = int(dv.starts[i])
                seg = arena[s:s + self.n_dim - abs(d)]
                re = np.ascontiguousarray(seg.real, dtype=self.dtype)
                im = np.ascontiguousarray(seg.imag, dtype=self.dtype)
                re.flags.writeable = False  # snapshots of the device arena: edit via set_diag
                im.flags.writeable = False
                host[d] = Diagonal(d, re, im)
            self._host = host
        return self._host

    def _struct(self) -> L.Matrix:
        dv = self._device()
        if dv.st is None:
            dv.st = L.mat_struct(self.n_dim, dv.offs, dv.starts, dv.vals)
        return dv.st

    def device_arena(self):
        """(offsets, starts, torch complex128 arena) -- the device layout."""
        dv = self._device()
        return dv.offs, dv.starts, dv.vals

    # -- storage API (matrix.py:66-102) ----------------------------------------

    def set_diag(self, d: int, re, im=None) -> None:
        """Install diagonal d from value arrays (copied)."""
        want = diag_len(d, self.n_dim)
        re = np.array(re, dtype=self.dtype, copy=True).reshape(-1)
        im = np.zeros(want, dtype=self.dtype) if im is None else np.array(im, dtype=self.dtype,
                                                                           copy=True).reshape(-1)
        if len(re) != want or len(im) != want:
            raise ShapeError(f"diagonal {d} of n_dim={self.n_dim} needs {want} values")
        self._hostmap()[int(d)] = Diagonal(int(d), re, im)
        self._dev = None

    def get(self, d: int) -> Diagonal | None:
        if self._host is None and int(d) not in set(self._dev.offs.tolist()):
            return None
        return self._hostmap().get(int(d))

    def drop(self, d: int) -> None:
        self._hostmap().pop(int(d), None)
        self._dev = None

    def diag_indices(self) -> list[int]:
        if self._host is None:
            return self._dev.offs.tolist()
        return sorted(self._host)

    def diagonals(self):
        """Yield stored diagonals in ascending index order."""
        h = self._hostmap()
        for d in sorted(h):
            yield h[d]

    def diag_count(self) -> int:
        return len(self._dev.offs) if self._host is None else len(self._host)

    def copy(self) -> "DiaqMatrix":
        if self._host is None:
            dv = self._dev
            return DiaqMatrix._from_device(self.n_dim, dv.offs.copy(), dv.starts.copy(),
                                           dv.vals.clone(), self.dtype)
        out = DiaqMatrix(self.n_dim, self.dtype, self.align)
        for diag in self.diagonals():
            out.set_diag(diag.index, diag.re, diag.im)
        return out

    # -- convenience -----------------------------------------------------------

    def to_dense(self) -> np.ndarray:
        return to_dense(self)

    def __matmul__(self, other: "DiaqMatrix") -> "DiaqMatrix":
        return matmul(self, other)

    def __eq__(self, other) -> bool:
        if not isinstance(other, DiaqMatrix):
            return NotImplemented
        if self.n_dim != other.n_dim or self.diag_indices() != other.diag_indices():
            return False
        return all(
            np.array_equal(a.re, b.re) and np.array_equal(a.im, b.im)
            for a, b in zip(self.diagonals(), other.diagonals())
        )

    __hash__ = None

    def __repr__(self) -> str:
        return f"DiaqMatrix(n_dim={self.n_dim}, diagonals={self.diag_indices()})"


def identity(n_dim: int, dtype=np.float64) -> DiaqMatrix:
    out = DiaqMatrix(n_dim, dtype)
    out.set_diag(0, np.ones(n_dim, dtype=dtype))
    return out


# -- conversions (device kernels) ----------------------------------------------


def from_dense(m, eps: float = 0.0, dtype=np.float64) -> DiaqMatrix:
    """Keep every diagonal of `m` with an entry |re|+|im| > eps (matrix.py:135-153).

    `m` may be a host array or a CUDA tensor.  Pass 1 (device) flags the
    diagonals, the host lays out the kept set, pass 2 (device) gathers them.
    """
    t = L.torch()
    if isinstance(m, t.Tensor):
        if m.dim() != 2 or m.shape[0] != m.shape[1]:
            raise ShapeError(f"expected a square matrix, got shape {tuple(m.shape)}")
        n = int(m.shape[0])
    else:
        m = np.asarray(m)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ShapeError(f"expected a square matrix, got shape {m.shape}")
        n = int(m.shape[0])
        if np.dtype(dtype) == np.float32:
            # values are rounded to the storage precision first (matrix.py:149-150)
            m = m.real.astype(np.float32).astype(np.float64) + 1j * m.imag.astype(np.float32).astype(np.float64) \
                if np.iscomplexobj(m) else m.astype(np.float32).astype(np.float64)
    dense = L.to_device_c128(m.reshape(-1) if not isinstance(m, t.Tensor) else m.reshape(-1))
    keep = t.empty(2 * n - 1, dtype=t.uint8, device=dense.device)
    s = L.stream_handle()
    L.call("diaq_from_dense_scan", n, dense.data_ptr(), float(eps), keep.data_ptr(), s)
    flags = keep.cpu().numpy()
    offs = np.nonzero(flags)[0].astype(np.int64) - (n - 1)
    out = DiaqMatrix._empty_device(n, offs, dtype)
    if len(offs):
        st = out._struct()
        L.call("diaq_from_dense_fill", dense.data_ptr(), ctypes.byref(st), s)
    return out


def to_dense(a: DiaqMatrix) -> np.ndarray:
    """Scatter all stored diagonals into a dense complex array (matrix.py:156-167)."""
    t = L.torch()
    n = a.n_dim
    dense = t.zeros(n * n, dtype=t.complex128, device=L.device())
    if a.diag_count():
        st = a._struct()
        L.call("diaq_to_dense", ctypes.byref(st), dense.data_ptr(), L.stream_handle())
    return dense.cpu().numpy().reshape(n, n)


# -- kernels -----------------------------------------------------------------------


def _pair_range(d_a: int, d_b: int, n: int) -> tuple[int, int]:
    """Valid row range [lo, hi) for combining diagonals d_a of A and d_b of B."""
    d_c = d_a + d_b
    return max(0, -d_a, -d_c), min(n, n - d_a, n - d_c)


def _spgemm(a: DiaqMatrix, b: DiaqMatrix, prune_eps: float):
    """Run the device spgemm; return (candidate offsets, keep flags, C arena, starts)."""
    t = L.torch()
    n = a.n_dim
    da, db = a._device(), b._device()
    cap = max(1, len(da.offs) * len(db.offs))
    offc = np.zeros(cap, dtype=np.int64)
    nc = ctypes.c_int64(0)
    L.call("diaq_spgemm_plan", n, len(da.offs), da.offs.ctypes.data if len(da.offs) else None,
           len(db.offs), db.offs.ctypes.data if len(db.offs) else None, offc.ctypes.data,
           ctypes.addressof(nc))
    offc = offc[: nc.value].copy()
    starts, total = L.layout(n, offc)
    cvals = L.empty_c128(max(total, 1))
    if len(offc) == 0:
        return offc, np.zeros(0, np.uint8), cvals, starts
    keep = t.empty(len(offc), dtype=t.uint8, device=cvals.device)
    if len(offc) <= 128 and len(da.offs) * len(db.offs) <= 512:
        ws, ws_bytes = None, 0  # the plan travels in the kernel parameters
    else:
        ws_bytes = int(L.load().diaq_spgemm_workspace(len(da.offs), len(db.offs), len(offc)))
        ws = t.empty(ws_bytes, dtype=t.uint8, device=cvals.device)
    sa = L.mat_struct(n, da.offs, da.starts, da.vals)
    sb = L.mat_struct(n, db.offs, db.starts, db.vals)
    sc = L.mat_struct(n, offc, starts, cvals)
    L.call("diaq_spgemm", ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(sc), keep.data_ptr(),
           float(prune_eps), ws.data_ptr() if ws is not None else None, ws_bytes, L.stream_handle())
    return offc, keep.cpu().numpy(), cvals, starts


def matmul(a: DiaqMatrix, b: DiaqMatrix) -> DiaqMatrix:
    """Sparse product A @ B over diagonal pairs (matrix.py:218-250).

    Device two-pass spgemm: bitwise equal to the reference (each result
    diagonal accumulates its pairs in ascending d_a from zero), structure
    included; result diagonals entirely below PRUNE_EPS are dropped.
    """
    if a.n_dim != b.n_dim:
        raise ShapeError(
            f"not multiplyable: {a.n_dim}x{a.n_dim} by {b.n_dim}x{b.n_dim}"
        )
    dtype = np.result_type(a.dtype, b.dtype)
    if dtype != np.float64:
        raise UnsupportedFeatureError("device spgemm computes in double precision only")
    offc, keep, cvals, starts = _spgemm(a, b, PRUNE_EPS)
    kept = keep.astype(bool)
    return DiaqMatrix._from_device(a.n_dim, offc[kept], starts[kept], cvals, dtype)


def multiply_diagonals(diag_a: Diagonal, diag_b: Diagonal, n_dim: int):
    """Combine one diagonal of A with one of B (matrix.py:181-199).

    Returns (d_c, Diagonal) with the contribution to d_c = d_a + d_b, or
    None when the pair contributes nothing.
    """
    d_a, d_b = diag_a.index, diag_b.index
    d_c = d_a + d_b
    if abs(d_c) >= n_dim:
        return None
    lo, hi = _pair_range(d_a, d_b, n_dim)
    if lo >= hi:
        return None
    a = DiaqMatrix(n_dim, diag_a.re.dtype)
    a.set_diag(d_a, diag_a.re, diag_a.im)
    b = DiaqMatrix(n_dim, diag_b.re.dtype)
    b.set_diag(d_b, diag_b.re, diag_b.im)
    offc, _, cvals, starts = _spgemm(a, b, -1.0)
    c = DiaqMatrix._from_device(n_dim, offc, starts, cvals, diag_a.re.dtype)
    return d_c, c.get(d_c)


def _as_device_vector(x, n: int):
    """(device complex128 vector, kind) with kind in {"numpy", "cuda", "cpu_tensor"}."""
    t = L.torch()
    if isinstance(x, t.Tensor):
        if tuple(x.shape) != (n,):
            raise ShapeError(f"not multiplyable: {n}x{n} by vector of shape {tuple(x.shape)}")
        return L.to_device_c128(x), ("cuda" if x.device.type == "cuda" else "cpu_tensor")
    x = np.asarray(x)
    if x.shape != (n,):
        raise ShapeError(f"not multiplyable: {n}x{n} by vector of shape {x.shape}")
    return L.to_device_c128(x), "numpy"


HOST_PIPELINE_MIN = 1 << 21  # rows; above this host vectors take the pipelined path
HOST_CHUNK_ROWS = 1 << 22


def spmv(a: DiaqMatrix, x, out=None):
    """Sparse matrix-vector product A @ x (matrix.py:253-278).

    Bitwise equal to the reference.  A host numpy `x` returns a host
    complex128 array (reference behaviour); a CUDA tensor returns a CUDA
    tensor.  `out` (extension): a complex128 torch tensor, on the device or in
    (pinned) host memory, that receives y.  Large host vectors go through
    diaq_spmv_host, which overlaps the H2D of x, the kernel and the D2H of y
    chunk by chunk.
    """
    n = a.n_dim
    t = L.torch()
    if out is not None and (not isinstance(out, t.Tensor) or tuple(out.shape) != (n,)
                            or out.dtype != t.complex128):
        raise ShapeError(f"out must be a complex128 tensor of shape ({n},)")
    on_host = not (isinstance(x, t.Tensor) and x.device.type == "cuda")
    if on_host and n >= HOST_PIPELINE_MIN and (out is None or out.device.type == "cpu"):
        if isinstance(x, t.Tensor):
            if tuple(x.shape) != (n,):
                raise ShapeError(f"not multiplyable: {n}x{n} by vector of shape {tuple(x.shape)}")
            xh = x.contiguous() if x.dtype == t.complex128 else x.to(t.complex128).contiguous()
        else:
            xa = np.asarray(x)
            if xa.shape != (n,):
                raise ShapeError(f"not multiplyable: {n}x{n} by vector of shape {xa.shape}")
            xh = t.from_numpy(np.ascontiguousarray(xa, dtype=np.complex128))
        yh = out if out is not None else t.empty(n, dtype=t.complex128, pin_memory=True)
        xd = L.empty_c128(n)
        yd = L.empty_c128(n)
        st = a._struct()
        L.call("diaq_spmv_host", ctypes.byref(st), xh.data_ptr(), yh.data_ptr(), xd.data_ptr(), yd.data_ptr(),
               HOST_CHUNK_ROWS, L.stream_handle())
        if out is not None:
            return out
        return yh.numpy() if not isinstance(x, t.Tensor) else yh
    xd, kind = _as_device_vector(x, n)
    y = out if out is not None and out.device.type == "cuda" else L.empty_c128(n)
    st = a._struct()
    L.call("diaq_spmv", ctypes.byref(st), xd.data_ptr(), y.data_ptr(), L.stream_handle())
    if out is not None:
        if out is not y:
            out.copy_(y)
        return out
    if kind == "numpy":
        return y.cpu().numpy()
    return y if kind == "cuda" else y.cpu()


# -- metadata operations (host side; not on the hot path) ---------------------


def transpose(a: DiaqMatrix) -> DiaqMatrix:
    """Transpose: diagonal d moves to -d, value arrays unchanged (matrix.py:281-290)."""
    out = DiaqMatrix(a.n_dim, a.dtype, a.align)
    for diag in a.diagonals():
        out.set_diag(-diag.index, diag.re, diag.im)
    return out


def adjoint(a: DiaqMatrix) -> DiaqMatrix:
    """Conjugate transpose (matrix.py:293-298)."""
    out = DiaqMatrix(a.n_dim, a.dtype, a.align)
    for diag in a.diagonals():
        out.set_diag(-diag.index, diag.re, -diag.im)
    return out


def add(a: DiaqMatrix, b: DiaqMatrix) -> DiaqMatrix:
    """Sum over the union of stored diagonals (matrix.py:301-315)."""
    if a.n_dim != b.n_dim:
        raise ShapeError(f"shape mismatch: {a.n_dim} vs {b.n_dim}")
    dtype = np.result_type(a.dtype, b.dtype)
    out = DiaqMatrix(a.n_dim, dtype)
    for d in sorted(set(a.diag_indices()) | set(b.diag_indices())):
        length = diag_len(d, a.n_dim)
        re = np.zeros(length, dtype=dtype)
        im = np.zeros(length, dtype=dtype)
        for src in (a.get(d), b.get(d)):
            if src is not None:
                re += src.re
                im += src.im
        out.set_diag(d, re, im)
    return out


def scale(a: DiaqMatrix, s: complex) -> DiaqMatrix:
    """Multiply every stored value by the complex scalar s (matrix.py:318-323)."""
    sr, si = s.real, s.imag
    out = DiaqMatrix(a.n_dim, a.dtype, a.align)
    for diag in a.diagonals():
        out.set_diag(diag.index, sr * diag.re - si * diag.im, sr * diag.im + si * diag.re)
    return out


def kron(a: DiaqMatrix, b: DiaqMatrix) -> DiaqMatrix:
    """General Kronecker product A (x) B (matrix.py:329-355; test-level API).

    Source pair (d_a, d_b) lands on result diagonal d_a*n_b + d_b at rows
    r_a*n_b + r_b; distinct pairs feeding one result diagonal never overlap.
    """
    n_a, n_b = a.n_dim, b.n_dim
    n = n_a * n_b
    dtype = np.result_type(a.dtype, b.dtype)
    bufs: dict[int, tuple[np.ndarray, np.ndarray]] = {}
    for diag_a in a.diagonals():
        rows_a = np.arange(len(diag_a)) - min(diag_a.index, 0)
        for diag_b in b.diagonals():
            rows_b = np.arange(len(diag_b)) - min(diag_b.index, 0)
            d = diag_a.index * n_b + diag_b.index
            if d not in bufs:
                bufs[d] = (np.zeros(n - abs(d), dtype=dtype), np.zeros(n - abs(d), dtype=dtype))
            re, im = bufs[d]
            k = (rows_a[:, None] * n_b + rows_b[None, :] + min(d, 0)).ravel()
            re[k] = (np.outer(diag_a.re, diag_b.re) - np.outer(diag_a.im, diag_b.im)).ravel()
            im[k] = (np.outer(diag_a.re, diag_b.im) + np.outer(diag_a.im, diag_b.re)).ravel()
    out = DiaqMatrix(n, dtype)
    for d in sorted(bufs):
        out.set_diag(d, *bufs[d])
    return out


def kron_identity(left_dim: int, m: DiaqMatrix, right_dim: int) -> DiaqMatrix:
    """Materialise I_left (x) m (x) I_right on the device (matrix.py:358-387).

    Diagonal d of m becomes diagonal d*right_dim; every value repeats
    right_dim times inside each of the left_dim blocks and the gaps between
    blocks stay explicit zeros (nothing is pruned).
    """
    if left_dim < 1 or right_dim < 1:
        raise ShapeError("left_dim and right_dim must be >= 1")
    n = int(left_dim) * m.n_dim * int(right_dim)
    offs = np.array([d * int(right_dim) for d in m.diag_indices()], dtype=np.int64)
    out = DiaqMatrix._empty_device(n, offs, m.dtype)
    if len(offs):
        sm = m._struct()
        so = out._struct()
        L.call("diaq_kron_identity", int(left_dim), ctypes.byref(sm), int(right_dim),
               ctypes.byref(so), L.stream_handle())
    return out


# -- accounting --------------------------------------------------------------------


def nnz(a: DiaqMatrix, eps: float = 1e-15) -> int:
    """Stored entries with |re| + |im| > eps (matrix.py:393-400), counted on the device."""
    if eps < 0:
        raise ValueError("eps must be >= 0")
    from .memory import device_counts
    return device_counts(a, eps)[0]


def sparsity(a: DiaqMatrix, eps: float = 1e-15) -> float:
    return 1.0 - nnz(a, eps) / (a.n_dim * a.n_dim)


# -- serialization (wire form of the kernel protocol, cli.py:251-287) -------------


def to_json_dict(a: DiaqMatrix) -> dict:
    """Wire form: {"n": N, "diags": {"<d>": [[re, im], ...]}} (matrix.py:410-418)."""
    return {
        "n": a.n_dim,
        "diags": {
            str(diag.index): [[float(r), float(i)] for r, i in zip(diag.re, diag.im)]
            for diag in a.diagonals()
        },
    }


def from_json_dict(obj: dict, dtype=np.float64) -> DiaqMatrix:
    out = DiaqMatrix(int(obj["n"]), dtype)
    for key, pairs in obj.get("diags", {}).items():
        arr = np.asarray(pairs, dtype=np.float64).reshape(-1, 2)
        out.set_diag(int(key), arr[:, 0], arr[:, 1])
    return out


def to_json(a: DiaqMatrix) -> str:
    return json.dumps(to_json_dict(a))


def from_json(text: str, dtype=np.float64) -> DiaqMatrix:
    return from_json_dict(json.loads(text), dtype)
