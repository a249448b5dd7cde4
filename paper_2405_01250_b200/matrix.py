"""Device-resident DiaQ matrices and their kernels (drop-in for diaqsim.matrix).

Reference: /root/reference/pkg/src/diaqsim/matrix.py.  Conventions are
unchanged: d = column - row, diagonal d holds n-|d| values, element (r, r+d)
sits at storage position k = r + min(d, 0), iteration is ascending in d, and
kernels take immutable inputs and return fresh matrices (matrix.py:1-14).

Storage (B200 layout): one device complex128 arena per matrix
(interleaved re/im: one 16-byte load per element) plus its structure table
(ascending offsets, row-aligned element starts; diaq_layout).  The table may
live on the host, on the device, or both: a product computed with the
device plan (diaq_spgemm_dev) knows its pruned structure only on the device
until someone asks for it, so chains of products never wait for the host.
Host `Diagonal(index, re, im)` views are downloaded one diagonal at a time
(read-only snapshots), so code written against the reference
(`a.get(d).re.tolist()`, `np.array_equal`) still works.

Every operation runs on the device through the C-ABI: from_dense, to_dense,
kron_identity, kron, matmul (spgemm), spmv, add, scale, adjoint; transpose
is a zero-copy relabel of the arena (position k of diagonal d and of -d are
transposes, matrix.py:281-290).
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .alloc import DEFAULT_ALIGNMENT
from .errors import ShapeError

# diagonals whose values all fall below this after a matmul are dropped
PRUNE_EPS = 1e-15

DTYPES = {"single": np.float32, "double": np.float64}

# products planned on the device: at most this many (dA, dB) pairs, and a
# candidate arena of at most this many bytes (else the host plans exactly)
DEV_PLAN_PAIRS = 1024
DEV_PLAN_BYTES = 256 << 20


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
    """Device arena + its structure table (host arrays and/or device table)."""

    __slots__ = ("offs", "starts", "vals", "st", "st_ref", "dtab", "cap", "rec")

    def __init__(self, offs, starts, vals, dtab=None, cap=None):
        self.offs = offs          # host int64 offsets (None: structure only on the device)
        self.starts = starts      # host int64 element starts
        self.vals = vals          # torch complex128 arena
        self.st = None            # diaq_matrix_t, built once (the arena never moves)
        self.st_ref = None        # ctypes.byref(st), for the per-call fast paths
        self.rec = None           # diaq_dev_matrix_t fields (device table), built once
        self.dtab = dtab          # device int64 [nd, offs[cap], starts[cap]]
        self.cap = cap if cap is not None else (len(offs) if offs is not None else 0)


def _single(*mats) -> int:
    return int(all(m.dtype == np.float32 for m in mats))


class DiaqMatrix:
    """Square complex matrix stored as ascending full diagonals on the device.

    Absent diagonals are all-zero; stored zeros are kept.  The matrix is
    either host-authoritative (built with set_diag, the reference's way) or
    device-authoritative (built by a kernel); the other side is produced on
    demand.  `_version` counts edits, so caches keyed on a matrix see them.
    """

    def __init__(self, n_dim: int, dtype=np.float64, align: int = DEFAULT_ALIGNMENT):
        if n_dim < 1:
            raise ShapeError(f"n_dim must be >= 1, got {n_dim}")
        self.n_dim = int(n_dim)
        self.dtype = np.dtype(dtype)
        self.align = align
        self._host: dict[int, Diagonal] | None = {}
        self._dev: _Dev | None = None
        self._views: dict[int, Diagonal] = {}
        self._version = 0

    # -- construction from a device arena -----------------------------------

    @classmethod
    def _from_device(cls, n_dim: int, offs, starts, vals, dtype=np.float64, dtab=None, cap=None) -> "DiaqMatrix":
        out = cls.__new__(cls)  # (a kernel's output: no validation, cheap per product of a sweep)
        out.n_dim = int(n_dim)
        out.dtype = dtype if isinstance(dtype, np.dtype) else np.dtype(dtype)
        out.align = DEFAULT_ALIGNMENT
        out._host = None
        out._views = {}
        out._version = 0
        if offs is not None:
            offs = np.ascontiguousarray(offs, dtype=np.int64)
            starts = np.ascontiguousarray(starts, dtype=np.int64)
        out._dev = _Dev(offs, starts, vals, dtab, cap)
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
            for s, d in zip(starts.tolist(), offs.tolist()):
                dg = self._host[d]
                seg = buf[s:s + len(dg)]
                seg.real = dg.re
                seg.imag = dg.im
            self._dev = _Dev(offs, starts, L.to_device_c128(buf))
        return self._dev

    def _tables(self) -> tuple[np.ndarray, np.ndarray]:
        """Host structure table (reads a device-only table back: one sync)."""
        dv = self._device()
        if dv.offs is None:
            t = dv.dtab.cpu().numpy()
            nd = int(t[0])
            if nd < 0:
                raise L.DeviceError(f"device spgemm plan failed (code {-nd})")
            dv.offs = np.ascontiguousarray(t[1:1 + nd])
            dv.starts = np.ascontiguousarray(t[1 + dv.cap:1 + dv.cap + nd])
        return dv.offs, dv.starts

    def _dev_table(self):
        """(device int64 [nd, offs[cap], starts[cap]], cap): uploaded once for
        a host-known structure (pinned, non-blocking)."""
        dv = self._device()
        if dv.dtab is None:
            nd = len(dv.offs)
            host = np.concatenate([np.array([nd], dtype=np.int64), dv.offs, dv.starts])
            t = L.torch()
            dv.dtab = t.from_numpy(host).pin_memory().to(dv.vals.device, non_blocking=True)
            dv.cap = nd
        return dv.dtab, dv.cap

    def _cap(self) -> int:
        """Upper bound of the stored diagonal count known without a sync."""
        if self._host is not None:
            return len(self._host)
        dv = self._dev
        return len(dv.offs) if dv.offs is not None else dv.cap

    def _struct(self) -> L.Matrix:
        dv = self._device()
        if dv.st is None:
            offs, starts = self._tables()
            dv.st = L.mat_struct(self.n_dim, offs, starts, dv.vals)
        return dv.st

    def _struct_ref(self):
        st = self._struct()
        self._dev.st_ref = ctypes.byref(st)
        return self._dev.st_ref

    def _dev_struct(self) -> L.DevMatrix:
        dtab, cap = self._dev_table()
        base = dtab.data_ptr()
        return L.DevMatrix(self.n_dim, cap, base, base + 8, base + 8 * (1 + cap), self._dev.vals.data_ptr())

    def device_arena(self):
        """(offsets, starts, torch complex128 arena) -- the device layout."""
        offs, starts = self._tables()
        return offs, starts, self._dev.vals

    def _download(self, i: int, d: int, arena=None) -> Diagonal:
        """Host view of stored diagonal i (offset d): read-only snapshot."""
        dv = self._dev
        s = int(dv.starts[i])
        length = self.n_dim - abs(d)
        seg = arena[s:s + length] if arena is not None else dv.vals[s:s + length].cpu().numpy()
        re = np.array(seg.real, dtype=self.dtype)
        im = np.array(seg.imag, dtype=self.dtype)
        re.flags.writeable = False  # snapshots of the device arena: edit via set_diag
        im.flags.writeable = False
        return Diagonal(int(d), re, im)

    # -- storage API (matrix.py:66-102) ----------------------------------------

    def _edited(self) -> None:
        self._dev = None
        self._views = {}
        self._version += 1

    def _to_host(self) -> dict[int, Diagonal]:
        """Make the host side authoritative (one download of the arena)."""
        if self._host is None:
            offs, _ = self._tables()
            arena = self._dev.vals.cpu().numpy() if len(offs) else None
            self._host = {}
            for i, d in enumerate(offs.tolist()):
                dg = self._views.get(d) or self._download(i, d, arena)
                self._host[d] = Diagonal(d, np.array(dg.re), np.array(dg.im))
        return self._host

    def set_diag(self, d: int, re, im=None) -> None:
        """Install diagonal d from value arrays (copied)."""
        want = diag_len(d, self.n_dim)
        re = np.array(re, dtype=self.dtype, copy=True).reshape(-1)
        im = np.zeros(want, dtype=self.dtype) if im is None else np.array(im, dtype=self.dtype,
                                                                           copy=True).reshape(-1)
        if len(re) != want or len(im) != want:
            raise ShapeError(f"diagonal {d} of n_dim={self.n_dim} needs {want} values")
        host = self._to_host()
        host[int(d)] = Diagonal(int(d), re, im)
        self._edited()

    def get(self, d: int) -> Diagonal | None:
        d = int(d)
        if self._host is not None:
            return self._host.get(d)
        if d in self._views:
            return self._views[d]
        offs, _ = self._tables()
        i = int(np.searchsorted(offs, d))
        if i >= len(offs) or offs[i] != d:
            return None
        self._views[d] = self._download(i, d)
        return self._views[d]

    def drop(self, d: int) -> None:
        d = int(d)
        if self._host is not None:
            self._host.pop(d, None)
            self._edited()
            return
        offs, starts = self._tables()
        keep = offs != d
        if keep.all():
            return
        # structure-only edit: the arena stays, the table loses the diagonal
        vals = self._dev.vals
        self._dev = _Dev(offs[keep].copy(), starts[keep].copy(), vals)
        self._views.pop(d, None)
        self._version += 1

    def diag_indices(self) -> list[int]:
        if self._host is not None:
            return sorted(self._host)
        return self._tables()[0].tolist()

    def diagonals(self):
        """Yield stored diagonals in ascending index order."""
        if self._host is not None:
            for d in sorted(self._host):
                yield self._host[d]
            return
        offs, _ = self._tables()
        missing = [d for d in offs.tolist() if d not in self._views]
        arena = self._dev.vals.cpu().numpy() if len(missing) > 1 else None
        for i, d in enumerate(offs.tolist()):
            if d not in self._views:
                self._views[d] = self._download(i, d, arena)
            yield self._views[d]

    def diag_count(self) -> int:
        return len(self._host) if self._host is not None else len(self._tables()[0])

    def copy(self) -> "DiaqMatrix":
        if self._host is None:
            offs, starts = self._tables()
            return DiaqMatrix._from_device(self.n_dim, offs.copy(), starts.copy(), self._dev.vals.clone(), self.dtype)
        out = DiaqMatrix(self.n_dim, self.dtype, self.align)
        out._host = {d: Diagonal(d, dg.re.copy(), dg.im.copy()) for d, dg in self._host.items()}
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
        if self._host is None and other._host is None:  # both on the device: compare there
            t = L.torch()
            oa, sa = self._tables()
            _, sb = other._tables()
            va, vb = self._dev.vals, other._dev.vals
            for d, s1, s2 in zip(oa.tolist(), sa.tolist(), sb.tolist()):
                n = self.n_dim - abs(d)
                a, b = t.view_as_real(va[s1:s1 + n]), t.view_as_real(vb[s2:s2 + n])
                if not bool((a == b).all()):  # == semantics: -0 equals +0, NaN never equal
                    return False
            return True
        return all(np.array_equal(x.re, y.re) and np.array_equal(x.im, y.im)
                   for x, y in zip(self.diagonals(), other.diagonals()))

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


# -- spgemm ------------------------------------------------------------------------


def _pair_range(d_a: int, d_b: int, n: int) -> tuple[int, int]:
    """Valid row range [lo, hi) for combining diagonals d_a of A and d_b of B."""
    d_c = d_a + d_b
    return max(0, -d_a, -d_c), min(n, n - d_a, n - d_c)


def _dev_plan_capacity(n: int, pair_cap: int) -> tuple[int, int]:
    """(candidate slots, arena elements) bounding a device-planned product."""
    ncap = max(1, min(pair_cap, 2 * n - 1))
    return ncap, ncap * (n + 7) + 8


def _use_dev_plan(a: DiaqMatrix, b: DiaqMatrix) -> bool:
    pc = a._cap() * b._cap()
    if pc < 1 or pc > DEV_PLAN_PAIRS:
        return False
    return 16 * _dev_plan_capacity(a.n_dim, pc)[1] <= DEV_PLAN_BYTES


def _spgemm_host(a: DiaqMatrix, b: DiaqMatrix, prune_eps: float):
    """Host-planned product (exact layout): returns (candidate offsets,
    starts, C arena, device keep flags)."""
    t = L.torch()
    n = a.n_dim
    oa, _ = a._tables()
    ob, _ = b._tables()
    cap = max(1, len(oa) * len(ob))
    offc = np.zeros(cap, dtype=np.int64)
    nc = ctypes.c_int64(0)
    L.call("diaq_spgemm_plan", n, len(oa), oa.ctypes.data if len(oa) else None,
           len(ob), ob.ctypes.data if len(ob) else None, offc.ctypes.data, ctypes.addressof(nc))
    offc = offc[: nc.value].copy()
    starts, total = L.layout(n, offc)
    cvals = L.empty_c128(max(total, 1))
    keep = t.empty(max(1, len(offc)), dtype=t.uint8, device=cvals.device)
    if len(offc) == 0:
        return offc, starts, cvals, keep
    if len(offc) <= 128 and len(oa) * len(ob) <= 512:
        ws, ws_bytes = None, 0  # the plan travels in the kernel parameters
    else:
        ws_bytes = int(L.load().diaq_spgemm_workspace(len(oa), len(ob), len(offc)))
        ws = t.empty(ws_bytes, dtype=t.uint8, device=cvals.device)
    sc = L.mat_struct(n, offc, starts, cvals)
    L.call("diaq_spgemm", ctypes.byref(a._struct()), ctypes.byref(b._struct()), ctypes.byref(sc), keep.data_ptr(),
           float(prune_eps), _single(a, b), ws.data_ptr() if ws is not None else None, ws_bytes, L.stream_handle())
    return offc, starts, cvals, keep


def _matmul_host(a: DiaqMatrix, b: DiaqMatrix, dtype) -> DiaqMatrix:
    """Host plan + device multiply; the prune is compacted on the device
    (no read back of the keep flags)."""
    t = L.torch()
    offc, starts, cvals, keep = _spgemm_host(a, b, PRUNE_EPS)
    nc = len(offc)
    if nc == 0:
        return DiaqMatrix._from_device(a.n_dim, offc, starts, cvals, dtype)
    cand = t.from_numpy(np.concatenate([offc, starts])).pin_memory().to(cvals.device, non_blocking=True)
    dtab = t.empty(1 + 2 * nc, dtype=t.int64, device=cvals.device)
    base = dtab.data_ptr()
    L.call("diaq_spgemm_compact", nc, cand.data_ptr(), keep.data_ptr(), base, base + 8, base + 8 * (1 + nc),
           L.stream_handle())
    # (cand is freed stream-ordered: its memory is reused only after the compaction ran)
    return DiaqMatrix._from_device(a.n_dim, None, None, cvals, dtype, dtab=dtab, cap=nc)


_WS: dict = {}


def _workspace(nbytes: int, dev):
    """Scratch for the device plan, reused across calls (stream-ordered: a
    later product on the same stream reuses it only after the earlier one
    consumed it)."""
    t = L.torch()
    key = (dev.index, L.stream_handle())
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = t.empty(max(nbytes, 1 << 16), dtype=t.uint8, device=dev)
        _WS[key] = ws
    return ws


# diaq_dev_matrix_t / diaq_dev_result_t as numpy records: a sweep's tables
# are filled column-wise (no per-product ctypes objects)
_DEVMAT = np.dtype([("n", "<i8"), ("nd_cap", "<i8"), ("nd", "<u8"), ("offs", "<u8"), ("starts", "<u8"),
                    ("vals", "<u8")])
_DEVRES = np.dtype([("nd", "<u8"), ("offs", "<u8"), ("starts", "<u8"), ("vals", "<u8"), ("capacity", "<i8"),
                    ("nd_cap", "<i8")])


def _dev_record(m: DiaqMatrix):
    """(n, cap, nd*, offs*, starts*, vals*) of m's device table, cached on m."""
    dv = m._dev
    if dv is not None and dv.rec is not None:
        return dv.rec
    dtab, cap = m._dev_table()
    base = dtab.data_ptr()
    m._dev.rec = (m.n_dim, cap, base, base + 8, base + 8 * (1 + cap), m._dev.vals.data_ptr())
    return m._dev.rec


def _dev_products(pairs, idx, out) -> None:
    """Device-planned products of `pairs` (all pass _use_dev_plan) into
    out[idx[j]]: one arena and one structure-table block for the sweep,
    carved into per-product views with one split each."""
    t = L.torch()
    count = len(pairs)
    pair_cap = max(a._cap() * b._cap() for a, b in pairs)
    n0 = pairs[0][0].n_dim
    same_n = all(a.n_dim == n0 for a, _ in pairs)
    caps = [_dev_plan_capacity(n0, pair_cap)] * count if same_n else \
        [_dev_plan_capacity(a.n_dim, pair_cap) for a, _ in pairs]
    sizes = [(c[1] + 31) & ~31 for c in caps]  # 512-byte aligned result arenas
    ncap_max = max(c[0] for c in caps)
    dev = L.device()
    arena = L.empty_c128(sum(sizes))
    row = 1 + 2 * ncap_max
    dtabs = t.empty((count, row), dtype=t.int64, device=dev)
    A = np.empty(count, dtype=_DEVMAT)
    B = np.empty(count, dtype=_DEVMAT)
    C = np.empty(count, dtype=_DEVRES)
    A[:] = [_dev_record(a) for a, _ in pairs]
    B[:] = [_dev_record(b) for _, b in pairs]
    tb = dtabs.data_ptr() + 8 * row * np.arange(count, dtype=np.uint64)
    C["nd"] = tb
    C["offs"] = tb + 8
    C["starts"] = tb + 8 * (1 + ncap_max)
    C["vals"] = arena.data_ptr() + 16 * np.concatenate([[0], np.cumsum(sizes[:-1])]).astype(np.uint64)
    C["capacity"] = [c[1] for c in caps]
    C["nd_cap"] = ncap_max
    singles = [_single(a, b) for a, b in pairs]
    ws_bytes = int(L.load().diaq_spgemm_dev_workspace(count, pair_cap))
    ws = _workspace(ws_bytes, dev)
    if all(singles) or not any(singles):
        L.call("diaq_spgemm_dev", count, A.ctypes.data, B.ctypes.data, C.ctypes.data, float(PRUNE_EPS),
               int(singles[0]), pair_cap, ws.data_ptr(), ws_bytes, L.stream_handle())
    else:  # mixed precisions in one sweep: one call per product
        for j in range(count):
            L.call("diaq_spgemm_dev", 1, A[j:].ctypes.data, B[j:].ctypes.data, C[j:].ctypes.data, float(PRUNE_EPS),
                   singles[j], pair_cap, ws.data_ptr(), ws_bytes, L.stream_handle())
    views = arena.split(sizes)
    rows = dtabs.unbind(0)
    for j, (a, b) in enumerate(pairs):
        out[idx[j]] = DiaqMatrix._from_device(a.n_dim, None, None, views[j], np.result_type(a.dtype, b.dtype),
                                              dtab=rows[j], cap=ncap_max)


def matmul_batch(pairs) -> list[DiaqMatrix]:
    """Products of many (A, B) pairs (a sweep, config 2) in one native call:
    the structure of every product is planned on the device (offset union,
    count and scan), multiplied and pruned in one launch of each kernel per
    64 products -- no host round trip.  Each result equals matmul(A, B)."""
    t = L.torch()
    pairs = list(pairs)
    if not pairs:
        return []
    out: list[DiaqMatrix | None] = [None] * len(pairs)
    dev_idx = []
    for i, (a, b) in enumerate(pairs):
        if a.n_dim != b.n_dim:
            raise ShapeError(f"not multiplyable: {a.n_dim}x{a.n_dim} by {b.n_dim}x{b.n_dim}")
        if _use_dev_plan(a, b):
            dev_idx.append(i)
        else:
            out[i] = matmul(a, b)
    if dev_idx:
        _dev_products([pairs[i] for i in dev_idx], dev_idx, out)
    return out


def matmul(a: DiaqMatrix, b: DiaqMatrix) -> DiaqMatrix:
    """Sparse product A @ B over diagonal pairs (matrix.py:218-250).

    Bitwise equal to the reference (each result diagonal accumulates its
    pairs in ascending d_a from zero, in the result precision), structure
    included; result diagonals entirely below PRUNE_EPS are dropped.  Small
    structures are planned on the device (north-star pass 1: offset union,
    count and scan), larger ones on the host; either way the prune is
    compacted on the device and nothing is read back.
    """
    if a.n_dim != b.n_dim:
        raise ShapeError(
            f"not multiplyable: {a.n_dim}x{a.n_dim} by {b.n_dim}x{b.n_dim}"
        )
    if a._cap() == 0 or b._cap() == 0:
        return DiaqMatrix(a.n_dim, np.result_type(a.dtype, b.dtype))
    if _use_dev_plan(a, b):
        return matmul_batch([(a, b)])[0]
    return _matmul_host(a, b, np.result_type(a.dtype, b.dtype))


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
    offc, starts, cvals, _ = _spgemm_host(a, b, -1.0)  # no prune: the partial diagonal as is
    c = DiaqMatrix._from_device(n_dim, offc, starts, cvals, diag_a.re.dtype)
    return d_c, c.get(d_c)


# -- spmv ----------------------------------------------------------------------------


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


def _overlaps(a, b) -> bool:
    """Do two tensors share any byte of storage?"""
    if a.device != b.device:
        return False
    a0, b0 = a.data_ptr(), b.data_ptr()
    return a0 < b0 + b.numel() * b.element_size() and b0 < a0 + a.numel() * a.element_size()


HOST_PIPELINE_MIN = 1 << 21  # rows; above this host vectors take the pipelined path
HOST_CHUNK_ROWS = 1 << 22


def spmv(a: DiaqMatrix, x, out=None):
    """Sparse matrix-vector product A @ x (matrix.py:253-278).

    Bitwise equal to the reference.  A host numpy `x` returns a host
    complex128 array (reference behaviour); a CUDA tensor returns a CUDA
    tensor.  `out` (extension): a complex128 torch tensor, on the device or in
    (pinned) host memory, that receives y; it must not overlap x (the
    kernel stages windows of x while other rows of y are written).  Large
    host vectors go through diaq_spmv_host, which overlaps the H2D of x, the
    kernel and the D2H of y chunk by chunk.
    """
    n = a.n_dim
    t = L.torch()
    if out is None and type(x) is t.Tensor and x.is_cuda and x.dtype is t.complex128 and x.shape == (n,) \
            and x.is_contiguous():
        # fast path (device vector in, device vector out): one allocation,
        # one C call with the matrix's cached descriptor
        dv = a._dev
        ref = dv.st_ref if dv is not None and dv.st_ref is not None else a._struct_ref()
        y = t.empty_like(x)
        rc = L._lib.diaq_spmv(ref, x.data_ptr(), y.data_ptr(), L.stream_handle())
        if rc:
            L.check(rc, "diaq_spmv")
        return y
    if out is not None and (not isinstance(out, t.Tensor) or tuple(out.shape) != (n,)
                            or out.dtype != t.complex128):
        raise ShapeError(f"out must be a complex128 tensor of shape ({n},)")
    if out is not None and isinstance(x, t.Tensor) and _overlaps(out, x):
        raise ValueError("spmv: out must not share storage with x")
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


# -- matrix algebra (device kernels, ops.cu) --------------------------------------


def transpose(a: DiaqMatrix) -> DiaqMatrix:
    """Transpose: diagonal d becomes -d over the SAME arena (matrix.py:281-290:
    position k of diagonal d and of -d are transposes) -- no data moves."""
    if a.diag_count() == 0:
        return DiaqMatrix(a.n_dim, a.dtype, a.align)
    offs, starts = a._tables()
    out = DiaqMatrix._from_device(a.n_dim, -offs[::-1], starts[::-1], a._dev.vals, a.dtype)
    out.align = a.align
    return out


def _arena_map(a: DiaqMatrix, op: int, s: complex = 0j) -> DiaqMatrix:
    offs, starts = a._tables()
    src = a._dev.vals
    dst = L.empty_c128(src.numel())
    L.call("diaq_arena_map", int(src.numel()), src.data_ptr(), dst.data_ptr(), int(op), float(s.real), float(s.imag),
           _single(a), L.stream_handle())
    return DiaqMatrix._from_device(a.n_dim, offs.copy(), starts.copy(), dst, a.dtype)


def adjoint(a: DiaqMatrix) -> DiaqMatrix:
    """Conjugate transpose (matrix.py:293-298): a conj pass over the arena,
    then the transpose relabel."""
    if a.diag_count() == 0:
        return DiaqMatrix(a.n_dim, a.dtype, a.align)
    return transpose(_arena_map(a, 0))


def scale(a: DiaqMatrix, s: complex) -> DiaqMatrix:
    """Every stored value times s: (sr*re - si*im, sr*im + si*re) in a's
    precision (matrix.py:318-323)."""
    if a.diag_count() == 0:
        return DiaqMatrix(a.n_dim, a.dtype, a.align)
    return _arena_map(a, 1, complex(s))


def add(a: DiaqMatrix, b: DiaqMatrix) -> DiaqMatrix:
    """Sum over the union of stored diagonals (matrix.py:301-315)."""
    if a.n_dim != b.n_dim:
        raise ShapeError(f"shape mismatch: {a.n_dim} vs {b.n_dim}")
    dtype = np.result_type(a.dtype, b.dtype)
    union = np.union1d(np.asarray(a.diag_indices(), dtype=np.int64), np.asarray(b.diag_indices(), dtype=np.int64))
    out = DiaqMatrix._empty_device(a.n_dim, union, dtype)
    if len(union):
        L.call("diaq_add", ctypes.byref(a._struct()), ctypes.byref(b._struct()), ctypes.byref(out._struct()),
               int(dtype == np.float32), L.stream_handle())
    return out


def kron(a: DiaqMatrix, b: DiaqMatrix) -> DiaqMatrix:
    """General Kronecker product A (x) B (matrix.py:329-355; test-level API):
    result diagonal d = d_a*n_b + d_b; each output element finds its unique
    source pair from its row and column on the device."""
    t = L.torch()
    nb = b.n_dim
    n = a.n_dim * nb
    dtype = np.result_type(a.dtype, b.dtype)
    oa, sa = a._tables()
    ob, sb = b._tables()
    offs = np.unique((oa[:, None] * nb + ob[None, :]).reshape(-1)) if len(oa) and len(ob) else np.zeros(0, np.int64)
    out = DiaqMatrix._empty_device(n, offs, dtype)
    if len(offs):
        tabs = t.from_numpy(np.concatenate([oa, sa, ob, sb]).astype(np.int64)).to(L.device())
        L.call("diaq_kron", ctypes.byref(a._struct()), ctypes.byref(b._struct()), tabs.data_ptr(),
               ctypes.byref(out._struct()), int(dtype == np.float32), L.stream_handle())
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
#
# {"n": N, "diags": {"<d>": [[re, im], ...]}} (reference matrix.py:410-434).
# Values travel as Python floats of the stored precision.


def to_json_dict(a: DiaqMatrix) -> dict:
    diags = {}
    for dg in a.diagonals():
        pairs = np.empty((len(dg), 2), dtype=np.float64)
        pairs[:, 0] = dg.re
        pairs[:, 1] = dg.im
        diags[str(dg.index)] = pairs.tolist()
    return {"n": a.n_dim, "diags": diags}


def from_json_dict(obj: dict, dtype=np.float64) -> DiaqMatrix:
    """Build the matrix in one piece: all wire diagonals parsed, then one
    host table (uploaded on first device use)."""
    n = int(obj["n"])
    out = DiaqMatrix(n, dtype)
    table = {}
    for key, pairs in obj.get("diags", {}).items():
        d = int(key)
        arr = np.asarray(pairs, dtype=np.float64).reshape(-1, 2)
        if len(arr) != diag_len(d, n):
            raise ShapeError(f"diagonal {d} of n_dim={n} needs {diag_len(d, n)} values")
        table[d] = Diagonal(d, np.ascontiguousarray(arr[:, 0], dtype=dtype), np.ascontiguousarray(arr[:, 1], dtype=dtype))
    out._host = table
    return out


def to_json(a: DiaqMatrix) -> str:
    return json.dumps(to_json_dict(a))


def from_json(text: str, dtype=np.float64) -> DiaqMatrix:
    return from_json_dict(json.loads(text), dtype)
