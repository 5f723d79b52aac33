"""Device sparse linear algebra for the stage-coupled solve.

Drop-in for implicitrk.sparsela (/root/reference/pkg/src/implicitrk/sparsela.py):
``SparseMatrix``, ``spmv``, ``dirichlet_constrain``, ``factorize_block`` /
``BlockFactorization``, ``KroneckerStageOperator``, ``KrylovSettings``,
``fgmres``, ``FgmresResult``, ``mm_read`` / ``mm_write`` and the exception
classes keep the reference's names, arguments and error behaviour; every
arithmetic operation runs in libirk's sm_100a kernels on float64 device data.

Differences by design (north_star):
* stage vectors are stage-INTERLEAVED (row r, stage i at r*s+i) on the device;
  the public ``apply``/``fgmres`` entry points accept and return the
  reference's stage-major vectors and permute at the boundary;
* ``factorize_block`` does not factorise: the block alpha*M + dt*K (with the
  reference's identity rows/columns on Dirichlet dofs) is stored on device
  and solved by Jacobi-preconditioned CG to ``rtol`` (default 1e-12, i.e. to
  round-off on well-conditioned blocks);
* ``fgmres`` orthogonalises with classical Gram-Schmidt in one fused pass
  (optional second pass, ``KrylovSettings.reorth``) instead of MGS.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import ctypes as C
import gc
import itertools
import os
from collections import OrderedDict

import numpy as np

from . import _lib
from ._lib import call, ctx, hptr, ptr


class FactorizationError(ArithmeticError):
    """A stage block was structurally or numerically singular (sparsela.py:20-21)."""


class NonConvergenceError(RuntimeError):
    """An iteration cap was reached; carries the residual history (sparsela.py:24-29)."""

    def __init__(self, message, residuals):
        super().__init__(message)
        self.residuals = residuals


class Splitting(Enum):
    """Kronecker factorisation of the stage system (sparsela.py:32-40)."""

    AI = "ai"
    IA = "ia"


# --------------------------------------------------------------- devices


def _torch():
    import torch

    return torch


def device():
    torch = _torch()
    return torch.device("cuda", _lib.device_index())


def dev_empty(n, dtype=None):
    torch = _torch()
    return torch.empty(int(n), dtype=dtype or torch.float64, device=device())


def dev_zeros(n, dtype=None):
    torch = _torch()
    return torch.zeros(int(n), dtype=dtype or torch.float64, device=device())


def to_dev(x, dtype=None):
    """numpy / torch / sequence -> contiguous float64 (or dtype) CUDA tensor."""
    torch = _torch()
    dt = dtype or torch.float64
    if isinstance(x, torch.Tensor):
        if x.device.type == "cuda" and x.dtype == dt and x.is_contiguous():
            return x
        if x.device.type == "cpu" and x.is_pinned() and x.dtype == dt and x.is_contiguous():
            # direct DMA from the caller's pinned buffer; synchronised so the
            # caller may reuse the buffer as soon as this returns
            out = x.to(device=device(), non_blocking=True)
            torch.cuda.current_stream(out.device).synchronize()
            return out
        return x.to(device=device(), dtype=dt).contiguous()
    np_dt = np.float64 if dt == torch.float64 else np.int64 if dt == torch.int64 else None
    arr = np.ascontiguousarray(np.asarray(x, dtype=np_dt))
    t = torch.from_numpy(arr)
    if arr.nbytes >= (1 << 20) and t.is_pinned():
        # numpy over pinned memory (e.g. an array step() returned): direct DMA
        out = t.to(device(), non_blocking=True)
        torch.cuda.current_stream(out.device).synchronize()
        return out
    return _STAGER.upload(t)


class _PinnedStager:
    """Host->device uploads through a ring of persistent pinned buffers: the
    copy is asynchronous (the host does not wait for the stream, unlike a
    pageable copy), and no pinned memory is allocated per call (a fresh
    cudaHostAlloc costs milliseconds).  A slot is reused once the event
    recorded after its last copy has completed."""

    SLOTS = 4

    def __init__(self):
        self._buf = [None] * self.SLOTS
        self._ev = [None] * self.SLOTS
        self._next = 0

    def upload(self, t):
        torch = _torch()
        nbytes = t.numel() * t.element_size()
        if nbytes == 0:
            return t.to(device())
        i = self._next
        self._next = (i + 1) % self.SLOTS
        ev = self._ev[i]
        if ev is not None:
            ev.synchronize()  # normally long complete
        buf = self._buf[i]
        if buf is None or buf.numel() < nbytes:
            buf = self._buf[i] = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8,
                                             pin_memory=True)
        host = buf[:nbytes].view(t.dtype).view(t.shape)
        # single-threaded numpy copy into the pinned slot (torch's CPU copy_
        # fans out to the intra-op thread pool: milliseconds on a busy host)
        np.copyto(host.numpy(), t.numpy())
        out = host.to(device(), non_blocking=True)
        ev = self._ev[i] = self._ev[i] or torch.cuda.Event()
        ev.record()
        return out


_STAGER = _PinnedStager()


def is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_host(t) -> np.ndarray:
    """Device tensor -> fresh numpy array.  Large device reads land in pinned
    memory (torch's caching host allocator recycles the block once the array
    is dropped): a direct DMA instead of the driver's pageable bounce."""
    t = t.detach()
    if t.device.type == "cuda" and t.numel() * t.element_size() >= (1 << 20):
        out = _torch().empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t)
        return out.numpy()
    return t.cpu().numpy()


def _like_input(dev_result, like):
    """Return numpy for numpy-ish input, a torch CUDA tensor for torch input."""
    if is_torch(like):
        return dev_result
    return to_host(dev_result)


# ------------------------------------------------------------ device matrix


_SERIAL = itertools.count(1)  # identities of device objects in graph keys


class DeviceMatrix:
    """Owner of one libirk irk_mat (CSR + SELL-32, float64 values)."""

    __slots__ = ("handle", "nrows", "ncols", "nnz", "_ccache", "serial", "__weakref__")

    def __init__(self, handle: C.c_void_p):
        self.handle = handle
        self.serial = next(_SERIAL)  # graph-key identity (handles are reused addresses)
        self._ccache = {}
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        call("irk_mat_info", handle, C.byref(r), C.byref(c), C.byref(z))
        self.nrows, self.ncols, self.nnz = r.value, c.value, z.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().irk_mat_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None

    @classmethod
    def from_csr(cls, nrows, ncols, rowptr, col, val):
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int64)
        val = np.ascontiguousarray(val, dtype=np.float64)
        h = C.c_void_p()
        call("irk_mat_from_csr", ctx(), int(nrows), int(ncols), int(len(val)), hptr(rowptr),
             hptr(col), hptr(val), C.byref(h))
        return cls(h)

    def same_pattern(self, other: "DeviceMatrix") -> bool:
        return bool(_lib.load().irk_mat_same_pattern(self.handle, other.handle))

    def union(self, other):
        a, b = C.c_void_p(), C.c_void_p()
        call("irk_mat_union", ctx(), self.handle, other.handle, C.byref(a), C.byref(b))
        return DeviceMatrix(a), DeviceMatrix(b)

    def on_pattern(self, template: "DeviceMatrix") -> "DeviceMatrix":
        h = C.c_void_p()
        call("irk_mat_on_pattern", ctx(), self.handle, template.handle, C.byref(h))
        return DeviceMatrix(h)

    def combine(self, alpha, other, beta) -> "DeviceMatrix":
        h = C.c_void_p()
        call("irk_mat_combine", ctx(), float(alpha), self.handle, float(beta), other.handle,
             C.byref(h))
        return DeviceMatrix(h)

    def constrain(self, mask, diag_value=1.0) -> "DeviceMatrix":
        h = C.c_void_p()
        call("irk_mat_constrain", ctx(), self.handle, ptr(mask), float(diag_value), C.byref(h))
        return DeviceMatrix(h)

    def eliminated(self, mask) -> "DeviceMatrix":
        """Copy with the flagged rows and columns zeroed (cached per mask):
        the form every masked kernel expects (flagged rows are identity rows
        in the kernels themselves)."""
        if mask is None:
            return self
        key = (mask.data_ptr(), mask.numel())
        hit = self._ccache.get(key)
        if hit is None or hit[0] is not mask:
            hit = self._ccache[key] = (mask, self.constrain(mask, 0.0))
        return hit[1]

    def diagonal(self):
        out = dev_empty(self.nrows)
        call("irk_mat_diagonal", ctx(), self.handle, ptr(out))
        return out

    def rowsum(self):
        out = dev_empty(self.nrows)
        call("irk_mat_rowsum", ctx(), self.handle, ptr(out))
        return out

    def spmv(self, x, y, k=1):
        call("irk_spmv", ctx(), self.handle, int(k), ptr(x), ptr(y))
        return y

    def download(self):
        rp = np.empty(self.nrows + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int64)
        va = np.empty(self.nnz, dtype=np.float64)
        call("irk_mat_download", ctx(), self.handle, hptr(rp), hptr(ci), hptr(va))
        return rp, ci, va


def shared_pattern(mats):
    """Re-express device matrices on one pattern object (union of patterns)."""
    mats = list(mats)
    first = mats[0]
    if all(first.same_pattern(x) for x in mats[1:]):
        return mats
    acc = first
    for x in mats[1:]:
        if not acc.same_pattern(x):
            acc, _ = acc.union(x)
    return [x if x.same_pattern(acc) else x.on_pattern(acc) for x in mats]


# ------------------------------------------------------------ SparseMatrix


class SparseMatrix:
    """Immutable CSR matrix (sparsela.py:43-115) backed by a device copy.

    Host arrays (int64 indices, float64 values, read-only) are materialised
    on first access when the matrix was produced on the device (assembly,
    combination); device storage is created on first use when the matrix was
    built from host arrays.
    """

    def __init__(self, nrows, ncols, row_offsets, col_indices, values):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self._ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self._ci = np.ascontiguousarray(col_indices, dtype=np.int64)
        self._va = np.ascontiguousarray(values, dtype=np.float64)
        self._validate(self._ro, self._ci, self._va)
        for a in (self._ro, self._ci, self._va):
            a.setflags(write=False)
        self._nnz = len(self._va)
        self._dev = None
        self._csr = None
        self._pattern_cache = {}

    # -- construction -------------------------------------------------
    def _validate(self, ro, ci, va):
        if ro.shape != (self.nrows + 1,):
            raise ValueError("row_offsets must have length nrows + 1")
        if ro[0] != 0 or ro[-1] != len(va) or len(ci) != len(va):
            raise ValueError("row_offsets endpoints inconsistent with nnz")
        lens = np.diff(ro)
        if np.any(lens < 0):
            raise ValueError("row_offsets must be nondecreasing")
        if len(ci) and (ci.min() < 0 or ci.max() >= self.ncols):
            raise ValueError("column index out of range")
        if len(ci) > 1:
            step = np.diff(ci)
            same_row = np.repeat(np.arange(self.nrows), lens)
            inside = same_row[1:] == same_row[:-1]
            if np.any(step[inside] <= 0):
                raise ValueError("col_indices must be strictly increasing per row")

    @classmethod
    def _from_device(cls, dm: DeviceMatrix) -> "SparseMatrix":
        obj = cls.__new__(cls)
        obj.nrows, obj.ncols, obj._nnz = dm.nrows, dm.ncols, dm.nnz
        obj._ro = obj._ci = obj._va = None
        obj._dev = dm
        obj._csr = None
        obj._pattern_cache = {}
        return obj

    @classmethod
    def from_scipy(cls, mat) -> "SparseMatrix":
        import scipy.sparse as sp

        m = sp.csr_matrix(mat, copy=True)
        m.sum_duplicates()
        m.sort_indices()
        return cls(m.shape[0], m.shape[1], m.indptr, m.indices, m.data)

    @classmethod
    def from_dense(cls, arr) -> "SparseMatrix":
        import scipy.sparse as sp

        return cls.from_scipy(sp.csr_matrix(np.asarray(arr, dtype=np.float64)))

    @classmethod
    def identity(cls, n) -> "SparseMatrix":
        n = int(n)
        return cls(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    # -- host view -------------------------------------------------------
    def _host(self):
        if self._ro is None:
            ro, ci, va = self._dev.download()
            for a in (ro, ci, va):
                a.setflags(write=False)
            self._ro, self._ci, self._va = ro, ci, va

    @property
    def row_offsets(self):
        self._host()
        return self._ro

    @property
    def col_indices(self):
        self._host()
        return self._ci

    @property
    def values(self):
        self._host()
        return self._va

    def to_scipy(self):
        import scipy.sparse as sp

        if self._csr is None:
            self._host()
            self._csr = sp.csr_matrix((self._va, self._ci, self._ro), shape=(self.nrows, self.ncols))
        return self._csr

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @property
    def nnz(self):
        return self._nnz

    def __repr__(self):
        return f"SparseMatrix({self.nrows}x{self.ncols}, nnz={self.nnz})"

    # -- device view -------------------------------------------------------
    def device(self) -> DeviceMatrix:
        if self._dev is None:
            self._dev = DeviceMatrix.from_csr(self.nrows, self.ncols, self._ro, self._ci, self._va)
        return self._dev

    def _dev_op(self):
        return _SpmvOp(self)


def spmv(A: SparseMatrix, x):
    """y = A x (sparsela.py:118-123) on the device; numpy in -> numpy out."""
    n = x.shape[0] if hasattr(x, "shape") else len(x)
    if (len(getattr(x, "shape", (n,))) != 1) or n != A.ncols:
        raise ValueError(f"spmv: x has shape {tuple(getattr(x, 'shape', (n,)))}, expected ({A.ncols},)")
    xd = to_dev(x)
    y = dev_empty(A.nrows)
    A.device().spmv(xd, y)
    return _like_input(y, x)


_MASKS: dict = {}


def dof_mask(m: int, dofs):
    """uint8 device mask with ones at ``dofs`` (read-only; cached by content,
    so every constrained operator of a problem shares one mask object and
    the per-mask caches of eliminated matrices keep hitting -- a fresh mask
    per step re-created, and freed with a device sync, both eliminated
    stage matrices every step)."""
    torch = _torch()
    d = np.ascontiguousarray(np.asarray(dofs, dtype=np.int64))
    key = (int(m), d.size, hash(d.tobytes()), _lib.device_index())
    hit = _MASKS.get(key)
    if hit is not None and np.array_equal(hit[0], d):
        return hit[1]
    idx = to_dev(d, dtype=torch.int64)
    mask = torch.empty(int(m), dtype=torch.uint8, device=device())
    call("irk_bc_mask", ctx(), int(m), int(idx.numel()), ptr(idx), ptr(mask))
    if len(_MASKS) >= 64:
        _MASKS.pop(next(iter(_MASKS)))
    _MASKS[key] = (d.copy(), mask)
    return mask


def dirichlet_constrain(A: SparseMatrix, dofs, diag_value: float = 1.0) -> SparseMatrix:
    """Identity rows/columns on ``dofs`` (sparsela.py:126-146).

    The result keeps A's pattern (zeroed entries stay stored); its values and
    dense form equal the reference's.
    """
    dofs = np.asarray(dofs, dtype=np.int64)
    if len(dofs) == 0:
        return A
    if dofs.min() < 0 or dofs.max() >= A.nrows:
        raise ValueError("constrained dof index out of range")
    if A.nrows != A.ncols:
        raise ValueError("dirichlet_constrain needs a square matrix")
    mask = dof_mask(A.nrows, dofs)
    try:
        dm = A.device().constrain(mask, diag_value)
    except ValueError:
        # constrained rows without a stored diagonal: add it via a union
        eye = SparseMatrix.identity(A.nrows).device()
        a2, e2 = A.device().union(eye)
        dm = a2.constrain(mask, diag_value)
    return SparseMatrix._from_device(dm)


# ---------------------------------------------------- device operator layer


class _DevOp:
    """Device linear operator: ``dev_apply(x, out)`` on length-n CUDA tensors.

    ``layout`` is (m, s) when the operator works on stage-interleaved data
    (s > 1), else None (natural ordering)."""

    n = 0
    layout = None

    def dev_apply(self, x, out):  # pragma: no cover - interface
        raise NotImplementedError

    def graph_key(self):
        """Hashable identity of the exact kernel launches ``dev_apply`` makes
        (fixed device objects and scalars, no host synchronisation), so that
        one application can be captured in a CUDA graph and replayed; None
        when it cannot (host callbacks, iterative solves that poll)."""
        return None

    def account(self, applications: int) -> None:
        """Book-keeping of ``applications`` replays of a captured
        application (the inner iteration counts a direct call records)."""

    def discard(self, applications: int) -> None:
        """Drop the book-keeping of the last ``applications`` direct calls
        (the warm-up and capture calls of a cycle graph are not solves)."""

    def fixed_solves(self) -> bool:
        """True when the application is a sweep of fixed-iteration
        sine-transform block solves (large systems keep device cycles)."""
        return False


class _SpmvOp(_DevOp):
    def __init__(self, A: SparseMatrix):
        self.A = A
        self.n = A.nrows
        self._dm = A.device()

    def dev_apply(self, x, out):
        self._dm.spmv(x, out)

    def graph_key(self):
        return ("spmv", self._dm.serial)


class _HostCallbackOp(_DevOp):
    """A user-supplied host callable (or object with .apply): data crosses to
    the host for the call.  Only reached for user code the reference also
    accepts (sparsela.py:282-296); every built-in operator is device-native."""

    def __init__(self, fn, n):
        self.fn = fn
        self.n = n

    def dev_apply(self, x, out):
        y = self.fn(to_host(x))
        out.copy_(to_dev(np.asarray(y, dtype=np.float64).reshape(-1)))


class _PermutedOp(_DevOp):
    """Adapter running a natural-order operator on interleaved (m, s) data."""

    def __init__(self, inner: _DevOp, m: int, s: int):
        self.inner, self.m, self.s = inner, m, s
        self.n = m * s
        self.layout = (m, s)

    def dev_apply(self, x, out):
        a = dev_empty(self.n)
        b = dev_empty(self.n)
        call("irk_to_stage_major", ctx(), self.m, self.s, ptr(x), ptr(a))
        self.inner.dev_apply(a, b)
        call("irk_to_interleaved", ctx(), self.m, self.s, ptr(b), ptr(out))


def as_dev_op(obj, n):
    """Interpret op/pc arguments the way the reference's _as_apply does
    (sparsela.py:282-296), returning device operators."""
    if obj is None:
        return None
    if isinstance(obj, _DevOp):
        return obj
    if hasattr(obj, "_dev_op"):
        return obj._dev_op()
    if isinstance(obj, np.ndarray):
        return _SpmvOp(SparseMatrix.from_dense(obj))
    try:
        import scipy.sparse as sp

        if sp.issparse(obj):
            return _SpmvOp(SparseMatrix.from_scipy(obj))
    except ImportError:  # pragma: no cover
        pass
    if is_torch(obj):
        return _SpmvOp(SparseMatrix.from_dense(to_host(obj)))
    if hasattr(obj, "apply"):
        return _HostCallbackOp(obj.apply, n)
    if callable(obj):
        return _HostCallbackOp(obj, n)
    raise TypeError(f"cannot interpret {type(obj).__name__} as a linear operator")


# -------------------------------------------------------- block solves


# blocks of at most this many rows are solved directly (dense inverse):
# below it the iterative solves are launch-latency-bound
DIRECT_MAX = 2048


@dataclass
class BlockSolveSettings:
    """Inner diagonal-block solver (replaces SuperLU, sparsela.py:149-191).

    method: "auto" (a direct solve for blocks of at most DIRECT_MAX rows;
    for larger blocks of P1 grid operators CG preconditioned by the fast
    sine transform where it applies (2D, full-boundary Dirichlet set, N a
    power of two <= 2048: the symmetrised grid stencil inverted exactly by
    DST-I, ~2 iterations to 1e-6), else by a multigrid V-cycle;
    Jacobi-PCG otherwise), "dst" (sine-transform-preconditioned CG
    required), "direct" (the block inverse, formed once on the
    device, applied by one dense matrix-vector kernel: the exact solve of
    the reference's SuperLU factorisation at sizes where the iterative
    solvers are launch-latency-bound), "mg" (multigrid required), "pcg"
    (Jacobi-preconditioned CG) or "chebyshev" (Jacobi-Chebyshev: no inner
    products, eigenvalue bounds of D^-1 B from Gershgorin discs -- the block
    must be strictly diagonally dominant with a positive diagonal, else
    ValueError; ``cheb_iters`` sweeps, 0 = as many as the Chebyshev error
    bound 2/T_k needs for ``rtol``, at most ``maxit``).
    mg_nu / mg_coarse_steps: Chebyshev smoothing steps per level (0: automatic
    = 2; the structured 2D path fuses up to 4) and on the coarsest level of the
    multigrid V-cycle; mg_coarse_ratio: coarsening stops
    once beta / (alpha H^2) of a level is at most this (mass-dominated).
    raise_on_maxit: when False (preconditioner use) an unconverged block
    returns its last iterate, FGMRES being flexible."""

    method: str = "auto"
    rtol: float = 1e-6
    atol: float = 0.0
    maxit: int = 20000
    raise_on_maxit: bool = False
    cheb_iters: int = 0
    mg_nu: int = 0
    mg_coarse_steps: int = 4
    mg_coarse_ratio: float = 0.5

    def __post_init__(self):
        if self.method not in ("auto", "pcg", "mg", "dst", "chebyshev", "direct"):
            raise ValueError(f"unknown block solver {self.method!r}")
        if self.rtol < 0 or self.atol < 0 or self.maxit < 0 or self.cheb_iters < 0:
            raise ValueError("block solver tolerances must be non-negative")


_DST_OFF = bool(os.environ.get("IRK_NO_DST"))  # A/B: multigrid V-cycle under "auto"
_DEVFG_DST_OFF = bool(os.environ.get("IRK_NO_DEVFG_DST"))  # A/B: no captured fixed solves


class _MgHierarchy:
    """Geometric multigrid levels of a P1 stage block alpha*M + beta*K
    (libirk irk_mg_*): level l re-assembles the operator with N/2^l cells per
    direction (nested P1 grids: the Galerkin operator), Dirichlet rows where
    the coincident fine node is constrained.  Coarsening stops at odd N, at
    N < 4, or once the level is mass-dominated (beta/(alpha H^2) <=
    mg_coarse_ratio), where a few Chebyshev steps solve it well enough."""

    def __init__(self, handle, keep):
        self.handle = handle
        self._keep = keep  # level matrices and masks referenced by the handle

    def __del__(self):
        try:
            if self.handle:
                _lib.load().irk_mg_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass

    @staticmethod
    def build(M, K, alpha, beta, mask, B, settings):
        grid = getattr(M, "_p1_grid", None)
        if grid is None or getattr(K, "_p1_grid", None) != grid or alpha <= 0 or beta < 0:
            return None
        dim, N = grid
        torch = _torch()
        n1 = N + 1
        if mask is not None:
            # only the full-boundary Dirichlet set (the coarse masks are the
            # boundaries of the coarse grids)
            idx = torch.arange(n1 ** dim, device=mask.device)
            on = torch.zeros_like(idx, dtype=torch.bool)
            for d in range(dim):
                k = (idx // n1 ** d) % n1
                on |= (k == 0) | (k == N)
            if not torch.equal(on, mask.bool()):
                return None
        Ns, mats, masks = [N], [B], [mask]
        while Ns[-1] % 2 == 0 and Ns[-1] // 2 >= 4 and len(Ns) < 12:
            H = 1.0 / Ns[-1]
            if beta / (alpha * H * H) <= settings.mg_coarse_ratio:
                break
            Nc = Ns[-1] // 2
            hM, hK = C.c_void_p(), C.c_void_p()
            call("irk_mat_assemble_p1", ctx(), dim, Nc, C.byref(hM), C.byref(hK))
            Mc, Kc = DeviceMatrix(hM), DeviceMatrix(hK)
            Bc = Mc.combine(alpha, Kc, beta)
            mc = None
            if mask is not None:
                shape = (Ns[-1] + 1,) * dim
                prev = masks[-1]
                mc = prev.reshape(shape)[(slice(None, None, 2),) * dim].contiguous().reshape(-1)
                Bc = Bc.constrain(mc, 1.0)
            Ns.append(Nc)
            mats.append(Bc)
            masks.append(mc)
        L = len(Ns)
        Nh = np.ascontiguousarray(Ns, dtype=np.int64)
        hm = (C.c_void_p * L)(*[A.handle for A in mats])
        mp = (C.c_void_p * L)(*[ptr(m) if m is not None else None for m in masks])
        h = C.c_void_p()
        call("irk_mg_create", ctx(), dim, L, hptr(Nh), C.cast(hm, C.c_void_p),
             C.cast(mp, C.c_void_p), int(settings.mg_nu), int(settings.mg_coarse_steps),
             C.byref(h))
        return _MgHierarchy(h, (mats, masks))

    @property
    def levels(self):
        return len(self._keep[0])

    @property
    def structured(self) -> bool:
        """True when the V-cycle runs the matrix-free 2D stencil kernels."""
        on = C.c_int()
        call("irk_mg_info", self.handle, None, C.byref(on))
        return bool(on.value)

    @structured.setter
    def structured(self, on: bool):
        call("irk_mg_set_structured", self.handle, int(bool(on)))

    @property
    def dst_available(self) -> bool:
        ok = C.c_int()
        call("irk_mg_dst_info", self.handle, C.byref(ok), None)
        return bool(ok.value)

    @property
    def dst(self) -> bool:
        """True when CG is preconditioned by the fast sine transform of the
        level-0 block (irk_dst.cuh) instead of the V-cycle."""
        on = C.c_int()
        call("irk_mg_dst_info", self.handle, None, C.byref(on))
        return bool(on.value)

    @dst.setter
    def dst(self, on: bool):
        call("irk_mg_set_dst", self.handle, int(bool(on)))


class _MgcHierarchy:
    """Complex multigrid of a Schur-pair block alpha*M + beta*K (complex
    alpha, beta; libirk irk_mgc_*): the P1 levels of M and K re-assembled on
    N/2^l grids, masked rows/columns eliminated, combined on the fly.  Same
    coarsening rule as _MgHierarchy with |beta| / (|alpha| H^2)."""

    def __init__(self, handle, keep):
        self.handle = handle
        self._keep = keep

    def __del__(self):
        try:
            if self.handle:
                _lib.load().irk_mgc_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass

    @property
    def levels(self):
        return len(self._keep[0])

    @property
    def structured(self) -> bool:
        """True when the V-cycle runs the matrix-free 3D stencil kernels."""
        on = C.c_int()
        call("irk_mgc_info", self.handle, None, C.byref(on))
        return bool(on.value)

    @structured.setter
    def structured(self, on: bool):
        call("irk_mgc_set_structured", self.handle, int(bool(on)))

    @property
    def dst_available(self) -> bool:
        ok = C.c_int()
        call("irk_mgc_dst_info", self.handle, C.byref(ok), None)
        return bool(ok.value)

    @property
    def dst(self) -> bool:
        """True when COCG is preconditioned by the 3D fast sine transform of
        the level-0 block (irk_dst3.cu) instead of the V-cycle."""
        on = C.c_int()
        call("irk_mgc_dst_info", self.handle, None, C.byref(on))
        return bool(on.value)

    @dst.setter
    def dst(self, on: bool):
        call("irk_mgc_set_dst", self.handle, int(bool(on)))

    @staticmethod
    def build(M, K, Md, Kd, alpha: complex, beta: complex, mask, settings):
        """M, K: the SparseMatrix pair (grid-tagged); Md, Kd: their device
        copies with the mask eliminated (level 0)."""
        grid = getattr(M, "_p1_grid", None)
        if grid is None or getattr(K, "_p1_grid", None) != grid or abs(alpha) == 0:
            return None
        if settings.method not in ("auto", "mg", "dst"):
            return None
        dim, N = grid
        torch = _torch()
        n1 = N + 1
        if mask is not None:
            idx = torch.arange(n1 ** dim, device=mask.device)
            on = torch.zeros_like(idx, dtype=torch.bool)
            for d in range(dim):
                k = (idx // n1 ** d) % n1
                on |= (k == 0) | (k == N)
            if not torch.equal(on, mask.bool()):
                return None
        Ns, ms, ks, masks = [N], [Md], [Kd], [mask]
        while Ns[-1] % 2 == 0 and Ns[-1] // 2 >= 4 and len(Ns) < 12:
            H = 1.0 / Ns[-1]
            if abs(beta) / (abs(alpha) * H * H) <= settings.mg_coarse_ratio:
                break
            Nc = Ns[-1] // 2
            hM, hK = C.c_void_p(), C.c_void_p()
            call("irk_mat_assemble_p1", ctx(), dim, Nc, C.byref(hM), C.byref(hK))
            Mc, Kc = DeviceMatrix(hM), DeviceMatrix(hK)
            mc = None
            if mask is not None:
                shape = (Ns[-1] + 1,) * dim
                mc = masks[-1].reshape(shape)[(slice(None, None, 2),) * dim].contiguous()
                mc = mc.reshape(-1)
                Mc, Kc = Mc.eliminated(mc), Kc.eliminated(mc)
            Ns.append(Nc)
            ms.append(Mc)
            ks.append(Kc)
            masks.append(mc)
        L = len(Ns)
        Nh = np.ascontiguousarray(Ns, dtype=np.int64)
        hm = (C.c_void_p * L)(*[A.handle for A in ms])
        hk = (C.c_void_p * L)(*[A.handle for A in ks])
        mp = (C.c_void_p * L)(*[ptr(m) if m is not None else None for m in masks])
        h = C.c_void_p()
        nu = int(settings.mg_nu) or 2
        call("irk_mgc_create", ctx(), dim, L, hptr(Nh), C.cast(hm, C.c_void_p),
             C.cast(hk, C.c_void_p), C.cast(mp, C.c_void_p), float(alpha.real),
             float(alpha.imag), float(beta.real), float(beta.imag), nu,
             int(settings.mg_coarse_steps), C.byref(h))
        hier = _MgcHierarchy(h, (ms, ks, masks))
        if settings.method in ("auto", "dst") and not _DST_OFF:
            if hier.dst_available:
                hier.dst = True
            elif settings.method == "dst":
                raise ValueError("sine-transform pair-block solver needs a 3D P1 grid block with "
                                 "the full-boundary Dirichlet set and 2N = 2^a or 3*2^a in "
                                 "[24, 384]")
        return hier


class BlockFactorization:
    """Stage block alpha*M + dt*K with Dirichlet identity rows/columns,
    solved on the device (drop-in for sparsela.py:149-168).

    ``solve``/``apply``/``matvec``/``matrix``/``n`` as in the reference;
    ``dev_solve`` is the device entry used by the preconditioners."""

    def __init__(self, M: SparseMatrix, K: SparseMatrix, alpha: float, dt: float, dofs=None,
                 settings: BlockSolveSettings | None = None):
        self.n = M.nrows
        self.alpha = float(alpha)
        self.beta = float(dt)
        self.dofs = np.asarray(dofs if dofs is not None else [], dtype=np.int64)
        self.settings = settings or BlockSolveSettings(rtol=1e-12, raise_on_maxit=True)
        Md, Kd = shared_pattern([M.device(), K.device()])
        B = Md.combine(self.alpha, Kd, self.beta)
        self.mask = dof_mask(self.n, self.dofs) if len(self.dofs) else None
        if self.mask is not None:
            B = B.constrain(self.mask, 1.0)
        self._B = B
        self._serial = next(_SERIAL)
        self._matrix = None
        self.last_iterations = 0
        self.last_relres = 0.0
        self._check_regular()
        self._mg = None
        self._inv = None
        self._cheb = None
        self._fixed = {}  # (rtol, atol, maxit) -> captured iteration count or None
        meth = self.settings.method
        # direct: the inverse is formed on the first solve, so factors that are
        # built but never solved with (regularity checks of per-Newton blocks
        # that the batched path handles) cost no inversion
        self.direct = meth == "direct" or (meth == "auto" and 0 < self.n <= DIRECT_MAX)
        if meth == "direct" and self.n > 8192:
            raise ValueError(f"direct block solve limited to 8192 rows, got {self.n}")
        if meth == "chebyshev":
            self._cheb = self._chebyshev_bounds()
        elif self.direct:
            pass
        elif meth in ("auto", "mg", "dst"):
            self._mg = _MgHierarchy.build(M, K, self.alpha, self.beta, self.mask, B,
                                          self.settings)
            if self._mg is None and meth != "auto":
                raise ValueError(f"{meth!r} block solver needs M, K from assemble_p1 "
                                 "(nested structured-grid P1 operators)")
            if self._mg is not None and meth in ("auto", "dst") and not _DST_OFF:
                if self._mg.dst_available:
                    self._mg.dst = True
                elif meth == "dst":
                    raise ValueError("sine-transform block solver needs a 2D P1 grid block with "
                                     "the full-boundary Dirichlet set and N a power of two in "
                                     "[32, 2048]")

    def _chebyshev_bounds(self):
        """[lmin, lmax] of D^-1 B from Gershgorin discs (irk_mat_absrowsum):
        disc r is centred at 1 with radius sum_c |B[r,c]| / |B[r,r]| - 1."""
        torch = _torch()
        if self.n == 0:
            return (0.5, 1.5)
        d = self._B.diagonal()
        a = dev_empty(self.n)
        call("irk_mat_absrowsum", ctx(), self._B.handle, ptr(a))
        if bool((d <= 0).any()):
            raise ValueError("Chebyshev block solver needs a positive diagonal")
        ratio = a / d
        lmin = float(torch.min(2.0 - ratio))
        lmax = float(torch.max(ratio))
        if not lmin > 1e-14 * lmax:
            raise ValueError("Chebyshev block solver: the block is not strictly diagonally "
                             f"dominant (Gershgorin lower bound {lmin:.3e}); use method='pcg'")
        if lmax <= lmin:
            lmax = lmin * (1.0 + 1e-12) + 1e-300
        return (lmin, lmax)

    def chebyshev_iterations(self, settings=None) -> int:
        """Sweeps of the Chebyshev solve: cheb_iters, or the smallest k with
        2 / T_k((lmax+lmin)/(lmax-lmin)) <= rtol (capped at maxit)."""
        st = settings or self.settings
        if st.cheb_iters > 0:
            return int(st.cheb_iters)
        lmin, lmax = self._cheb
        if st.rtol <= 0:
            return max(1, int(st.maxit))
        sigma = (lmax + lmin) / (lmax - lmin)
        k = np.arccosh(2.0 / min(st.rtol, 1.0)) / np.arccosh(sigma)
        return int(max(1, min(int(np.ceil(k)), max(1, int(st.maxit)))))

    def _dense_inverse(self):
        """B^-1 as a dense row-major device array (one-time setup: the CSR
        scattered into a dense block on the device, inverted by cuSOLVER
        through torch; the per-solve work is irk_dense_gemv)."""
        torch = _torch()
        if self.n > 8192:
            raise ValueError(f"direct block solve limited to 8192 rows, got {self.n}")
        dense = torch.empty((self.n, self.n), dtype=torch.float64, device=device())
        call("irk_mat_to_dense", ctx(), self._B.handle, ptr(dense))
        try:
            inv = torch.linalg.inv(dense)
        except RuntimeError as exc:  # torch.linalg.LinAlgError
            raise FactorizationError(f"stage block is singular: {exc}") from exc
        if not bool(torch.isfinite(inv).all()):
            raise FactorizationError("stage block is singular (non-finite inverse)")
        return inv.contiguous()

    def _check_regular(self):
        torch = _torch()
        d = self._B.diagonal()
        if self.n == 0:
            return
        if not bool(torch.isfinite(d).all()) or bool((d == 0).any()):
            raise FactorizationError("stage block has a zero or non-finite diagonal entry")
        # pure-Neumann detection: the constants lie in the nullspace
        rs = self._B.rowsum()
        scale = float(torch.abs(d).max())
        if float(torch.abs(rs).max()) <= 1e-13 * scale:
            raise FactorizationError("stage block is singular (constant vectors in its nullspace)")

    @property
    def matrix(self) -> SparseMatrix:
        if self._matrix is None:
            self._matrix = SparseMatrix._from_device(self._B)
        return self._matrix

    def dev_solve(self, rhs, x, ld_rhs=1, ld_x=1, nb=1, settings: BlockSolveSettings | None = None,
                  defer: bool = False, checked: bool = False):
        """Solve on device data.  defer=True (inside _lib.deferred_solves, for
        preconditioner use that never raises): no host synchronisation, the
        outcome goes to the context's solve log and None is returned.
        checked=True defers even with raise_on_maxit: the caller reads the
        log codes (1 cap, 2 breakdown) and raises."""
        st = settings or self.settings
        if self.direct and st.method in ("auto", "direct"):
            if self._inv is None:
                self._inv = self._dense_inverse()
            call("irk_dense_gemv", ctx(), self.n, ptr(self._inv), ptr(rhs), int(ld_rhs), ptr(x),
                 int(ld_x))
            self.last_iterations, self.last_relres = 1, 0.0
            return 1  # exact: no log entry even when deferred
        if st.method == "chebyshev":
            if self._cheb is None:
                self._cheb = self._chebyshev_bounds()
            k = self.chebyshev_iterations(st)
            one = np.ones(1)
            lo, hi = np.array([self._cheb[0]]), np.array([self._cheb[1]])
            call("irk_chebyshev", ctx(), 1, hptr(one), None, self._B.handle, None, None, None,
                 hptr(lo), hptr(hi), ptr(rhs), int(ld_rhs), ptr(x), int(ld_x), int(k))
            self.last_iterations, self.last_relres = k, float("nan")
            return k  # fixed sweep count: nothing to log or check
        if self._fixed and _torch().cuda.is_current_stream_capturing():
            k = self._fixed_iterations(st)
            if k is None:
                raise RuntimeError("block solve is not capturable with these settings")
            call("irk_mg_pcg", ctx(), self._mg.handle, ptr(rhs), int(ld_rhs), ptr(x), int(ld_x),
                 float(st.rtol), float(st.atol), int(k), None, None)
            self.last_iterations, self.last_relres = k, float("nan")
            return k  # fixed straight-line iterations: nothing logged
        its = np.zeros(8, dtype=np.int32)
        rel = np.zeros(8, dtype=np.float64)
        one = np.ones(8)
        defer = defer and (checked or not st.raise_on_maxit)
        its_p, rel_p = (None, None) if defer else (hptr(its), hptr(rel))
        if self._mg is not None and st.method in ("auto", "mg", "dst"):
            status = _lib.load().irk_mg_pcg(
                ctx(), self._mg.handle, ptr(rhs), int(ld_rhs), ptr(x), int(ld_x),
                float(st.rtol), float(st.atol), int(st.maxit), its_p, rel_p)
        else:
            status = _lib.load().irk_pcg(
                ctx(), 1, hptr(one), C.c_void_p(), self._B.handle, C.c_void_p(), C.c_void_p(),
                C.c_void_p(), ptr(rhs), int(ld_rhs), ptr(x), int(ld_x), float(st.rtol),
                float(st.atol), int(st.maxit), its_p, rel_p)
        if defer:
            _lib.check(status, "deferred block solve")
            return None
        self.last_iterations = int(its[0])
        self.last_relres = float(rel[0])
        if status == _lib.IRK_ENOCONV:
            if st.raise_on_maxit:
                raise NonConvergenceError(
                    f"block PCG: no convergence in {st.maxit} iterations "
                    f"(relative residual {rel[0]:.3e})", [float(rel[0])])
            return int(its[0])
        if status == _lib.IRK_ESINGULAR:
            if not st.raise_on_maxit:
                return int(its[0])  # preconditioner use: keep the last iterate
            raise FactorizationError(f"block PCG breakdown: {_lib.last_error()}")
        _lib.check(status, "irk_pcg")
        return int(its[0])

    def solve(self, b):
        bd = to_dev(b)
        if bd.shape != (self.n,):
            raise ValueError(f"block solve expects length {self.n}, got {tuple(bd.shape)}")
        x = dev_empty(self.n)
        self.dev_solve(bd, x)
        return _like_input(x, b)

    apply = solve

    def matvec(self, x):
        xd = to_dev(x)
        y = dev_empty(self.n)
        self._B.spmv(xd, y)
        return _like_input(y, x)

    def graph_safe(self, settings: BlockSolveSettings | None = None) -> bool:
        """dev_solve is a fixed kernel sequence without host synchronisation
        (direct inverse or fixed-sweep Chebyshev): capturable in a graph."""
        st = settings or self.settings
        meth = st.method
        if (self.direct and meth in ("auto", "direct")) or meth == "chebyshev":
            return True
        return self._fixed_iterations(st) is not None

    def _fixed_iterations(self, st) -> int | None:
        """Iteration count of a capturable sine-transform-preconditioned CG
        solve, or None.  The preconditioner is the exact inverse of the
        symmetrised stencil, so CG converges in a problem-independent handful
        of iterations: a probe solve (random right-hand side, once per factor
        and tolerance) measures the count, and a captured solve issues exactly
        that many straight-line iterations (run_cg's captured branch).  Only
        for preconditioner use (raise_on_maxit False: FGMRES is flexible, an
        iterate short of rtol costs outer iterations, not correctness)."""
        if _DEVFG_DST_OFF or st.raise_on_maxit or self._mg is None or self.direct:
            return None
        if st.method not in ("auto", "mg", "dst") or not self._mg.dst:
            return None
        key = (float(st.rtol), float(st.atol), int(st.maxit))
        if key not in self._fixed:
            torch = _torch()
            g = torch.Generator(device="cuda").manual_seed(7)
            b = torch.rand(self.n, dtype=torch.float64, device="cuda", generator=g)
            x = dev_empty(self.n)
            k = self.dev_solve(b, x, settings=st)
            ok = self.last_relres <= st.rtol or st.atol > 0
            self._fixed[key] = int(k) if (ok and 1 <= int(k) <= 4) else None
        return self._fixed[key]

    def _dev_op(self):
        fac = self

        class _Op(_DevOp):
            n = fac.n

            def dev_apply(self, x, out):
                fac.dev_solve(x, out)

            def graph_key(self):
                return ("fac", fac._serial) if fac.graph_safe() else None

        return _Op()


def factorize_block(M: SparseMatrix, K: SparseMatrix, alpha: float, dt: float, dirichlet=None,
                    settings: BlockSolveSettings | None = None) -> BlockFactorization:
    """Prepare alpha*M + dt*K (optionally Dirichlet-constrained) for device
    solves (sparsela.py:171-191)."""
    if M.shape != K.shape or M.nrows != M.ncols:
        raise ValueError("factorize_block needs square M, K of equal shape")
    dofs = None
    if dirichlet is not None and len(dirichlet):
        dofs = np.asarray(dirichlet, dtype=np.int64)
        if dofs.min() < 0 or dofs.max() >= M.nrows:
            raise ValueError("constrained dof index out of range")
    return BlockFactorization(M, K, alpha, dt, dofs, settings)


# -------------------------------------------------- Kronecker stage operator


class KroneckerStageOperator:
    """Matrix-free C1 (x) M + dt C2 (x) K on stacked stage vectors
    (sparsela.py:194-250), executed by the fused interleaved kernel K2.

    ``Ks`` is one stiffness matrix or one (row-indexed) matrix per stage."""

    def __init__(self, C1, C2, M: SparseMatrix, Ks, dt: float):
        self.C1 = np.ascontiguousarray(C1, dtype=np.float64)
        self.C2 = np.ascontiguousarray(C2, dtype=np.float64)
        self.M = M
        self.Ks = list(Ks) if isinstance(Ks, (list, tuple)) else [Ks]
        self.dt = float(dt)
        s = self.C1.shape[0] if self.C1.ndim == 2 else -1
        if self.C1.shape != (s, s) or self.C2.shape != (s, s):
            raise ValueError("C1, C2 must be square and of equal size")
        if len(self.Ks) not in (1, s):
            raise ValueError("Ks must hold one matrix or one per stage")
        m = M.nrows
        for K in self.Ks:
            if K.shape != (m, m) or M.shape != (m, m):
                raise ValueError("M and K blocks must be square and of equal shape")
        if s > 8:
            raise ValueError("at most 8 stages are supported on the device")
        self.s = s
        self.m = m
        self.n = s * m
        self._mats = None

    # -- device ---------------------------------------------------------
    def _device_mats(self):
        if self._mats is None:
            self._mats = shared_pattern([self.M.device()] + [K.device() for K in self.Ks])
        return self._mats

    def dev_apply(self, Y, Out, mask=None):
        mats = [d.eliminated(mask) for d in self._device_mats()]
        Md, Ks = mats[0], mats[1:]
        arr = (C.c_void_p * len(Ks))(*[k.handle.value for k in Ks])
        call("irk_stage_apply", ctx(), self.s, hptr(self.C1), hptr(self.C2), self.dt, Md.handle,
             C.cast(arr, C.c_void_p), len(Ks), ptr(mask), ptr(Y), ptr(Out))
        return Out

    def _dev_op(self, mask=None):
        op = self

        class _Op(_DevOp):
            n = op.n
            layout = (op.m, op.s) if op.s > 1 else None

            def dev_apply(self, x, out):
                op.dev_apply(x, out, mask)

            def graph_key(self):
                mats = [d.eliminated(mask) for d in op._device_mats()]
                return ("kron", op.s, op.C1.tobytes(), op.C2.tobytes(), op.dt,
                        tuple(d.serial for d in mats),
                        mask.data_ptr() if mask is not None else 0)

        return _Op()

    # -- reference API --------------------------------------------------
    def apply(self, v):
        vd = to_dev(v)
        if tuple(vd.shape) != (self.n,):
            raise ValueError(f"operator expects length {self.n}, got {tuple(vd.shape)}")
        out = stage_major_apply(self._dev_op(), vd, self.m, self.s)
        return _like_input(out, v)

    def to_dense(self) -> np.ndarray:
        """Explicit Kronecker assembly (host, small-m cross-checks only)."""
        Md = self.M.to_dense()
        out = np.kron(self.C1, Md)
        if len(self.Ks) == 1:
            out += self.dt * np.kron(self.C2, self.Ks[0].to_dense())
        else:
            m = self.m
            for i in range(self.s):
                Kd = self.Ks[i].to_dense()
                for j in range(self.s):
                    out[i * m:(i + 1) * m, j * m:(j + 1) * m] += self.dt * self.C2[i, j] * Kd
        return out


def stage_major_apply(devop: _DevOp, vd, m, s):
    """Apply an interleaved device operator to a stage-major vector."""
    if s == 1 or devop.layout is None:
        out = dev_empty(vd.numel())
        devop.dev_apply(vd, out)
        return out
    a = dev_empty(m * s)
    b = dev_empty(m * s)
    out = dev_empty(m * s)
    call("irk_to_interleaved", ctx(), m, s, ptr(vd), ptr(a))
    devop.dev_apply(a, b)
    call("irk_to_stage_major", ctx(), m, s, ptr(b), ptr(out))
    return out


def apply_kronecker(op: KroneckerStageOperator, v):
    return op.apply(v)


# ------------------------------------------------------------------ FGMRES


@dataclass
class KrylovSettings:
    """FGMRES controls (sparsela.py:257-272) + ``reorth`` (CGS2 pass)."""

    rtol: float = 1e-8
    atol: float = 1e-50
    restart: int = 50
    maxit: int = 500
    right_pc: bool = True
    reorth: bool = False

    def __post_init__(self):
        if self.rtol <= 0 or self.atol <= 0:
            raise ValueError("rtol and atol must be positive")
        if self.restart < 1:
            raise ValueError("restart must be >= 1")
        if self.restart > 63:
            raise ValueError("restart must be <= 63 on the device (fused basis limit)")


@dataclass
class FgmresResult:
    x: object
    iterations: int
    residuals: list


def _norm(x) -> float:
    out = dev_empty(1)
    call("irk_norm2", ctx(), int(x.numel()), ptr(x), ptr(out))
    return float(out.item())


def _all_finite(x) -> bool:
    res = C.c_int(0)
    call("irk_all_finite", ctx(), int(x.numel()), ptr(x), C.byref(res))
    return bool(res.value)


# diagnostics (env IRK_FGMRES_GAPS): CUDA events around the per-iteration
# host read of the Hessenberg column; profiles/fgmres_gaps.py reads them
_GAPS = [] if __import__("os").environ.get("IRK_FGMRES_GAPS") else None


def _ev_rec():
    e = _torch().cuda.Event(enable_timing=True)
    e.record()
    return e


# ------------------------------------------- device-resident FGMRES cycles
# Systems of at most this many unknowns whose operator and preconditioner
# are graph-capturable run each restart cycle as ONE CUDA graph (libirk
# irk_fgmres_graph_*: Arnoldi, Givens and the stop tests on the device);
# larger ones keep the host Givens loop (its per-iteration round trip is a
# small share of their iteration).  Env IRK_NO_DEVFGMRES: always the host loop.
DEVFG_MAX_N = 1 << 16
_DEVFG_OFF = bool(os.environ.get("IRK_NO_DEVFGMRES"))
# Above DEVFG_MAX_N the cycles still run on the device when the preconditioner
# is a sweep over sine-transform-preconditioned blocks (fixed straight-line
# solves, BlockFactorization._fixed_iterations): there the host round trip per
# Arnoldi step and the eager <-> graph boundaries around every block solve are
# ~15 % of a step.  The basis (restart + 1 vectors) and Z stay allocated with
# the cached graph, so the size is bounded.  Env IRK_NO_DEVFG_DST: host loop.
DEVFG_DST_MAX_N = 1 << 23
_FG_CACHE: "OrderedDict[tuple, _FgmresGraph]" = OrderedDict()
_FG_SEEN: dict = {}


class _FgmresGraph:
    """Cached cycle graph for one (operator, preconditioner, n, restart):
    the application w = A P v_j is captured once with torch.cuda.graph on
    fixed buffers and embedded in libirk's WHILE-loop graph."""

    def __init__(self, A: _DevOp, P: _DevOp | None, n: int, cycle: int, reorth: bool):
        torch = _torch()
        lib = _lib.load()
        self.n, self.cycle, self.P = n, cycle, P
        self.V = dev_empty((cycle + 1) * n)
        self.Z = dev_empty(cycle * n) if P is not None else None
        self.vj = dev_zeros(n)
        self.zj = dev_zeros(n) if P is not None else None
        self.w = dev_empty(n)
        self.work = dev_zeros(int(lib.irk_fgmres_work_doubles(cycle)))
        self.st = torch.zeros(8, dtype=torch.int32, device="cuda")
        self.hist = np.zeros(cycle + 1)
        self.k = C.c_int(0)
        self.conv = C.c_int(0)
        self.handle = None
        self._step(A)  # lazy set-up (inverses, eliminated matrices) outside the capture
        torch.cuda.synchronize()
        self.tg = torch.cuda.CUDAGraph(keep_graph=True)
        # no garbage collection inside the capture: a finalizer freeing device
        # memory (cudaFree) would invalidate it
        was = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(self.tg, capture_error_mode="thread_local"):
                self._step(A)
        finally:
            if was:
                gc.enable()
        if P is not None:
            P.discard(2)  # the warm-up and the captured application
        h = C.c_void_p()
        call("irk_fgmres_graph_create", ctx(), C.c_void_p(self.tg.raw_cuda_graph()), n, cycle,
             1 if reorth else 0, ptr(self.V), n, ptr(self.Z), n, ptr(self.vj), ptr(self.zj),
             ptr(self.w), ptr(self.work), ptr(self.st), C.byref(h))
        self.handle = h

    def _step(self, A):
        if self.P is not None:
            self.P.dev_apply(self.vj, self.zj)
            A.dev_apply(self.zj, self.w)
        else:
            A.dev_apply(self.vj, self.w)

    def run(self, cap, r, beta, target, breakdown, x):
        """One cycle: (steps taken, converged, residual estimates 1..k)."""
        status = _lib.load().irk_fgmres_graph_run(
            ctx(), self.handle, int(cap), ptr(r), float(beta), float(target), float(breakdown),
            ptr(x), C.byref(self.k), C.byref(self.conv), hptr(self.hist))
        if status == _lib.IRK_EINVAL:
            return None  # the context scratch moved: the caller rebuilds
        _lib.check(status, "irk_fgmres_graph_run")
        k = int(self.k.value)
        if self.P is not None:
            self.P.account(k)
        return k, bool(self.conv.value), [float(v) for v in self.hist[1:k + 1]]

    def __del__(self):
        try:
            if self.handle:
                _lib.load().irk_fgmres_graph_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass


def _fgmres_graph(A, P, n, st, rebuild=False):
    """The cached cycle graph for (A, P), or None (not capturable, too large,
    or a key seen for the first time: one-off operators are not captured)."""
    if _DEVFG_OFF or st.restart >= 64 or not st.right_pc:
        return None
    if n > DEVFG_MAX_N and (P is None or n > DEVFG_DST_MAX_N or not P.fixed_solves()):
        return None
    ka = A.graph_key()
    kp = P.graph_key() if P is not None else ()
    if ka is None or kp is None:
        return None
    key = (ka, kp, n, st.restart, bool(st.reorth))
    g = None if rebuild else _FG_CACHE.get(key)
    if g is not None:
        _FG_CACHE.move_to_end(key)
        return g
    if not rebuild:
        if len(_FG_SEEN) > 4096:
            _FG_SEEN.clear()
        _FG_SEEN[key] = _FG_SEEN.get(key, 0) + 1
        if _FG_SEEN[key] < 2:
            return None
    try:
        g = _FgmresGraph(A, P, n, st.restart, st.reorth)
    except Exception:
        # not capturable after all: the host loop from now on for this key
        _FG_SEEN[key] = -(1 << 30)
        _torch().cuda.synchronize()
        return None
    _FG_CACHE[key] = g
    while len(_FG_CACHE) > 8:
        _FG_CACHE.popitem(last=False)
    return g


def fgmres_device(A: _DevOp, b, P: _DevOp | None = None, settings: KrylovSettings | None = None,
                  x0=None) -> FgmresResult:
    """Restarted flexible GMRES on device vectors (control flow of
    sparsela.py:299-403): right preconditioning by default, Givens rotations
    and convergence test on the host, Arnoldi step = one fused CGS
    projection pass + one fused update/norm pass on the device."""
    st = settings or KrylovSettings()
    n = int(b.numel())
    left = P is not None and not st.right_pc
    # one host synchronisation for the finiteness check and ||rhs|| (the
    # norm of a finite vector is finite unless its entries exceed ~1e154)
    normb = _norm(b) if not left else None
    if (normb is None or not np.isfinite(normb)) and not _all_finite(b):
        raise ValueError("right-hand side contains non-finite entries")
    if left:
        rhs = dev_empty(n)
        P.dev_apply(b, rhs)
        normb = _norm(rhs)
    else:
        rhs = b
    x = dev_zeros(n) if x0 is None else to_dev(x0).clone()

    def residual_of(xv):
        t = dev_empty(n)
        A.dev_apply(xv, t)
        r_ = b.clone()
        call("irk_axpby", ctx(), n, -1.0, ptr(t), 1.0, ptr(r_))
        if left:
            pr = dev_empty(n)
            P.dev_apply(r_, pr)
            return pr
        return r_

    r = rhs.clone() if x0 is None else residual_of(x)
    target = max(st.rtol * normb, st.atol)
    residuals = [normb if x0 is None else _norm(r)]
    iterations = 0
    if residuals[0] <= target:
        return FgmresResult(x, 0, residuals)
    breakdown_tol = 1e-14 * normb
    dg = None if left else _fgmres_graph(A, P, n, st)
    if dg is not None:
        # device-resident cycles: one graph launch and one host read per cycle
        while True:
            cycle = min(st.restart, st.maxit - iterations)
            if cycle <= 0:
                raise NonConvergenceError(
                    f"fgmres: no convergence in {st.maxit} iterations "
                    f"(residual {residuals[-1]:.3e}, target {target:.3e})", residuals)
            beta = residuals[-1] if iterations == 0 else _norm(r)
            out = dg.run(cycle, r, beta, target, breakdown_tol, x)
            if out is None:
                dg = _fgmres_graph(A, P, n, st, rebuild=True)
                out = dg.run(cycle, r, beta, target, breakdown_tol, x)
            k, conv, hist = out
            iterations += k
            residuals.extend(hist)
            if conv or residuals[-1] <= target:
                return FgmresResult(x, iterations, residuals)
            if iterations >= st.maxit:
                raise NonConvergenceError(
                    f"fgmres: no convergence in {st.maxit} iterations "
                    f"(residual {residuals[-1]:.3e}, target {target:.3e})", residuals)
            r = residual_of(x)
    hbuf = dev_empty(128)
    tmp = dev_empty(n) if left else None
    while True:
        cycle = min(st.restart, st.maxit - iterations)
        if cycle <= 0:
            raise NonConvergenceError(
                f"fgmres: no convergence in {st.maxit} iterations "
                f"(residual {residuals[-1]:.3e}, target {target:.3e})", residuals)
        beta = residuals[-1] if iterations == 0 else _norm(r)
        V = dev_empty((cycle + 1) * n).view(cycle + 1, n)
        store_z = P is not None and not left
        Z = dev_empty(cycle * n).view(cycle, n) if store_z else V
        call("irk_axpby", ctx(), n, 1.0 / beta, ptr(r), 0.0, ptr(V[0]))
        H = np.zeros((cycle + 1, cycle))
        cs = np.zeros(cycle)
        sn = np.zeros(cycle)
        g = np.zeros(cycle + 1)
        g[0] = beta
        converged = False
        j = -1
        for j in range(cycle):
            w = V[j + 1]
            if _GAPS is not None and j > 0:
                _GAPS.append(_ev_rec())  # first enqueue after the host read of h
            if left:
                A.dev_apply(V[j], tmp)
                P.dev_apply(tmp, w)
            else:
                if store_z:
                    P.dev_apply(V[j], Z[j])
                    A.dev_apply(Z[j], w)
                else:
                    A.dev_apply(V[j], w)
            iterations += 1
            call("irk_multidot", ctx(), n, j + 1, ptr(V), n, ptr(w), ptr(hbuf))
            call("irk_orth_update", ctx(), n, j + 1, ptr(V), n, ptr(hbuf), ptr(w),
                 1 if st.reorth else 0)
            if _GAPS is not None:
                _GAPS.append(_ev_rec())  # GPU work of the iteration ends here
            hcol = hbuf[: j + 2].cpu().numpy()
            H[: j + 2, j] = hcol
            lucky = H[j + 1, j] < breakdown_tol
            if not lucky:
                call("irk_axpby", ctx(), n, 1.0 / H[j + 1, j], ptr(w), 0.0, ptr(w))
            for i in range(j):
                t_ = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t_
            d = np.hypot(H[j, j], H[j + 1, j])
            if d == 0.0:
                cs[j], sn[j] = 1.0, 0.0
                d = 1e-300
            else:
                cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
            H[j, j] = d
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            residuals.append(abs(float(g[j + 1])))
            if residuals[-1] <= target or lucky:
                converged = True
                break
        k = j + 1
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        yh = np.ascontiguousarray(y)
        call("irk_lincomb", ctx(), n, k, ptr(Z), n, hptr(yh), ptr(x))
        if converged or residuals[-1] <= target:
            return FgmresResult(x, iterations, residuals)
        if iterations >= st.maxit:
            raise NonConvergenceError(
                f"fgmres: no convergence in {st.maxit} iterations "
                f"(residual {residuals[-1]:.3e}, target {target:.3e})", residuals)
        r = residual_of(x)


def fgmres(op, b, pc=None, settings: KrylovSettings | None = None, x0=None) -> FgmresResult:
    """Restarted flexible GMRES (drop-in for sparsela.py:299-403).

    ``op``/``pc`` may be a SparseMatrix, ndarray, scipy sparse matrix, an
    object with ``.apply``, a callable, or one of this package's stage
    operators / preconditioners.  Vectors are in the reference's layout
    (stage-major for stage systems); numpy in -> numpy out."""
    bd = to_dev(b).reshape(-1)
    n = int(bd.numel())
    A = as_dev_op(op, n)
    P = as_dev_op(pc, n)
    layouts = {o.layout for o in (A, P) if o is not None and o.layout is not None}
    if len(layouts) > 1:
        raise ValueError("operator and preconditioner disagree on the stage layout")
    x0d = to_dev(x0).reshape(-1) if x0 is not None else None
    if layouts:
        m, s = layouts.pop()
        A = A if A.layout else _PermutedOp(A, m, s)
        P = P if (P is None or P.layout) else _PermutedOp(P, m, s)
        bi = dev_empty(n)
        call("irk_to_interleaved", ctx(), m, s, ptr(bd), ptr(bi))
        xi = None
        if x0d is not None:
            xi = dev_empty(n)
            call("irk_to_interleaved", ctx(), m, s, ptr(x0d), ptr(xi))
        res = fgmres_device(A, bi, P, settings, xi)
        xs = dev_empty(n)
        call("irk_to_stage_major", ctx(), m, s, ptr(res.x), ptr(xs))
        res.x = xs
    else:
        res = fgmres_device(A, bd, P, settings, x0d)
    res.x = _like_input(res.x, b)
    return res


# ------------------------------------------------------------ Matrix Market


def mm_write(path, A: SparseMatrix) -> None:
    """Coordinate Matrix Market, general symmetry (sparsela.py:410-413)."""
    import scipy.io

    scipy.io.mmwrite(str(path), A.to_scipy().tocoo(), symmetry="general")


def mm_read(path) -> SparseMatrix:
    """Matrix Market file -> SparseMatrix (sparsela.py:414-416)."""
    import scipy.io
    import scipy.sparse

    try:
        A = scipy.io.mmread(str(path), spmatrix=False)
    except TypeError:  # scipy without the spmatrix switch
        A = scipy.io.mmread(str(path))
    return SparseMatrix.from_scipy(scipy.sparse.csr_matrix(A))
