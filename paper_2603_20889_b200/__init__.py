"""skinnyqr-b200: B200-native Q-less tall-and-very-skinny QR (FP64, column-major).

Python host-side mirror of the reference's public interface (reference: proj/include/skinnyqr/
{tsqr,gram,gram_qr,lstsq,plan,types}.hpp), bound with ctypes to the C ABI in
``include/skinnyqr_b200.h`` (``libskinnyqr_b200.so``: hand-written sm_100a CUDA kernels).  Same
function names, argument meaning and error behaviour as the reference:

    tsqr_qless, tsqr_stage1, block_qless_qr, tsmttsm, tsmRttsmR, tsmmttsmm, cholesky, eigh_small,
    cholqr2, svqb_pass, svqb2, reconstruct_q, solve_lstsq, default_tsqr_plan, default_gram_plan,
    PanelPlan, sign_normalize, and the exception hierarchy rooted at ``Error``.

Inputs may be

* numpy arrays (host memory): routed through the ``*_host`` entry points, which stream X to the
  GPU in slabs; results come back as Fortran-ordered numpy arrays;
* torch CUDA tensors in column-major layout (``x.stride() == (1, ld)``): routed through the
  ``*_dev`` entry points on torch's current stream; results are torch tensors on the same device
  and numerical failures surface at ``synchronize()``.

There is no CPU fallback: importing works anywhere (so that CPU-only tooling can inspect the ABI),
but every computation needs the CUDA library and an sm_100 device and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = [
    "Error", "DimensionError", "ArgumentError", "BreakdownError", "SingularFactorError",
    "ZeroMatrixError", "RankDeficiencyError", "CudaError", "NcclError", "PanelPlan", "Context",
    "default_context", "tsqr_qless", "tsqr_stage1", "block_qless_qr", "tsmttsm", "tsmRttsmR",
    "tsmmttsmm", "cholesky", "eigh_small", "cholqr2", "svqb_pass", "svqb2", "reconstruct_q",
    "solve_lstsq", "default_tsqr_plan", "default_gram_plan", "sign_normalize", "library_path",
    "load_library", "ABI_SYMBOLS",
]

PKG_DIR = Path(__file__).resolve().parent
LIB_NAME = "libskinnyqr_b200.so"

I64 = C.c_int64
DP = C.POINTER(C.c_double)
# sqb_allgather_fn (include/skinnyqr_b200.h): user, d_send, d_recv, count -> status
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)
TSQR_KERNELS = {"auto": -1, "thread": 0, "fold": 1, "mma": 2}


# ---- exception hierarchy (reference include/skinnyqr/types.hpp:11-77) -------------------------
class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class ArgumentError(Error):
    pass


class BreakdownError(Error):
    def __init__(self, what, index):
        super().__init__(what)
        self.pivot_index = index


class ZeroMatrixError(Error):
    pass


class SingularFactorError(Error):
    def __init__(self, what, index):
        super().__init__(what)
        self.diagonal_index = index


class RankDeficiencyError(Error):
    def __init__(self, what, index):
        super().__init__(what)
        self.diagonal_index = index


class CudaError(Error):
    """No sm_100 device, the CUDA library is missing, or a CUDA call failed."""


class NcclError(Error):
    pass


SQB_OK = 0
METHODS = {"tsqr": 0, "cholqr2": 1, "svqb2": 2}


@dataclass
class PanelPlan:
    """reference include/skinnyqr/plan.hpp:13-38.  On the GPU num_blocks is the CTA count of the
    streaming kernel and panel_rows the block alignment; 0 selects the device default."""

    num_blocks: int = 0
    panel_rows: int = 0
    deterministic: bool = True

    def validate(self):
        if self.num_blocks < 1 or self.panel_rows < 1:
            raise ArgumentError("PanelPlan: num_blocks and panel_rows must be >= 1")

    def rows_per_block(self, m):
        kb = self.num_blocks * self.panel_rows
        return ((m + kb - 1) // kb) * self.panel_rows

    def block_begin(self, m, block):
        return min(block * self.rows_per_block(m), m)

    def block_end(self, m, block):
        return min((block + 1) * self.rows_per_block(m), m)


# ---- library loading ---------------------------------------------------------------------------
ABI_SYMBOLS = [
    "sqb_create", "sqb_destroy", "sqb_set_stream", "sqb_use_own_stream", "sqb_get_stream", "sqb_sync",
    "sqb_set_tsqr_kernel", "sqb_set_host_slab_bytes", "sqb_copy_h2d", "sqb_copy_d2h", "sqb_device_alloc",
    "sqb_device_free",
    "sqb_last_error_index", "sqb_status_string", "sqb_device_sm_count", "sqb_launch_count",
    "sqb_default_tsqr_plan", "sqb_default_gram_plan",
    "sqb_tsqr_qless_dev", "sqb_tsqr_stage1_dev", "sqb_block_qless_qr_dev", "sqb_tsmttsm_dev",
    "sqb_tsmRttsmR_dev", "sqb_tsmmttsmm_dev", "sqb_cholesky_dev", "sqb_eigh_small_dev",
    "sqb_cholqr2_dev", "sqb_svqb2_dev", "sqb_svqb_pass_dev", "sqb_reconstruct_q_dev",
    "sqb_solve_lstsq_dev",
    "sqb_tsqr_qless_host", "sqb_tsqr_stage1_host", "sqb_block_qless_qr_host", "sqb_tsmttsm_host",
    "sqb_tsmRttsmR_host", "sqb_tsmmttsmm_host", "sqb_cholesky_host", "sqb_eigh_small_host",
    "sqb_cholqr2_host", "sqb_svqb_pass_host", "sqb_svqb2_host", "sqb_reconstruct_q_host",
    "sqb_solve_lstsq_host",
    "sqb_fill_gaussian_dev", "sqb_generate_dev",
    "sqb_attach_nccl", "sqb_nccl_unique_id", "sqb_init_nccl", "sqb_set_allgather", "sqb_tsqr_local_dev",
    "sqb_tsqr_combine_dev", "sqb_gram_combine_dev", "sqb_tsqr_qless_sharded_dev", "sqb_tsqr_qless_sharded_host",
    "sqb_cholqr2_sharded_dev", "sqb_svqb2_sharded_dev", "sqb_solve_lstsq_sharded_dev",
]

_lib = None


def library_path() -> Path:
    return PKG_DIR / LIB_NAME


def load_library():
    """Load libskinnyqr_b200.so (built by paper_2603_20889_b200/build.py).  Never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise CudaError(f"{path} is missing: run `python -m paper_2603_20889_b200.build` "
                        "(there is no CPU fallback)")
    lib = C.CDLL(str(path))
    lib.sqb_status_string.restype = C.c_char_p
    lib.sqb_last_error_index.restype = C.c_longlong
    lib.sqb_launch_count.restype = C.c_longlong
    lib.sqb_get_stream.restype = C.c_void_p
    for name in ABI_SYMBOLS:
        getattr(lib, name)  # AttributeError here = ABI drift
    _lib = lib
    return lib


def _raise(status, index, where):
    msg = f"{where}: {load_library().sqb_status_string(status).decode()}"
    if status == -1:
        raise DimensionError(msg)
    if status == -2:
        raise ArgumentError(msg)
    if status == -3:
        raise BreakdownError(msg, index)
    if status == -4:
        raise SingularFactorError(msg, index)
    if status == -5:
        raise ZeroMatrixError(msg)
    if status == -6:
        raise RankDeficiencyError(msg, index)
    if status == -7:
        raise Error(msg)
    if status == -9:
        raise NcclError(msg)
    raise CudaError(msg)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _hp(a):
    return a.ctypes.data_as(DP)


def _fmat(a):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError("expected a 2-D matrix")
    return np.asfortranarray(a)


def _plan(plan):
    if plan is None:
        return 0, 0
    if isinstance(plan, PanelPlan):
        return int(plan.num_blocks), int(plan.panel_rows)
    k, b = plan
    return int(k), int(b)


class Context:
    """One per GPU/thread: stream, workspaces, device status word (C ABI sqb_context)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.handle = C.c_void_p()
        st = self.lib.sqb_create(C.byref(self.handle), C.c_int(device))
        if st != SQB_OK:
            self.handle = None
            _raise(st, -1, "sqb_create")
        self.device = device
        self.host_slab_bytes = 256 << 20
        self._torch_stream = -1  # cudaStream_t of torch's current stream once device tensors are used

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sqb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- bookkeeping
    @property
    def sm_count(self):
        return int(self.lib.sqb_device_sm_count(self.handle))

    @property
    def launch_count(self):
        return int(self.lib.sqb_launch_count(self.handle))

    def set_stream(self, cuda_stream_ptr):
        """Enqueue on a caller-owned cudaStream_t (0 / None = the CUDA default stream)."""
        self._check(self.lib.sqb_set_stream(self.handle, C.c_void_p(cuda_stream_ptr or None)), "set_stream")

    def use_own_stream(self):
        self._torch_stream = -1
        self._check(self.lib.sqb_use_own_stream(self.handle), "use_own_stream")

    def use_torch_stream(self):
        import torch
        self._torch_stream = torch.cuda.current_stream(self.device).cuda_stream
        self.set_stream(self._torch_stream)

    def synchronize(self, where="synchronize"):
        self._check(self.lib.sqb_sync(self.handle), where)

    def _check(self, st, where):
        if st != SQB_OK:
            _raise(st, int(self.lib.sqb_last_error_index(self.handle)), where)

    def default_tsqr_plan(self, m, n):
        k, b = I64(0), I64(0)
        self._check(self.lib.sqb_default_tsqr_plan(self.handle, I64(m), I64(n), C.byref(k), C.byref(b)),
                    "default_tsqr_plan")
        return PanelPlan(int(k.value), int(b.value), True)

    def default_gram_plan(self, m, n):
        k, b = I64(0), I64(0)
        self._check(self.lib.sqb_default_gram_plan(self.handle, I64(m), I64(n), C.byref(k), C.byref(b)),
                    "default_gram_plan")
        return PanelPlan(int(k.value), int(b.value), True)

    # -- device-side helpers (torch tensors are only memory handles here)
    def _follow_torch_stream(self):
        # device tensors are produced by torch kernels on torch's current stream: enqueue behind them
        # (an own stream would race with the producer); host-pointer calls keep the own stream
        import torch
        cur = torch.cuda.current_stream(self.device).cuda_stream
        if cur != self._torch_stream:
            self.set_stream(cur)
            self._torch_stream = cur

    def _dev(self, t):
        import torch
        if t.dtype != torch.float64 or not t.is_cuda:
            raise ArgumentError("device inputs must be float64 CUDA tensors")
        self._follow_torch_stream()
        if t.dim() == 1:
            return C.c_void_p(t.data_ptr()), t.shape[0], 1, max(t.shape[0], 1)
        m, n = t.shape
        s0, s1 = t.stride()
        if (m > 1 and s0 != 1) or (n > 1 and s1 < m):
            raise ArgumentError("device matrices must be column-major (stride (1, ld))")
        return C.c_void_p(t.data_ptr()), m, n, (s1 if n > 1 else max(m, 1))

    def _dev_square(self, t, n, what):
        """A secondary n x n device operand (R, B, C): float64, same device, packed column-major."""
        p, fm, fn_, fld = self._dev(t)
        if t.dim() != 2 or (fm, fn_) != (n, n):
            raise DimensionError(f"{what} must be n x n")
        if fld != n:
            raise ArgumentError(f"{what} must be a packed column-major n x n matrix (leading dimension n)")
        if t.device.index != self.device:
            raise ArgumentError(f"{what} lives on another device")
        return p

    def _dev_vector(self, t, m, what):
        """A device vector operand (rhs): float64, same device, unit stride, m entries."""
        import torch
        if not _is_torch(t) or t.dtype != torch.float64 or not t.is_cuda:
            raise ArgumentError(f"{what} must be a float64 CUDA tensor")
        if t.dim() != 1 or t.shape[0] != m:
            raise DimensionError(f"{what} must have {m} entries")
        if m > 1 and t.stride(0) != 1:
            raise ArgumentError(f"{what} must have unit stride")
        if t.device.index != self.device:
            raise ArgumentError(f"{what} lives on another device")
        return C.c_void_p(t.data_ptr())

    def set_tsqr_kernel(self, kind="auto"):
        """Force one TSQR kernel family ("thread", "fold", "mma") or return to the table ("auto")."""
        self._check(self.lib.sqb_set_tsqr_kernel(self.handle, C.c_int(TSQR_KERNELS[kind])), "set_tsqr_kernel")

    def set_host_slab_bytes(self, nbytes):
        self._check(self.lib.sqb_set_host_slab_bytes(self.handle, I64(int(nbytes))), "set_host_slab_bytes")
        self.host_slab_bytes = int(nbytes)

    def empty_matrix(self, m, n):
        """Column-major m x n float64 CUDA tensor (shape (m, n), stride (1, m))."""
        import torch
        return torch.empty((n, m), dtype=torch.float64, device=f"cuda:{self.device}").t()

    def _square(self, n):
        return self.empty_matrix(n, n)

    def _ptr(self, t):
        return C.c_void_p(t.data_ptr())

    # -- TSQR (tsqr.hpp:59-68)
    def tsqr_qless(self, x, plan=None):
        k, b = _plan(plan)
        if _is_torch(x):
            p, m, n, ld = self._dev(x)
            r = self._square(n)
            self._check(self.lib.sqb_tsqr_qless_dev(self.handle, p, I64(m), I64(n), I64(ld), I64(k), I64(b),
                                                    self._ptr(r)), "tsqr_qless")
            return r
        x = _fmat(x)
        m, n = x.shape
        r = np.zeros((n, n), order="F")
        self._check(self.lib.sqb_tsqr_qless_host(self.handle, _hp(x), I64(m), I64(n), I64(m), I64(k), I64(b),
                                                 _hp(r)), "tsqr_qless")
        return r

    def tsqr_stage1(self, x, plan=None):
        if _is_torch(x):
            p, m, n, ld = self._dev(x)
            pl = plan if plan is not None and _plan(plan)[0] > 0 else self.default_tsqr_plan(m, n)
            k, b = _plan(pl)
            y = self.empty_matrix(k * n, n)
            self._check(self.lib.sqb_tsqr_stage1_dev(self.handle, p, I64(m), I64(n), I64(ld), I64(k), I64(b),
                                                     self._ptr(y)), "tsqr_stage1")
            return y
        x = _fmat(x)
        m, n = x.shape
        pl = plan if plan is not None and _plan(plan)[0] > 0 else self.default_tsqr_plan(m, n)
        k, b = _plan(pl)
        y = np.zeros((k * n, n), order="F")
        self._check(self.lib.sqb_tsqr_stage1_host(self.handle, _hp(x), I64(m), I64(n), I64(m), I64(k), I64(b),
                                                  _hp(y)), "tsqr_stage1")
        return y

    def block_qless_qr(self, x, b=0):
        if _is_torch(x):
            p, m, n, ld = self._dev(x)
            r = self._square(n)
            self._check(self.lib.sqb_block_qless_qr_dev(self.handle, p, I64(m), I64(n), I64(ld), I64(b),
                                                        self._ptr(r)), "block_qless_qr")
            return r
        x = _fmat(x)
        m, n = x.shape
        r = np.zeros((n, n), order="F")
        self._check(self.lib.sqb_block_qless_qr_host(self.handle, _hp(x), I64(m), I64(n), I64(m), I64(b),
                                                     _hp(r)), "block_qless_qr")
        return r

    # -- Gram kernels (gram.hpp:12-21)
    def _gram(self, name, x, factor, plan):
        k, b = _plan(plan)
        if _is_torch(x):
            p, m, n, ld = self._dev(x)
            c = self._square(n)
            fn = getattr(self.lib, f"sqb_{name}_dev")
            if factor is None:
                st = fn(self.handle, p, I64(m), I64(n), I64(ld), I64(k), I64(b), self._ptr(c))
            else:
                fp = self._dev_square(factor, n, f"{name}: factor")
                st = fn(self.handle, p, I64(m), I64(n), I64(ld), fp, I64(k), I64(b), self._ptr(c))
            self._check(st, name)
            return c
        x = _fmat(x)
        m, n = x.shape
        c = np.zeros((n, n), order="F")
        fn = getattr(self.lib, f"sqb_{name}_host")
        if factor is None:
            st = fn(self.handle, _hp(x), I64(m), I64(n), I64(m), I64(k), I64(b), _hp(c))
        else:
            f = _fmat(factor)
            if f.shape != (n, n):
                raise DimensionError(f"{name}: factor must be n x n")
            st = fn(self.handle, _hp(x), I64(m), I64(n), I64(m), _hp(f), I64(k), I64(b), _hp(c))
        self._check(st, name)
        return c

    def tsmttsm(self, x, plan=None):
        return self._gram("tsmttsm", x, None, plan)

    def tsmRttsmR(self, x, r, plan=None):
        return self._gram("tsmRttsmR", x, r, plan)

    def tsmmttsmm(self, x, b, plan=None):
        return self._gram("tsmmttsmm", x, b, plan)

    # -- n x n factorisations and Gram-based drivers (gram_qr.hpp:37-59)
    def cholesky(self, c):
        if _is_torch(c):
            if c.dim() != 2 or c.shape[0] != c.shape[1]:
                raise DimensionError("cholesky: C must be square")
            n = c.shape[0]
            p = self._dev_square(c, n, "cholesky: C")
            r = self._square(n)
            self._check(self.lib.sqb_cholesky_dev(self.handle, p, I64(n), self._ptr(r)), "cholesky")
            return r
        c = _fmat(c)
        n = c.shape[0]
        r = np.zeros((n, n), order="F")
        self._check(self.lib.sqb_cholesky_host(self.handle, _hp(c), I64(n), _hp(r)), "cholesky")
        return r

    def eigh_small(self, c):
        c = _fmat(c)
        n = c.shape[0]
        vals, vecs = np.zeros(n), np.zeros((n, n), order="F")
        self._check(self.lib.sqb_eigh_small_host(self.handle, _hp(c), I64(n), _hp(vals), _hp(vecs)),
                    "eigh_small")
        return vals, vecs

    def cholqr2(self, x, plan=None):
        k, b = _plan(plan)
        if _is_torch(x):
            p, m, n, ld = self._dev(x)
            r = self._square(n)
            self._check(self.lib.sqb_cholqr2_dev(self.handle, p, I64(m), I64(n), I64(ld), I64(k), I64(b),
                                                 self._ptr(r)), "cholqr2")
            return r
        x = _fmat(x)
        m, n = x.shape
        r = np.zeros((n, n), order="F")
        self._check(self.lib.sqb_cholqr2_host(self.handle, _hp(x), I64(m), I64(n), I64(m), I64(k), I64(b),
                                              _hp(r)), "cholqr2")
        return r

    def svqb_pass(self, c):
        c = _fmat(c)
        n = c.shape[0]
        b, z, sg, rank = np.zeros((n, n), order="F"), np.zeros((n, n), order="F"), np.zeros(n), I64(0)
        self._check(self.lib.sqb_svqb_pass_host(self.handle, _hp(c), I64(n), _hp(b), _hp(z), _hp(sg),
                                                C.byref(rank)), "svqb_pass")
        return b, z, sg, int(rank.value)

    def svqb2(self, x, plan=None):
        k, b = _plan(plan)
        if _is_torch(x):
            import torch
            p, m, n, ld = self._dev(x)
            tr, z = self._square(n), self._square(n)
            sg = torch.empty(n, dtype=torch.float64, device=x.device)
            rank = torch.zeros(1, dtype=torch.int64, device=x.device)
            self._check(self.lib.sqb_svqb2_dev(self.handle, p, I64(m), I64(n), I64(ld), I64(k), I64(b),
                                               self._ptr(tr), self._ptr(z), self._ptr(sg), self._ptr(rank)),
                        "svqb2")
            return tr, z, sg, rank
        x = _fmat(x)
        m, n = x.shape
        tr, z = np.zeros((n, n), order="F"), np.zeros((n, n), order="F")
        sg, rank = np.zeros(n), I64(0)
        self._check(self.lib.sqb_svqb2_host(self.handle, _hp(x), I64(m), I64(n), I64(m), I64(k), I64(b),
                                            _hp(tr), _hp(z), _hp(sg), C.byref(rank)), "svqb2")
        return tr, z, sg, int(rank.value)

    def reconstruct_q(self, x, r):
        if _is_torch(x):
            p, m, n, ld = self._dev(x)
            rp = self._dev_square(r, n, "reconstruct_q: R")
            q = self.empty_matrix(m, n)
            self._check(self.lib.sqb_reconstruct_q_dev(self.handle, p, I64(m), I64(n), I64(ld), rp,
                                                       self._ptr(q), I64(m)), "reconstruct_q")
            return q
        x, r = _fmat(x), _fmat(r)
        m, n = x.shape
        if r.shape != (n, n):
            raise DimensionError("reconstruct_q: R must be n x n")
        q = np.zeros((m, n), order="F")
        self._check(self.lib.sqb_reconstruct_q_host(self.handle, _hp(x), I64(m), I64(n), I64(m), _hp(r),
                                                    _hp(q), I64(m)), "reconstruct_q")
        return q

    # -- least squares (lstsq.hpp:21)
    def solve_lstsq(self, a, rhs, method="tsqr"):
        meth = METHODS[method] if isinstance(method, str) else int(method)
        if _is_torch(a):
            import torch
            p, m, n, ld = self._dev(a)
            rp = self._dev_vector(rhs, m, "solve_lstsq: rhs")
            x = torch.empty(n, dtype=torch.float64, device=a.device)
            res = torch.empty(1, dtype=torch.float64, device=a.device)
            self._check(self.lib.sqb_solve_lstsq_dev(self.handle, p, I64(m), I64(n), I64(ld), rp,
                                                     C.c_int(meth), self._ptr(x), self._ptr(res)),
                        "solve_lstsq")
            return x, res
        a = _fmat(a)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        m, n = a.shape
        if rhs.shape != (m,):
            raise DimensionError("solve_lstsq: rhs length != rows of A")
        x, res = np.zeros(n), C.c_double(0.0)
        self._check(self.lib.sqb_solve_lstsq_host(self.handle, _hp(a), I64(m), I64(n), I64(m), _hp(rhs),
                                                  C.c_int(meth), _hp(x), C.byref(res)), "solve_lstsq")
        return x, float(res.value)

    # -- synthetic inputs on the device
    def fill_gaussian(self, m, n, seed=1234, row_offset=0, m_total=None, out=None):
        x = out if out is not None else self.empty_matrix(m, n)
        p, mm, nn, ld = self._dev(x)
        self._check(self.lib.sqb_fill_gaussian_dev(self.handle, p, I64(m), I64(n), I64(ld), C.c_uint64(seed),
                                                   I64(row_offset), I64(m_total if m_total else m)),
                    "fill_gaussian")
        return x

    def generate(self, m, n, kappa, seed=42, linear=False, out=None):
        x = out if out is not None else self.empty_matrix(m, n)
        p, mm, nn, ld = self._dev(x)
        self._check(self.lib.sqb_generate_dev(self.handle, p, I64(m), I64(n), I64(ld), C.c_double(kappa),
                                              C.c_int(int(linear)), C.c_uint64(seed)), "generate")
        return x

    # -- multi-GPU
    def nccl_unique_id(self) -> bytes:
        buf = C.create_string_buffer(128)
        self._check(self.lib.sqb_nccl_unique_id(buf), "nccl_unique_id")
        return buf.raw

    def init_nccl(self, unique_id: bytes, rank: int, world: int):
        self._check(self.lib.sqb_init_nccl(self.handle, C.c_char_p(unique_id), C.c_int(rank), C.c_int(world)),
                    "init_nccl")

    def set_allgather(self, gather, rank: int, world: int):
        """Route the n x n exchange of the sharded drivers through `gather(d_send, d_recv, count)`
        (integer device addresses; return 0 on success) instead of NCCL - see sharding.TorchExchange."""
        def _cb(_user, send, recv, count):
            try:
                return int(gather(send, recv, int(count)) or 0)
            except Exception:  # an exception must not unwind through the C frames
                import traceback
                traceback.print_exc()
                return 1
        self._gather_cb = ALLGATHER_FN(_cb)  # keep the thunk alive as long as the context uses it
        self._check(self.lib.sqb_set_allgather(self.handle, self._gather_cb, None, C.c_int(rank), C.c_int(world)),
                    "set_allgather")

    def copy_d2h(self, host_array, dev_ptr):
        self._check(self.lib.sqb_copy_d2h(self.handle, host_array.ctypes.data_as(C.c_void_p), C.c_void_p(dev_ptr),
                                          I64(host_array.nbytes)), "copy_d2h")

    def copy_h2d(self, dev_ptr, host_array):
        self._check(self.lib.sqb_copy_h2d(self.handle, C.c_void_p(dev_ptr), host_array.ctypes.data_as(C.c_void_p),
                                          I64(host_array.nbytes)), "copy_h2d")

    def tsqr_local(self, x):
        """This rank's un-normalised triangle (first half of the sharded TSQR)."""
        p, m, n, ld = self._dev(x)
        r = self._square(n)
        self._check(self.lib.sqb_tsqr_local_dev(self.handle, p, I64(m), I64(n), I64(ld), self._ptr(r)), "tsqr_local")
        return r

    def _gathered(self, blocks, what):
        """(world, n, n) stack of column-major n x n blocks -> contiguous device buffer."""
        import torch
        if _is_torch(blocks):
            g = blocks
        else:
            g = torch.stack([b.t().contiguous() for b in blocks])  # each block column-major in memory
        if g.dim() != 3 or g.shape[1] != g.shape[2] or not g.is_contiguous():
            raise DimensionError(f"{what}: expected world contiguous n x n blocks")
        if g.dtype != torch.float64 or not g.is_cuda or g.device.index != self.device:
            raise ArgumentError(f"{what}: blocks must be float64 CUDA tensors on this device")
        self._follow_torch_stream()
        return g, g.shape[0], g.shape[1]

    def tsqr_combine(self, blocks):
        """Stage 2 over gathered triangles (list of n x n device tensors in rank order)."""
        g, world, n = self._gathered(blocks, "tsqr_combine")
        r = self._square(n)
        self._check(self.lib.sqb_tsqr_combine_dev(self.handle, self._ptr(g), I64(world), I64(n), self._ptr(r)),
                    "tsqr_combine")
        return r

    def gram_combine(self, blocks):
        """Sum of gathered Gram partials in ascending rank order."""
        g, world, n = self._gathered(blocks, "gram_combine")
        c = self._square(n)
        self._check(self.lib.sqb_gram_combine_dev(self.handle, self._ptr(g), I64(world), I64(n), self._ptr(c)),
                    "gram_combine")
        return c

    def tsqr_qless_sharded(self, x):
        p, m, n, ld = self._dev(x)
        r = self._square(n)
        self._check(self.lib.sqb_tsqr_qless_sharded_dev(self.handle, p, I64(m), I64(n), I64(ld), self._ptr(r)),
                    "tsqr_qless_sharded")
        return r

    def tsqr_qless_sharded_host(self, x):
        """Host slab of this rank in, host R out (slab ring + exchange)."""
        x = _fmat(x)
        m, n = x.shape
        r = np.zeros((n, n), order="F")
        self._check(self.lib.sqb_tsqr_qless_sharded_host(self.handle, _hp(x), I64(m), I64(n), I64(m), _hp(r)),
                    "tsqr_qless_sharded_host")
        return r

    def cholqr2_sharded(self, x):
        p, m, n, ld = self._dev(x)
        r = self._square(n)
        self._check(self.lib.sqb_cholqr2_sharded_dev(self.handle, p, I64(m), I64(n), I64(ld), self._ptr(r)),
                    "cholqr2_sharded")
        return r

    def svqb2_sharded(self, x):
        import torch
        p, m, n, ld = self._dev(x)
        tr, z = self._square(n), self._square(n)
        sg = torch.empty(n, dtype=torch.float64, device=x.device)
        rank = torch.zeros(1, dtype=torch.int64, device=x.device)
        self._check(self.lib.sqb_svqb2_sharded_dev(self.handle, p, I64(m), I64(n), I64(ld), self._ptr(tr),
                                                   self._ptr(z), self._ptr(sg), self._ptr(rank)),
                    "svqb2_sharded")
        return tr, z, sg, rank

    def solve_lstsq_sharded(self, a, rhs):
        import torch
        p, m, n, ld = self._dev(a)
        rp = self._dev_vector(rhs, m, "solve_lstsq_sharded: rhs")
        x = torch.empty(n, dtype=torch.float64, device=a.device)
        res = torch.empty(1, dtype=torch.float64, device=a.device)
        self._check(self.lib.sqb_solve_lstsq_sharded_dev(self.handle, p, I64(m), I64(n), I64(ld),
                                                         rp, self._ptr(x), self._ptr(res)),
                    "solve_lstsq_sharded")
        return x, res


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _ctx_for(x):
    if _is_torch(x):
        ctx = default_context(x.device.index or 0)
        ctx.use_torch_stream()
        return ctx
    return default_context(0)


def _call(x, name, args, check):
    """Module-level entry: host arrays are synchronous anyway; for device tensors `check=True`
    (the default) synchronises and raises the reference's exception for a numerical failure right
    here - with check=False the call stays asynchronous and failures surface at the next
    Context.synchronize()."""
    ctx = _ctx_for(x)
    out = getattr(ctx, name)(*args)
    if check and _is_torch(x):
        ctx.synchronize(name)
    return out


def sign_normalize(r):
    """reference types.cpp:8-14 (host n x n helper): negate row i from the diagonal on when
    R(i,i) < 0."""
    r = np.array(r, dtype=np.float64, order="F")
    for i in range(r.shape[0]):
        if r[i, i] < 0.0:
            r[i, i:] = -r[i, i:]
    return r


def default_tsqr_plan(m, n):
    return default_context().default_tsqr_plan(m, n)


def default_gram_plan(m, n):
    return default_context().default_gram_plan(m, n)


def tsqr_qless(x, plan=None, check=True):
    return _call(x, "tsqr_qless", (x, plan), check)


def tsqr_stage1(x, plan=None, check=True):
    return _call(x, "tsqr_stage1", (x, plan), check)


def block_qless_qr(x, b=0, check=True):
    return _call(x, "block_qless_qr", (x, b), check)


def tsmttsm(x, plan=None, check=True):
    return _call(x, "tsmttsm", (x, plan), check)


def tsmRttsmR(x, r, plan=None, check=True):
    return _call(x, "tsmRttsmR", (x, r, plan), check)


def tsmmttsmm(x, b, plan=None, check=True):
    return _call(x, "tsmmttsmm", (x, b, plan), check)


def cholesky(c, check=True):
    return _call(c, "cholesky", (c,), check)


def eigh_small(c):
    return default_context().eigh_small(c)


def cholqr2(x, plan=None, check=True):
    return _call(x, "cholqr2", (x, plan), check)


def svqb_pass(c):
    return default_context().svqb_pass(c)


def svqb2(x, plan=None, check=True):
    return _call(x, "svqb2", (x, plan), check)


def reconstruct_q(x, r, check=True):
    return _call(x, "reconstruct_q", (x, r), check)


def solve_lstsq(a, rhs, method="tsqr", check=True):
    return _call(a, "solve_lstsq", (a, rhs, method), check)
