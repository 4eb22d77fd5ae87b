"""B200-native exhaustive Gray-code search for the L_d norms of arXiv 2503.21596.

Thin ctypes binding over the C ABI of ``liblnorm.so`` (declared in
``include/lnorm.h``): argument marshalling only -- every step of the search
runs in the library's sm_100a kernels.  If the library is missing or no CUDA
device is present the calls raise; there is no CPU fallback.

    value, argmax = compute(M, d=1)                 # L_1      (Eq. 1)
    value, argmax = compute(M, d=1, with_marginals=True)   # L_marg (Eq. 2)
    value, argmax = compute(M, d=3)                 # L_3      (Eq. 6)
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

__all__ = [
    "LNormError", "load", "compute", "compute_device", "compute_reduced", "compute_batch", "compute_multi", "Comm",
    "compute_rank", "compute_rank_device", "torch_nccl_comm", "prefix_maxima", "unit_maxima",
    "walk_trace", "imma_l1", "gray_digit", "gray_change", "partition", "reduction_key", "key_decode", "last_stats", "status_string", "SYMBOLS", "plan",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LNORM_LIB") or os.path.join(_HERE, "liblnorm.so")   # LNORM_LIB: experiment builds

# every function include/lnorm.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "lnorm_status_string", "lnorm_version", "lnorm_compute", "lnorm_compute_device", "lnorm_compute_multi",
    "lnorm_comm_unique_id", "lnorm_comm_create", "lnorm_comm_nccl", "lnorm_comm_destroy", "lnorm_compute_rank",
    "lnorm_compute_rank_device",
    "lnorm_prefix_maxima", "lnorm_unit_maxima", "lnorm_walk_trace", "lnorm_gray_digit", "lnorm_gray_change", "lnorm_partition",
    "lnorm_reduction_key", "lnorm_key_decode",
    "lnorm_last_stats", "lnorm_plan", "lnorm_compute_sliced", "lnorm_compute_reduced", "lnorm_compute_batch",
    "lnorm_compute_checkpointed", "lnorm_imma_l1",
]

STATUS = {0: "OK", 1: "EINVAL", 2: "EOVERFLOW", 3: "ETOOLARGE", 4: "ENODEV", 5: "ECUDA", 6: "ENCCL", 7: "ENOMEM",
          8: "EINTERNAL"}


class LNormError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{what}: {self.name} ({_status_text(status)})")


class Stats(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32), ("transposed", ctypes.c_int32),
        ("prefix_digits", ctypes.c_int32), ("suffix_digits", ctypes.c_int32), ("d", ctypes.c_int32),
        ("units", ctypes.c_int64), ("units_total", ctypes.c_int64), ("steps", ctypes.c_double),
        ("column_updates", ctypes.c_double), ("walk_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
        ("launches", ctypes.c_int32), ("variant", ctypes.c_int32), ("block_threads", ctypes.c_int32),
        ("grid_blocks", ctypes.c_int32), ("paired_rows", ctypes.c_int32), ("packed_units", ctypes.c_int32),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32), ("transposed", ctypes.c_int32),
        ("d_walked", ctypes.c_int32), ("prefix_digits", ctypes.c_int32), ("suffix_digits", ctypes.c_int32),
        ("variant", ctypes.c_int32), ("packed_ok", ctypes.c_int32), ("units", ctypes.c_int64),
        ("steps", ctypes.c_double), ("lanes_per_unit", ctypes.c_int32), ("words", ctypes.c_int32),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


VARIANTS = {0: "bin_int32", 1: "ld_int32", 2: "generic", 3: "bin_packed16", 4: "ld_packed16", 5: "bin_pair16", 6: "ld_pair16",
            7: "bin_u8", 8: "ld_u8"}

_lock = threading.Lock()
_lib = None


def load():
    """Load liblnorm.so (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -m paper_2503_21596_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        i32p, i8p, i64p = P(i32), P(ctypes.c_int8), P(i64)
        vp = ctypes.c_void_p
        sig = {
            "lnorm_status_string": ([ctypes.c_int], ctypes.c_char_p),
            "lnorm_version": ([], i32),
            "lnorm_compute": ([i32p, i32, i32, i32, i32, i64p, i8p], ctypes.c_int),
            "lnorm_compute_device": ([vp, i32, i32, i32, i32, vp, i64p, i8p], ctypes.c_int),
            "lnorm_compute_multi": ([i32p, i32, i32, i32, i32, i32, i32p, i64p, i8p], ctypes.c_int),
            "lnorm_comm_unique_id": ([P(ctypes.c_uint8)], ctypes.c_int),
            "lnorm_comm_create": ([P(ctypes.c_uint8), i32, i32, i32, P(vp)], ctypes.c_int),
            "lnorm_comm_nccl": ([vp, P(vp)], ctypes.c_int),
            "lnorm_comm_destroy": ([vp], ctypes.c_int),
            "lnorm_compute_rank": ([i32p, i32, i32, i32, i32, vp, i32, i32, vp, i64p, i8p], ctypes.c_int),
            "lnorm_compute_rank_device": ([vp, i32, i32, i32, i32, vp, i32, i32, vp, i64p, i8p], ctypes.c_int),
            "lnorm_prefix_maxima": ([i32p, i32, i32, i32, i32, i32, i8p, i64, i64p], ctypes.c_int),
            "lnorm_unit_maxima": ([i32p, i32, i32, i32, i32, i32, P(u64), i64, i32p], ctypes.c_int),
            "lnorm_walk_trace": ([i32p, i32, i32, i32, i32, i32, i8p, i64, i64p, i8p], ctypes.c_int),
            "lnorm_gray_digit": ([i32, i32, u64], i32),
            "lnorm_gray_change": ([i32, u64, i32p, i32p, i32p], ctypes.c_int),
            "lnorm_partition": ([u64, i64, i64, i64p, i64p], ctypes.c_int),
            "lnorm_reduction_key": ([i32, ctypes.c_uint32], u64),
            "lnorm_key_decode": ([u64, i32p, P(ctypes.c_uint32)], ctypes.c_int),
            "lnorm_last_stats": ([P(Stats)], ctypes.c_int),
            "lnorm_compute_checkpointed": ([i32p, i32, i32, i32, i32, ctypes.c_char_p, i64, i32, i64p, i8p, i32p, i64p],
                                           ctypes.c_int),
            "lnorm_compute_batch": ([i32p, i32, i32, i32, i32, i32, i64p, i8p], ctypes.c_int),
            "lnorm_compute_reduced": ([i32p, i32, i32, i32, i32, i64p, i8p, i32p], ctypes.c_int),
            "lnorm_compute_sliced": ([i32p, i32, i32, i32, i32, i32, i64p, i8p], ctypes.c_int),
            "lnorm_plan": ([i32p, i32, i32, i32, i32, i32, P(PlanInfo)], ctypes.c_int),
            "lnorm_imma_l1": ([i32p, i32, i32, u64, u64, i64p, i8p, P(u64), P(ctypes.c_double)], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
        return lib


def _status_text(status: int) -> str:
    try:
        return load().lnorm_status_string(status).decode()
    except Exception:
        return STATUS.get(status, "?")


def status_string(status: int) -> str:
    return _status_text(status)


def _check(rc: int, what: str):
    if rc != 0:
        raise LNormError(rc, what)


_I32 = np.iinfo(np.int32)


def _int32(M, ndim: int, what: str):
    """Exact int32 copy of an integer array: non-integer dtypes and out-of-range entries raise
    (never a silent wrap or truncation, which would search a different matrix)."""
    A = np.asarray(M)
    if A.ndim != ndim:
        raise ValueError(f"{what} must be a {ndim}-D integer array")
    if A.dtype == np.bool_ or not np.issubdtype(A.dtype, np.integer):
        raise TypeError(f"{what} must have an integer dtype, got {A.dtype}")
    if A.size and A.dtype != np.int32 and (int(A.min()) < _I32.min or int(A.max()) > _I32.max):
        raise LNormError(2, f"{what} has entries outside int32")
    return np.ascontiguousarray(A, dtype=np.int32)


def _mat(M):
    return _int32(M, 2, "M")


def _stream_ptr(stream):
    """cudaStream_t of a torch.cuda.Stream, a raw int handle, or None (library stream)."""
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(int(stream.cuda_stream))
    return ctypes.c_void_p(int(stream))


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def compute(M, d: int = 1, with_marginals: bool = False):
    """Exact L_1 / L_marg / L_d of the host matrix M on the current CUDA device.

    Returns (value, argmax) -- argmax is int8[n] (+-1 for d = 1, RGS labels for d >= 2)."""
    A = _mat(M)
    n, m = A.shape
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_compute(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), ctypes.byref(v),
                                _p(arg, ctypes.c_int8)), "lnorm_compute")
    return int(v.value), arg


def _dev_mat(M_dev):
    if len(M_dev.shape) != 2:
        raise ValueError("M_dev must be 2-D")
    dt = getattr(M_dev, "dtype", None)
    if dt is not None and "int32" not in str(dt):
        raise TypeError(f"M_dev must be int32, got {dt}")
    if hasattr(M_dev, "is_contiguous") and not M_dev.is_contiguous():
        raise ValueError("M_dev must be contiguous")
    return int(M_dev.shape[0]), int(M_dev.shape[1])


def compute_device(M_dev, d: int = 1, with_marginals: bool = False, stream=None):
    """Same as compute() for a matrix already resident on the device.

    M_dev: a CUDA tensor-like object with ``data_ptr()`` and ``shape`` (int32, contiguous).
    stream: torch.cuda.Stream / raw cudaStream_t / None; the search is enqueued on it, after
    the work the caller queued there (e.g. the kernel that produced M_dev)."""
    n, m = _dev_mat(M_dev)
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_compute_device(ctypes.c_void_p(M_dev.data_ptr()), n, m, d, int(with_marginals),
                                       _stream_ptr(stream), ctypes.byref(v), _p(arg, ctypes.c_int8)),
           "lnorm_compute_device")
    return int(v.value), arg


def compute_checkpointed(M, path: str, d: int = 1, with_marginals: bool = False, chunk_units: int = 0,
                         max_chunks: int = 0):
    """Resumable search: returns (done, value, argmax or None, units_done); state persisted in `path`."""
    A = _mat(M)
    n, m = A.shape
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    done = ctypes.c_int32()
    udone = ctypes.c_int64()
    _check(load().lnorm_compute_checkpointed(_p(A, ctypes.c_int32), n, m, d, int(with_marginals),
                                             os.fsencode(path), chunk_units, max_chunks, ctypes.byref(v),
                                             _p(arg, ctypes.c_int8), ctypes.byref(done), ctypes.byref(udone)),
           "lnorm_compute_checkpointed")
    return bool(done.value), int(v.value), (arg if done.value else None), int(udone.value)


def compute_batch(Ms, d: int = 1, with_marginals: bool = False):
    """Many same-shape matrices in one call (batched walk when the packed guard holds).

    Ms: array-like (batch, n, m).  Returns (values int64[batch], argmax int8[batch, n])."""
    A = _int32(Ms, 3, "Ms (batch, n, m)")
    b, n, m = A.shape
    vals = np.zeros(b, dtype=np.int64)
    args = np.zeros((b, n), dtype=np.int8)
    _check(load().lnorm_compute_batch(_p(A, ctypes.c_int32), b, n, m, d, int(with_marginals), _p(vals, ctypes.c_int64),
                                      _p(args, ctypes.c_int8)), "lnorm_compute_batch")
    return vals, args


def compute_reduced(M, d: int = 1, with_marginals: bool = False):
    """Exact norm after the paper's norm-preserving reductions (zero / proportional / sign-uniform lines).

    Returns (value, argmax, (n', m')); argmax attains the value on the ORIGINAL matrix."""
    A = _mat(M)
    n, m = A.shape
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    shape = np.zeros(2, dtype=np.int32)
    _check(load().lnorm_compute_reduced(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), ctypes.byref(v),
                                        _p(arg, ctypes.c_int8), _p(shape, ctypes.c_int32)), "lnorm_compute_reduced")
    return int(v.value), arg, (int(shape[0]), int(shape[1]))


def compute_sliced(M, slices: int, d: int = 1, with_marginals: bool = False):
    """Test hook: the multi-rank unit split walked slice by slice on one GPU (bit-identical results)."""
    A = _mat(M)
    n, m = A.shape
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_compute_sliced(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), slices,
                                       ctypes.byref(v), _p(arg, ctypes.c_int8)), "lnorm_compute_sliced")
    return int(v.value), arg


def compute_multi(M, d: int = 1, with_marginals: bool = False, devices=None):
    """One process, several GPUs: Algorithm-1 unit split + one NCCL all-reduce(max)."""
    A = _mat(M)
    n, m = A.shape
    if devices is None:
        import torch
        devices = list(range(torch.cuda.device_count()))
    ids = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_compute_multi(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), len(ids),
                                      _p(ids, ctypes.c_int32), ctypes.byref(v), _p(arg, ctypes.c_int8)),
           "lnorm_compute_multi")
    return int(v.value), arg


def compute_rank(M, nccl_comm, rank: int, world: int, d: int = 1, with_marginals: bool = False, stream=None):
    """One rank of a multi-GPU search (lnorm_compute_rank): `nccl_comm` is a caller-owned
    ncclComm_t (int / c_void_p, e.g. ``torch_nccl_comm()``) spanning `world` ranks, or None
    when world == 1.  Every rank returns the same (value, argmax)."""
    A = _mat(M)
    n, m = A.shape
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_compute_rank(_p(A, ctypes.c_int32), n, m, d, int(with_marginals),
                                     ctypes.c_void_p(int(nccl_comm) if nccl_comm else 0), rank, world,
                                     _stream_ptr(stream), ctypes.byref(v), _p(arg, ctypes.c_int8)),
           "lnorm_compute_rank")
    return int(v.value), arg


def compute_rank_device(M_dev, nccl_comm, rank: int, world: int, d: int = 1, with_marginals: bool = False,
                        stream=None):
    """compute_rank with the matrix resident on this rank's device."""
    n, m = _dev_mat(M_dev)
    v = ctypes.c_int64()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_compute_rank_device(ctypes.c_void_p(M_dev.data_ptr()), n, m, d, int(with_marginals),
                                            ctypes.c_void_p(int(nccl_comm) if nccl_comm else 0), rank, world,
                                            _stream_ptr(stream), ctypes.byref(v), _p(arg, ctypes.c_int8)),
           "lnorm_compute_rank_device")
    return int(v.value), arg


def torch_nccl_comm(group=None, device=None) -> int:
    """The ncclComm_t of a torch.distributed NCCL process group (caller-owned; torch keeps it).

    The group must have been initialised eagerly (``init_process_group(..., device_id=dev)``)
    or have run a collective on `device`."""
    import torch
    import torch.distributed as dist
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return int(pg._get_backend(dev)._comm_ptr())


class Comm:
    """A library-made NCCL communicator for one rank (lnorm_comm_create / _destroy).

    Rank 0 creates the 128-byte unique id with ``Comm.unique_id()`` and broadcasts it
    (e.g. ``torch.distributed.broadcast_object_list``).  uid=None is allowed for world 1
    and gives a handle without a communicator (no collective)."""

    def __init__(self, uid: bytes | None, rank: int, world: int, device: int):
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
        _check(load().lnorm_comm_create(buf, rank, world, device, ctypes.byref(self._h)), "lnorm_comm_create")
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(load().lnorm_comm_unique_id(buf), "lnorm_comm_unique_id")
        return bytes(buf)

    @property
    def nccl(self) -> int:
        """The ncclComm_t this handle owns (0 if none)."""
        out = ctypes.c_void_p()
        _check(load().lnorm_comm_nccl(self._h, ctypes.byref(out)), "lnorm_comm_nccl")
        return int(out.value or 0)

    def compute(self, M, d: int = 1, with_marginals: bool = False, stream=None):
        return compute_rank(M, self.nccl, self.rank, self.world, d=d, with_marginals=with_marginals, stream=stream)

    def compute_device(self, M_dev, d: int = 1, with_marginals: bool = False, stream=None):
        return compute_rank_device(M_dev, self.nccl, self.rank, self.world, d=d, with_marginals=with_marginals,
                                   stream=stream)

    def close(self):
        if self._h:
            load().lnorm_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def prefix_maxima(M, prefixes, d: int = 1, with_marginals: bool = False):
    """Per-prefix maxima (test hook): max over completions of each fixed prefix of rows 0..nfixed-1."""
    A = _mat(M)
    n, m = A.shape
    P = np.ascontiguousarray(np.asarray(prefixes, dtype=np.int8))
    if P.ndim != 2:
        raise ValueError("prefixes must be 2-D (count x nfixed)")
    out = np.zeros(P.shape[0], dtype=np.int64)
    _check(load().lnorm_prefix_maxima(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), P.shape[1],
                                      _p(P, ctypes.c_int8), P.shape[0], _p(out, ctypes.c_int64)),
           "lnorm_prefix_maxima")
    return out


def unit_maxima(M, prefix_digits: int, units, d: int = 1, with_marginals: bool = False):
    """Per-unit maxima in the library's unit coordinates (lnorm_unit_maxima)."""
    A = _mat(M)
    n, m = A.shape
    U = np.ascontiguousarray(np.asarray(units, dtype=np.uint64).reshape(-1))
    out = np.zeros(U.shape[0], dtype=np.int32)
    _check(load().lnorm_unit_maxima(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), prefix_digits,
                                    _p(U, ctypes.c_uint64), U.shape[0], _p(out, ctypes.c_int32)), "lnorm_unit_maxima")
    return out


def imma_l1(M, tile_begin: int = 0, tile_count: int = 0):
    """SURVEY §8(f4) experiment: max of Eq. (1) over tiles [tile_begin, tile_begin + tile_count) of
    512 strategies whose column sums come from one tcgen05 kind::i8 MMA each (tile_count = 0: all
    tiles = the exact L_1 of M, rows as given).  Returns (value, argmax, strategies, kernel_ms)."""
    A = _mat(M)
    n, m = A.shape
    v, cnt, ms = ctypes.c_int64(), ctypes.c_uint64(), ctypes.c_double()
    arg = np.zeros(n, dtype=np.int8)
    _check(load().lnorm_imma_l1(_p(A, ctypes.c_int32), n, m, tile_begin, tile_count, ctypes.byref(v),
                                _p(arg, ctypes.c_int8), ctypes.byref(cnt), ctypes.byref(ms)), "lnorm_imma_l1")
    return int(v.value), arg, int(cnt.value), float(ms.value)


def walk_trace(M, prefix, d: int = 1, with_marginals: bool = False):
    """Per-step values and digits of the device walk of one unit (test hook)."""
    A = _mat(M)
    n, m = A.shape
    pre = np.ascontiguousarray(np.asarray(prefix, dtype=np.int8))
    base = 2 if d == 1 else d
    steps = base ** (n - len(pre))
    vals = np.zeros(steps, dtype=np.int64)
    digs = np.zeros((steps, n), dtype=np.int8)
    _check(load().lnorm_walk_trace(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), len(pre),
                                   _p(pre, ctypes.c_int8), steps, _p(vals, ctypes.c_int64),
                                   _p(digs, ctypes.c_int8)), "lnorm_walk_trace")
    return vals, digs


def gray_digit(d: int, i: int, j: int) -> int:
    return int(load().lnorm_gray_digit(d, i, j))


def gray_change(d: int, j: int):
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(load().lnorm_gray_change(d, j, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "lnorm_gray_change")
    return a.value, b.value, c.value


def reduction_key(value: int, unit: int) -> int:
    """The library's 8-byte max-reduction key (lnorm_reduction_key; csrc/common.cuh make_key)."""
    return int(load().lnorm_reduction_key(value, unit))


def key_decode(key: int):
    v, u = ctypes.c_int32(), ctypes.c_uint32()
    _check(load().lnorm_key_decode(key, ctypes.byref(v), ctypes.byref(u)), "lnorm_key_decode")
    return v.value, u.value


def partition(C: int, T: int, t: int):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(load().lnorm_partition(C, T, t, ctypes.byref(lo), ctypes.byref(hi)), "lnorm_partition")
    return lo.value, hi.value


def plan(M, d: int = 1, with_marginals: bool = False, world: int = 1) -> dict:
    """Host-only plan lnorm_compute would use (orientation, unit split, kernel variant)."""
    A = _mat(M)
    n, m = A.shape
    info = PlanInfo()
    _check(load().lnorm_plan(_p(A, ctypes.c_int32), n, m, d, int(with_marginals), world, ctypes.byref(info)),
           "lnorm_plan")
    out = info.as_dict()
    out["variant_name"] = VARIANTS.get(out["variant"], "?")
    return out


def last_stats() -> dict:
    s = Stats()
    _check(load().lnorm_last_stats(ctypes.byref(s)), "lnorm_last_stats")
    return s.as_dict()
