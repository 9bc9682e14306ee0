"""Python host mirror of libtoesplit.so.1 (B200 split-FFT block-Toeplitz MVM).

A thin ctypes binding of the C ABI declared in ``include/toesplit.h`` (the
reference interface, /root/reference/proj/include/toesplit.h) and
``include/toesplit_ext.h`` (B200 extensions). Names, argument meaning and
error behaviour follow the reference C API: every failing call raises
``TsError`` carrying the ``ts_status`` code and ``ts_last_error()`` detail.

The compute path is the in-tree CUDA library; there is no Python or CPU
fallback: if ``libtoesplit.so.1`` is missing, importing this module raises.
PyTorch is used only for device memory/streams in ``apply_device``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TSK_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("TSK_LIB") or os.path.join(HERE, "libtoesplit.so.1")

TS_OK = 0
TS_ERR_INVALID_ARGUMENT, TS_ERR_SHAPE, TS_ERR_SYMMETRY, TS_ERR_CAP_EXCEEDED = 1, 2, 3, 4
TS_ERR_RESOURCE, TS_ERR_IO, TS_ERR_LOGIC, TS_ERR_INTERNAL = 5, 6, 7, 8
SYM_GENERAL, SYM_SYMMETRIC, SYM_SKEW = 0, 1, 2
STORAGE_AUTO, STORAGE_FULL, STORAGE_COMPRESSED = -1, 0, 1
POLICY_LAZY, POLICY_PARALLEL = 0, 1
C128, C64 = 0, 1

# every symbol the public headers declare (checked by tests/test_abi_cpu.py)
REFERENCE_SYMBOLS = [
    "ts_version", "ts_status_name", "ts_last_error", "ts_generator_create",
    "ts_generator_random", "ts_generator_from_json_file", "ts_generator_to_json_file",
    "ts_generator_dims", "ts_generator_levels", "ts_generator_destroy", "ts_random_vector",
    "ts_operator_create_split", "ts_operator_create_embed", "ts_operator_apply",
    "ts_operator_dims", "ts_operator_levels", "ts_operator_kernel_elems",
    "ts_operator_save_kernel", "ts_operator_load_split", "ts_operator_destroy",
    "ts_naive_matvec", "ts_predict",
]
EXTENSION_SYMBOLS = [
    "ts_block_generator_create", "ts_block_generator_dyadic", "ts_block_generator_from_scalar",
    "ts_block_generator_components", "ts_block_generator_destroy", "ts_split_options_default",
    "ts_operator_create_split_ex", "ts_operator_apply_device", "ts_operator_apply_batch_device", "ts_operator_get_info",
    "ts_device_count", "ts_operator_profile_device", "ts_generator_get_lags",
    "ts_device_memory_stats", "ts_device_memory_reset_peak", "ts_operator_create_split_multi",
    "ts_comm_unique_id", "ts_comm_create", "ts_comm_destroy", "ts_operator_apply_device_comm",
    "ts_operator_create_embed_ex",
]
LAUNCHER_SYMBOLS = [
    "tsk_fwd_split", "tsk_inv_merge", "tsk_leaf_pair", "tsk_embed_generator", "tsk_embed_dyadic",
    "tsk_fold_axis", "tsk_mirror_check", "tsk_store_block", "tsk_convert", "tsk_embed_corner",
    "tsk_symbol_multiply", "tsk_embed_fold0", "tsk_block_symbol_multiply",
]


class TsMetrics(C.Structure):
    _fields_ = [("fft_forward", C.c_uint64), ("fft_inverse", C.c_uint64),
                ("diag_mults", C.c_uint64), ("phase_mults", C.c_uint64),
                ("peak_live_elems", C.c_int64), ("kernel_elems", C.c_uint64),
                ("apply_ns", C.c_uint64), ("precompute_ns", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TsPolicy(C.Structure):
    _fields_ = [("mode", C.c_int), ("task_budget", C.c_int32)]


class TsComplexity(C.Structure):
    _fields_ = [("d", C.c_int32), ("n", C.c_double), ("s", C.c_double), ("c_embed", C.c_double),
                ("c_split", C.c_double), ("r_c", C.c_double), ("r_c_asymptote", C.c_double),
                ("r_m", C.c_double), ("r_m_sym", C.c_double)]


class TsSplitOptions(C.Structure):
    _fields_ = [("precision", C.c_int32), ("storage", C.c_int32), ("device", C.c_int32),
                ("part", C.c_int32), ("nparts", C.c_int32), ("s0_re", C.c_double),
                ("s0_im", C.c_double)]


class TsOperatorInfo(C.Structure):
    _fields_ = [("d", C.c_int32), ("m", C.c_int32), ("n_unique", C.c_int32),
                ("precision", C.c_int32), ("storage", C.c_int32), ("is_embed", C.c_int32),
                ("device", C.c_int32), ("part", C.c_int32), ("nparts", C.c_int32),
                ("reserved", C.c_int32), ("elem_bytes", C.c_uint64),
                ("spectra_bytes", C.c_uint64), ("workspace_bytes", C.c_uint64),
                ("launches", C.c_uint64), ("table_bytes", C.c_uint64),
                ("cached_bytes", C.c_uint64), ("graph_replays", C.c_uint64),
                ("ndevices", C.c_int32), ("reserved2", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TsMemoryStats(C.Structure):
    _fields_ = [("live_bytes", C.c_uint64), ("peak_bytes", C.c_uint64),
                ("spectra_bytes", C.c_uint64), ("table_bytes", C.c_uint64),
                ("workspace_bytes", C.c_uint64), ("staging_bytes", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TsLaunchRecord(C.Structure):
    _fields_ = [("kind", C.c_int32), ("axis", C.c_int32), ("single_child", C.c_int32),
                ("reserved", C.c_int32), ("ms", C.c_double), ("alg_bytes", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python paper_2406_17981_b200/build.py` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.ts_version.restype = C.c_char_p
    L.ts_status_name.restype = C.c_char_p
    L.ts_last_error.restype = C.c_char_p
    L.ts_generator_create.argtypes = [C.c_int32, _i64p, _dp, C.c_int, C.POINTER(_vp)]
    L.ts_generator_random.argtypes = [C.c_int32, _i64p, C.c_uint64, C.c_double, C.c_int,
                                      C.POINTER(_vp)]
    L.ts_generator_from_json_file.argtypes = [C.c_char_p, C.POINTER(_vp)]
    L.ts_generator_to_json_file.argtypes = [_vp, C.c_char_p]
    L.ts_generator_dims.argtypes = [_vp]
    L.ts_generator_levels.argtypes = [_vp, _i64p]
    L.ts_generator_destroy.argtypes = [_vp]
    L.ts_random_vector.argtypes = [C.c_int32, _i64p, C.c_uint64, C.c_double, _dp]
    L.ts_operator_create_split.argtypes = [_vp, C.c_double, C.c_double, C.c_int, C.POINTER(_vp)]
    L.ts_operator_create_embed.argtypes = [_vp, C.c_double, C.c_double, C.c_int, C.POINTER(_vp)]
    L.ts_operator_apply.argtypes = [_vp, _dp, _dp, C.POINTER(TsPolicy), C.POINTER(TsMetrics)]
    L.ts_operator_dims.argtypes = [_vp]
    L.ts_operator_levels.argtypes = [_vp, _i64p]
    L.ts_operator_kernel_elems.argtypes = [_vp, C.POINTER(C.c_uint64)]
    L.ts_operator_save_kernel.argtypes = [_vp, C.c_char_p]
    L.ts_operator_load_split.argtypes = [C.c_char_p, C.POINTER(_vp)]
    L.ts_operator_destroy.argtypes = [_vp]
    L.ts_naive_matvec.argtypes = [_vp, _dp, _dp, C.c_int64]
    L.ts_predict.argtypes = [C.c_int32, C.c_double, C.POINTER(TsComplexity)]
    L.ts_block_generator_create.argtypes = [C.c_int32, _i64p, C.c_int32, C.c_int32,
                                            C.POINTER(C.c_int32), C.POINTER(_dp),
                                            C.POINTER(C.c_int32), C.POINTER(_vp)]
    L.ts_block_generator_dyadic.argtypes = [C.c_int32, _i64p, C.c_double, C.c_double, C.c_double,
                                            C.POINTER(_vp)]
    L.ts_block_generator_from_scalar.argtypes = [_vp, C.POINTER(_vp)]
    L.ts_generator_get_lags.argtypes = [_vp, _dp]
    L.ts_block_generator_components.argtypes = [_vp]
    L.ts_block_generator_destroy.argtypes = [_vp]
    L.ts_split_options_default.argtypes = [C.POINTER(TsSplitOptions)]
    L.ts_operator_create_split_ex.argtypes = [_vp, C.POINTER(TsSplitOptions), C.POINTER(_vp)]
    L.ts_operator_apply_device.argtypes = [_vp, _vp, _vp, _vp, C.POINTER(TsMetrics)]
    L.ts_operator_apply_batch_device.argtypes = [_vp, _vp, _vp, C.c_int64, _vp, C.POINTER(TsMetrics)]
    L.ts_operator_get_info.argtypes = [_vp, C.POINTER(TsOperatorInfo)]
    L.ts_device_count.restype = C.c_int32
    L.ts_operator_profile_device.argtypes = [_vp, _vp, _vp, _vp, C.POINTER(TsLaunchRecord),
                                             C.c_int32, C.POINTER(C.c_int32)]
    L.ts_operator_create_embed_ex.argtypes = [_vp, C.POINTER(TsSplitOptions), C.POINTER(_vp)]
    L.ts_device_memory_stats.argtypes = [C.c_int32, C.POINTER(TsMemoryStats)]
    L.ts_device_memory_reset_peak.argtypes = [C.c_int32]
    L.ts_operator_create_split_multi.argtypes = [_vp, C.POINTER(TsSplitOptions), C.c_int32,
                                                 C.POINTER(C.c_int32), C.POINTER(_vp)]
    L.ts_comm_unique_id.argtypes = [C.c_char_p]
    L.ts_comm_create.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_vp)]
    L.ts_comm_destroy.argtypes = [_vp]
    L.ts_operator_apply_device_comm.argtypes = [_vp, _vp, _vp, _vp, C.c_int32, C.c_int32, _vp,
                                                C.POINTER(TsMetrics)]
    return L


lib = _load()


class TsError(RuntimeError):
    def __init__(self, code: int, detail: str):
        name = lib.ts_status_name(code).decode()
        super().__init__(f"{name} ({code}): {detail}")
        self.code = code
        self.detail = detail


def _ok(st: int) -> None:
    if st != TS_OK:
        raise TsError(st, lib.ts_last_error().decode())


def version() -> str:
    return lib.ts_version().decode()


def device_count() -> int:
    return int(lib.ts_device_count())


def memory_stats(device: int = 0) -> dict:
    """The library's device-memory meter (ts_device_memory_stats)."""
    m = TsMemoryStats()
    _ok(lib.ts_device_memory_stats(device, C.byref(m)))
    return m.as_dict()


def reset_memory_peak(device: int = 0) -> None:
    _ok(lib.ts_device_memory_reset_peak(device))


class Comm:
    """ts_comm: a library-owned NCCL communicator, one rank per process
    (torchrun layout). Rank 0 calls unique_id() and ships the 128 bytes to the
    other ranks; every rank then constructs Comm(uid, nranks, rank, device)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _ok(lib.ts_comm_unique_id(buf))
        return buf.raw

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        h = _vp()
        _ok(lib.ts_comm_create(C.create_string_buffer(bytes(uid), 128), nranks, rank, device,
                               C.byref(h)))
        self._h = h
        self.nranks, self.rank, self.device = nranks, rank, device

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ts_comm_destroy(self._h)
        self._h = None

    __del__ = close


def _levels(levels):
    a = np.ascontiguousarray(levels, dtype=np.int64)
    return a, a.ctypes.data_as(_i64p)


def _cbuf(x, count=None):
    a = np.ascontiguousarray(x, dtype=np.complex128).reshape(-1)
    if count is not None and a.size != count:
        raise ValueError(f"expected {count} complex values, got {a.size}")
    return a, a.ctypes.data_as(_dp)


class Generator:
    """ts_generator: scalar per-level Toeplitz lags (ref generator.hpp:20-46)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def create(cls, levels, lags, symmetry=SYM_GENERAL):
        lv, lp = _levels(levels)
        la, ldp = _cbuf(lags)
        h = _vp()
        _ok(lib.ts_generator_create(len(lv), lp, ldp, symmetry, C.byref(h)))
        return cls(h)

    @classmethod
    def random(cls, levels, seed, variance=1.0, symmetry=SYM_GENERAL):
        lv, lp = _levels(levels)
        h = _vp()
        _ok(lib.ts_generator_random(len(lv), lp, seed, variance, symmetry, C.byref(h)))
        return cls(h)

    @classmethod
    def from_json_file(cls, path):
        h = _vp()
        _ok(lib.ts_generator_from_json_file(os.fsencode(path), C.byref(h)))
        return cls(h)

    def to_json_file(self, path):
        _ok(lib.ts_generator_to_json_file(self._h, os.fsencode(path)))

    @property
    def dims(self) -> int:
        return int(lib.ts_generator_dims(self._h))

    @property
    def levels(self):
        out = np.zeros(self.dims, np.int64)
        _ok(lib.ts_generator_levels(self._h, out.ctypes.data_as(_i64p)))
        return [int(v) for v in out]

    def lags(self):
        out = np.zeros(int(np.prod([2 * n - 1 for n in self.levels])), np.complex128)
        _ok(lib.ts_generator_get_lags(self._h, out.ctypes.data_as(_dp)))
        return out

    def naive_matvec(self, v, cap=4096):
        s = int(np.prod(self.levels))
        va, vp = _cbuf(v, s)
        y = np.zeros(s, np.complex128)
        _ok(lib.ts_naive_matvec(self._h, vp, y.ctypes.data_as(_dp), cap))
        return y

    def close(self):
        if self._h and lib is not None:
            lib.ts_generator_destroy(self._h)
        self._h = None

    __del__ = close


def random_vector(levels, seed, variance=1.0):
    lv, lp = _levels(levels)
    out = np.zeros(int(np.prod(lv)), np.complex128)
    _ok(lib.ts_random_vector(len(lv), lp, seed, variance, out.ctypes.data_as(_dp)))
    return out


def predict(d, n):
    c = TsComplexity()
    _ok(lib.ts_predict(d, n, C.byref(c)))
    return {k: getattr(c, k) for k, _ in c._fields_}


class BlockGenerator:
    """ts_block_generator (extension): m x m blocks, unique-component map and
    per-axis symmetry signs."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep

    @classmethod
    def create(cls, levels, m, comp_map, lags_list, axis_signs):
        lv, lp = _levels(levels)
        U = len(lags_list)
        cm = (C.c_int32 * (m * m))(*[int(v) for v in np.asarray(comp_map).reshape(-1)])
        arrs = [np.ascontiguousarray(l, dtype=np.complex128).reshape(-1) for l in lags_list]
        ptrs = (_dp * U)(*[a.ctypes.data_as(_dp) for a in arrs])
        sg = (C.c_int32 * (U * len(lv)))(*[int(v) for v in np.asarray(axis_signs).reshape(-1)])
        h = _vp()
        _ok(lib.ts_block_generator_create(len(lv), lp, m, U, cm, ptrs, sg, C.byref(h)))
        return cls(h)

    @classmethod
    def dyadic(cls, levels, k=2 * np.pi / 10, self_term=1 + 0.1j):
        lv, lp = _levels(levels)
        h = _vp()
        _ok(lib.ts_block_generator_dyadic(len(lv), lp, k, self_term.real, self_term.imag,
                                          C.byref(h)))
        return cls(h)

    @classmethod
    def from_scalar(cls, g: Generator):
        h = _vp()
        _ok(lib.ts_block_generator_from_scalar(g._h, C.byref(h)))
        return cls(h)

    @property
    def components(self):
        return int(lib.ts_block_generator_components(self._h))

    def close(self):
        if self._h and lib is not None:
            lib.ts_block_generator_destroy(self._h)
        self._h = None

    __del__ = close


class Operator:
    """ts_operator: split (device spectra) or full-embedding operator."""

    def __init__(self, handle):
        self._h = handle

    # -- constructors (ref toesplit.h:124-146 + extensions) ----------------
    @classmethod
    def split(cls, g: Generator, s0=0j, storage=STORAGE_AUTO):
        h = _vp()
        _ok(lib.ts_operator_create_split(g._h, s0.real, s0.imag, storage, C.byref(h)))
        return cls(h)

    @classmethod
    def embed(cls, g: Generator, s0=0j, storage=STORAGE_AUTO):
        h = _vp()
        _ok(lib.ts_operator_create_embed(g._h, s0.real, s0.imag, storage, C.byref(h)))
        return cls(h)

    @classmethod
    def split_ex(cls, bg: BlockGenerator, precision=C128, storage=STORAGE_AUTO, device=-1,
                 part=0, nparts=1, s0=0j):
        opt = TsSplitOptions()
        lib.ts_split_options_default(C.byref(opt))
        opt.precision, opt.storage, opt.device = precision, storage, device
        opt.part, opt.nparts, opt.s0_re, opt.s0_im = part, nparts, s0.real, s0.imag
        h = _vp()
        _ok(lib.ts_operator_create_split_ex(bg._h, C.byref(opt), C.byref(h)))
        return cls(h)

    @classmethod
    def embed_ex(cls, bg: BlockGenerator, precision=C128, storage=STORAGE_AUTO, device=-1, s0=0j):
        """Full circulant-embedding operator for block generators on this
        library's FFT passes (ts_operator_create_embed_ex)."""
        opt = TsSplitOptions()
        lib.ts_split_options_default(C.byref(opt))
        opt.precision, opt.storage, opt.device = precision, storage, device
        opt.s0_re, opt.s0_im = s0.real, s0.imag
        h = _vp()
        _ok(lib.ts_operator_create_embed_ex(bg._h, C.byref(opt), C.byref(h)))
        return cls(h)

    @classmethod
    def split_multi(cls, bg: BlockGenerator, devices, precision=C128, storage=STORAGE_AUTO, s0=0j):
        """One operator over several GPUs (ts_operator_create_split_multi):
        branch partition, x broadcast and NCCL reduce inside the library."""
        opt = TsSplitOptions()
        lib.ts_split_options_default(C.byref(opt))
        opt.precision, opt.storage, opt.s0_re, opt.s0_im = precision, storage, s0.real, s0.imag
        devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        h = _vp()
        _ok(lib.ts_operator_create_split_multi(bg._h, C.byref(opt), len(devices), devs, C.byref(h)))
        return cls(h)

    @classmethod
    def load_split(cls, path):
        h = _vp()
        _ok(lib.ts_operator_load_split(os.fsencode(path), C.byref(h)))
        return cls(h)

    # -- queries ------------------------------------------------------------
    @property
    def dims(self):
        return int(lib.ts_operator_dims(self._h))

    @property
    def levels(self):
        out = np.zeros(self.dims, np.int64)
        _ok(lib.ts_operator_levels(self._h, out.ctypes.data_as(_i64p)))
        return [int(v) for v in out]

    @property
    def kernel_elems(self):
        v = C.c_uint64()
        _ok(lib.ts_operator_kernel_elems(self._h, C.byref(v)))
        return int(v.value)

    def info(self):
        i = TsOperatorInfo()
        _ok(lib.ts_operator_get_info(self._h, C.byref(i)))
        return i.as_dict()

    def save_kernel(self, path):
        _ok(lib.ts_operator_save_kernel(self._h, os.fsencode(path)))

    # -- apply ---------------------------------------------------------------
    def apply(self, v, policy=None, metrics=False, out=None):
        """Host apply through ts_operator_apply (interleaved doubles). out: an
        optional complex128 array to write y into (reused across calls)."""
        inf = self.info()
        count = int(np.prod(self.levels)) * inf["m"]
        va, vp = _cbuf(v, count)
        if out is None:
            y = np.zeros(count, np.complex128)
        else:
            y = out
            if y.dtype != np.complex128 or y.size != count or not y.flags.c_contiguous:
                raise ValueError(f"out must be a contiguous complex128 array of {count} values")
        m = TsMetrics()
        pol = None
        if policy is not None:
            pol = TsPolicy(policy[0], policy[1])
        _ok(lib.ts_operator_apply(self._h, vp, y.ctypes.data_as(_dp),
                                  C.byref(pol) if pol is not None else None, C.byref(m)))
        return (y, m.as_dict()) if metrics else y

    def _check_device(self, x, y, nrhs=1):
        """x, y: contiguous device tensors of the operator's precision holding
        nrhs * m * prod(levels) elements on the operator's device (raises
        ValueError otherwise: the C ABI takes raw pointers)."""
        import torch

        inf = self.info()
        want = torch.complex64 if inf["precision"] == C64 else torch.complex128
        count = int(np.prod(self.levels)) * inf["m"] * int(nrhs)
        for name, t in (("x", x), ("y", y)):
            if not isinstance(t, torch.Tensor) or not t.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor")
            if t.device.index != inf["device"]:
                raise ValueError(f"{name} is on cuda:{t.device.index}, the operator on cuda:{inf['device']}")
            if t.dtype != want:
                raise ValueError(f"{name} must be {want} for this operator, got {t.dtype}")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            if t.numel() != count:
                raise ValueError(f"{name} must hold {count} elements, got {t.numel()}")

    def apply_device(self, x, y, stream=None, metrics=False):
        """y = T x on device tensors (torch complex64/complex128, contiguous,
        m * prod(levels) elements). stream: torch.cuda.Stream or None
        (current stream)."""
        import torch

        self._check_device(x, y)
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        m = TsMetrics()
        _ok(lib.ts_operator_apply_device(self._h, C.c_void_p(x.data_ptr()),
                                         C.c_void_p(y.data_ptr()),
                                         C.c_void_p(stream.cuda_stream), C.byref(m)))
        return m.as_dict() if metrics else None

    def apply_batch_device(self, x, y, nrhs, stream=None, metrics=False):
        """nrhs vectors back to back in x (and y), each as for apply_device."""
        import torch

        self._check_device(x, y, nrhs)
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        m = TsMetrics()
        _ok(lib.ts_operator_apply_batch_device(self._h, C.c_void_p(x.data_ptr()),
                                               C.c_void_p(y.data_ptr()), int(nrhs),
                                               C.c_void_p(stream.cuda_stream), C.byref(m)))
        return m.as_dict() if metrics else None

    def apply_device_comm(self, comm: "Comm", x, y, root=0, bcast_x=True, stream=None,
                          metrics=False):
        """Collective apply of a partition operator (part = rank): x broadcast
        from root, partials summed onto root's y (NCCL inside the library)."""
        import torch

        self._check_device(x, y)
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        m = TsMetrics()
        _ok(lib.ts_operator_apply_device_comm(self._h, comm._h, C.c_void_p(x.data_ptr()),
                                              C.c_void_p(y.data_ptr()), int(root), int(bool(bcast_x)),
                                              C.c_void_p(stream.cuda_stream), C.byref(m)))
        return m.as_dict() if metrics else None

    def profile_device(self, x, y, stream=None):
        """Per-launch device times (CUDA events) and algorithmic bytes."""
        import torch

        self._check_device(x, y)
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        cap = 4096
        recs = (TsLaunchRecord * cap)()
        cnt = C.c_int32()
        _ok(lib.ts_operator_profile_device(self._h, C.c_void_p(x.data_ptr()),
                                           C.c_void_p(y.data_ptr()),
                                           C.c_void_p(stream.cuda_stream), recs, cap,
                                           C.byref(cnt)))
        return [recs[i].as_dict() for i in range(min(cnt.value, cap))]

    def close(self):
        if self._h and lib is not None:
            lib.ts_operator_destroy(self._h)
        self._h = None

    __del__ = close
