"""TEST INFRASTRUCTURE ONLY — the CPU oracle and the reference build.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product library
(``paper_2406_17981_b200``) never imports, links or calls anything here.

Two checkers live here:

* ``Oracle`` — ctypes binding of ``liboracle.so``, the plain-C restatement of
  the reference algorithm (``toesplit_oracle.c``; each function cites the
  reference file:line it follows).
* ``RefLib`` — ctypes binding of ``_ref/libtoesplit_ref.so``, the UNMODIFIED
  reference core + C ABI (``/root/reference/proj/src``) compiled by
  ``oracle/Makefile`` against the FFTW-API shim ("reference engine +
  substitute FFT"). Present wherever it was built (it travels to the GPU box
  as a prebuilt file; ``/root/reference`` itself does not).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtoesplit_ref.so")
REF_SRC = "/root/reference/proj"

_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

SYM_GENERAL, SYM_SYMMETRIC, SYM_SKEW = 0, 1, 2


def build(ref: bool = True) -> None:
    """Compile liboracle.so and (when the reference sources exist) _ref/."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _arr(x, dtype):
    return np.ascontiguousarray(x, dtype=dtype)


def _lv(levels):
    a = _arr(levels, np.int64)
    return a, a.ctypes.data_as(_i64p)


def _cd(x):
    """complex128 array -> contiguous interleaved double pointer."""
    a = np.ascontiguousarray(x, dtype=np.complex128)
    return a, a.ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: status {code}")
        self.code = code


def axis_signs(d: int, symmetry: int):
    return [0 if symmetry == SYM_GENERAL else (1 if symmetry == SYM_SYMMETRIC else -1)] * d


class Oracle:
    """Plain-C restatement of the reference split-FFT engine."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.orc_random_lags.argtypes = [C.c_int, _i64p, C.c_uint64, C.c_double, C.c_int, _dp]
        L.orc_random_vector.argtypes = [C.c_int, _i64p, C.c_uint64, C.c_double, _dp]
        L.orc_dyadic_lags.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.c_double, _dp]
        L.orc_dyadic_lags_slab.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_double,
                                           C.c_double, C.c_double, C.c_int64, C.c_int64, _dp]
        L.orc_validate_symmetry.argtypes = [C.c_int, _i64p, _dp, _ip]
        L.orc_spectra_elems.argtypes = [C.c_int, _i64p, C.c_int]
        L.orc_spectra_elems.restype = C.c_int64
        L.orc_precompute.argtypes = [C.c_int, _i64p, _dp, C.c_double, C.c_double, C.c_int, _ip, _dp]
        L.orc_split_apply.argtypes = [C.c_int, _i64p, _dp, C.c_int, _ip, _dp, _dp, _i64p]
        L.orc_split_apply_partial.argtypes = [C.c_int, _i64p, _dp, C.c_int, _ip, _dp, _dp,
                                              C.c_int, C.c_int]
        L.orc_embed_apply.argtypes = [C.c_int, _i64p, _dp, C.c_double, C.c_double, _dp, _dp]
        L.orc_naive_matvec.argtypes = [C.c_int, _i64p, _dp, _dp, _dp, C.c_int64]
        L.orc_fft_axis.argtypes = [C.c_int, _i64p, _dp, C.c_int, C.c_int]
        L.orc_phase_axis.argtypes = [C.c_int, _i64p, _dp, C.c_int, C.c_int]
        L.orc_embed_generator.argtypes = [C.c_int, _i64p, _dp, C.c_double, C.c_double, _dp]
        L.orc_predict.argtypes = [C.c_int, C.c_double, _dp]
        L.orc_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_splitmix_next.restype = C.c_uint64

    @staticmethod
    def _ok(st, what):
        if st != 0:
            raise OracleError(st, what)

    # -- instances --------------------------------------------------------
    def random_lags(self, levels, seed, variance=1.0, symmetry=SYM_GENERAL):
        lv, lp = _lv(levels)
        out = np.zeros(int(np.prod(2 * lv - 1)), np.complex128)
        self._ok(self.L.orc_random_lags(len(lv), lp, seed, variance, symmetry,
                                        out.ctypes.data_as(_dp)), "random_lags")
        return out

    def random_vector(self, levels, seed, variance=1.0):
        lv, lp = _lv(levels)
        out = np.zeros(int(np.prod(lv)), np.complex128)
        self._ok(self.L.orc_random_vector(len(lv), lp, seed, variance, out.ctypes.data_as(_dp)),
                 "random_vector")
        return out

    def dyadic_lags(self, levels, i, j, k=2 * np.pi / 10, self_term=1 + 0.1j, threads=1):
        lv, lp = _lv(levels)
        out = np.empty(int(np.prod(2 * lv - 1)), np.complex128)
        rows = int(2 * lv[0] - 1)
        if threads <= 1 or rows < 2:
            self._ok(self.L.orc_dyadic_lags(len(lv), lp, i, j, k, self_term.real, self_term.imag,
                                            out.ctypes.data_as(_dp)), "dyadic_lags")
            return out
        # axis-0 slabs on several threads (ctypes releases the GIL)
        from concurrent.futures import ThreadPoolExecutor

        cuts = np.linspace(0, rows, min(threads, rows) + 1).astype(np.int64)
        op = out.ctypes.data_as(_dp)

        def slab(t):
            return self.L.orc_dyadic_lags_slab(len(lv), lp, i, j, k, self_term.real,
                                               self_term.imag, int(cuts[t]), int(cuts[t + 1]), op)

        with ThreadPoolExecutor(len(cuts) - 1) as ex:
            for st in ex.map(slab, range(len(cuts) - 1)):
                self._ok(st, "dyadic_lags_slab")
        return out

    def validate_symmetry(self, levels, lags, signs):
        lv, lp = _lv(levels)
        la, ldp = _cd(lags)
        sg = _arr(signs, np.int32)
        return self.L.orc_validate_symmetry(len(lv), lp, ldp, sg.ctypes.data_as(_ip))

    # -- spectra ----------------------------------------------------------
    def spectra_elems(self, levels, compressed):
        lv, lp = _lv(levels)
        return int(self.L.orc_spectra_elems(len(lv), lp, int(compressed)))

    def precompute(self, levels, lags, s0=0j, compressed=False, signs=None):
        lv, lp = _lv(levels)
        la, ldp = _cd(lags)
        sg = _arr(signs if signs is not None else [0] * len(lv), np.int32)
        out = np.zeros(self.spectra_elems(levels, compressed), np.complex128)
        self._ok(self.L.orc_precompute(len(lv), lp, ldp, s0.real, s0.imag, int(compressed),
                                       sg.ctypes.data_as(_ip), out.ctypes.data_as(_dp)),
                 "precompute")
        return out

    # -- engines ----------------------------------------------------------
    def split_apply(self, levels, blocks, v, compressed=False, signs=None, counters=False):
        lv, lp = _lv(levels)
        ba, bp = _cd(blocks)
        va, vp = _cd(v)
        sg = _arr(signs if signs is not None else [0] * len(lv), np.int32)
        y = np.zeros_like(va)
        cnt = np.zeros(5, np.int64)
        self._ok(self.L.orc_split_apply(len(lv), lp, bp, int(compressed), sg.ctypes.data_as(_ip),
                                        vp, y.ctypes.data_as(_dp), cnt.ctypes.data_as(_i64p)),
                 "split_apply")
        return (y, cnt) if counters else y

    def split_apply_partial(self, levels, blocks, v, part, nparts, compressed=False, signs=None):
        lv, lp = _lv(levels)
        ba, bp = _cd(blocks)
        va, vp = _cd(v)
        sg = _arr(signs if signs is not None else [0] * len(lv), np.int32)
        y = np.zeros_like(va)
        self._ok(self.L.orc_split_apply_partial(len(lv), lp, bp, int(compressed),
                                                sg.ctypes.data_as(_ip), vp,
                                                y.ctypes.data_as(_dp), part, nparts),
                 "split_apply_partial")
        return y

    def embed_apply(self, levels, lags, v, s0=0j):
        lv, lp = _lv(levels)
        la, ldp = _cd(lags)
        va, vp = _cd(v)
        y = np.zeros_like(va)
        self._ok(self.L.orc_embed_apply(len(lv), lp, ldp, s0.real, s0.imag, vp,
                                        y.ctypes.data_as(_dp)), "embed_apply")
        return y

    def naive(self, levels, lags, v, cap=4096):
        lv, lp = _lv(levels)
        la, ldp = _cd(lags)
        va, vp = _cd(v)
        y = np.zeros_like(va)
        self._ok(self.L.orc_naive_matvec(len(lv), lp, ldp, vp, y.ctypes.data_as(_dp), cap),
                 "naive")
        return y

    def fft_axis(self, shape, t, axis, inverse=False):
        lv, lp = _lv(shape)
        a = np.array(t, dtype=np.complex128, copy=True).reshape(-1)
        self._ok(self.L.orc_fft_axis(len(lv), lp, a.ctypes.data_as(_dp), axis, int(inverse)),
                 "fft_axis")
        return a

    def phase_axis(self, shape, t, axis, conjugate=False):
        lv, lp = _lv(shape)
        a = np.array(t, dtype=np.complex128, copy=True).reshape(-1)
        self._ok(self.L.orc_phase_axis(len(lv), lp, a.ctypes.data_as(_dp), axis, int(conjugate)),
                 "phase_axis")
        return a

    def embed_generator(self, levels, lags, s0=0j):
        lv, lp = _lv(levels)
        la, ldp = _cd(lags)
        out = np.zeros(int(np.prod(2 * lv)), np.complex128)
        self._ok(self.L.orc_embed_generator(len(lv), lp, ldp, s0.real, s0.imag,
                                            out.ctypes.data_as(_dp)), "embed_generator")
        return out

    def predict(self, d, n):
        out = np.zeros(9)
        self._ok(self.L.orc_predict(d, n, out.ctypes.data_as(_dp)), "predict")
        return dict(zip(["d", "n", "s", "c_embed", "c_split", "r_c", "r_c_asymptote", "r_m",
                         "r_m_sym"], out))

    # -- 3x3 dyadic composition -------------------------
    def dyadic_apply(self, levels, x3, k=2 * np.pi / 10, self_term=1 + 0.1j, mode="ref"):
        """y_i = sum_j T_ij x_j with the dyadic G. mode "ref" composes the
        reference's way (G_ii symmetric compressed, G_ij general full);
        mode "signs" uses per-axis parity compression for every component."""
        d = len(levels)
        ys = [np.zeros(int(np.prod(levels)), np.complex128) for _ in range(3)]
        for i in range(3):
            for j in range(i, 3):
                lags = self.dyadic_lags(levels, i, j, k, self_term)
                if mode == "ref":
                    if i == j:
                        signs, comp = [1] * d, True
                    else:
                        signs, comp = [0] * d, False
                else:
                    signs = [(-1) ** ((i == a) + (j == a)) for a in range(d)]
                    comp = True
                blocks = self.precompute(levels, lags, 0j, comp, signs)
                ys[i] += self.split_apply(levels, blocks, x3[j], comp, signs)
                if i != j:
                    ys[j] += self.split_apply(levels, blocks, x3[i], comp, signs)
        return ys


class RefStatus(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


class TsMetrics(C.Structure):
    _fields_ = [("fft_forward", C.c_uint64), ("fft_inverse", C.c_uint64),
                ("diag_mults", C.c_uint64), ("phase_mults", C.c_uint64),
                ("peak_live_elems", C.c_int64), ("kernel_elems", C.c_uint64),
                ("apply_ns", C.c_uint64), ("precompute_ns", C.c_uint64)]


class TsPolicy(C.Structure):
    _fields_ = [("mode", C.c_int), ("task_budget", C.c_int32)]


class RefLib:
    """The unmodified reference library (oracle/_ref), through its C ABI."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        vp = C.c_void_p
        L.ts_version.restype = C.c_char_p
        L.ts_last_error.restype = C.c_char_p
        L.ts_generator_create.argtypes = [C.c_int32, _i64p, _dp, C.c_int, C.POINTER(vp)]
        L.ts_generator_random.argtypes = [C.c_int32, _i64p, C.c_uint64, C.c_double, C.c_int,
                                          C.POINTER(vp)]
        L.ts_generator_destroy.argtypes = [vp]
        L.ts_random_vector.argtypes = [C.c_int32, _i64p, C.c_uint64, C.c_double, _dp]
        L.ts_operator_create_split.argtypes = [vp, C.c_double, C.c_double, C.c_int, C.POINTER(vp)]
        L.ts_operator_create_embed.argtypes = [vp, C.c_double, C.c_double, C.c_int, C.POINTER(vp)]
        L.ts_operator_apply.argtypes = [vp, _dp, _dp, C.POINTER(TsPolicy), C.POINTER(TsMetrics)]
        L.ts_operator_destroy.argtypes = [vp]
        L.ts_operator_kernel_elems.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.ts_operator_save_kernel.argtypes = [vp, C.c_char_p]
        L.ts_operator_load_split.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ts_naive_matvec.argtypes = [vp, _dp, _dp, C.c_int64]
        L.ts_generator_to_json_file.argtypes = [vp, C.c_char_p]

    def _ok(self, st):
        if st != 0:
            raise RefStatus(st, self.L.ts_last_error().decode())

    def generator(self, levels, lags=None, symmetry=SYM_GENERAL, seed=None, variance=1.0):
        lv, lp = _lv(levels)
        g = C.c_void_p()
        if lags is None:
            self._ok(self.L.ts_generator_random(len(lv), lp, seed, variance, symmetry, C.byref(g)))
        else:
            la, ldp = _cd(lags)
            self._ok(self.L.ts_generator_create(len(lv), lp, ldp, symmetry, C.byref(g)))
        return g

    def random_vector(self, levels, seed, variance=1.0):
        lv, lp = _lv(levels)
        out = np.zeros(int(np.prod(lv)), np.complex128)
        self._ok(self.L.ts_random_vector(len(lv), lp, seed, variance, out.ctypes.data_as(_dp)))
        return out

    def split(self, gen, s0=0j, storage=-1):
        op = C.c_void_p()
        self._ok(self.L.ts_operator_create_split(gen, s0.real, s0.imag, storage, C.byref(op)))
        return op

    def embed(self, gen, s0=0j, storage=-1):
        op = C.c_void_p()
        self._ok(self.L.ts_operator_create_embed(gen, s0.real, s0.imag, storage, C.byref(op)))
        return op

    def apply(self, op, v, parallel=0, metrics=False):
        va, vp = _cd(v)
        y = np.zeros_like(va)
        m = TsMetrics()
        pol = TsPolicy(1, parallel) if parallel else None
        self._ok(self.L.ts_operator_apply(op, vp, y.ctypes.data_as(_dp),
                                          C.byref(pol) if pol else None, C.byref(m)))
        return (y, m) if metrics else y

    def naive(self, gen, v, cap=4096):
        va, vp = _cd(v)
        y = np.zeros_like(va)
        self._ok(self.L.ts_naive_matvec(gen, vp, y.ctypes.data_as(_dp), cap))
        return y

    def destroy_op(self, op):
        self.L.ts_operator_destroy(op)

    def destroy_gen(self, g):
        self.L.ts_generator_destroy(g)

    def dyadic_apply(self, levels, x3, oracle: Oracle, k=2 * np.pi / 10, self_term=1 + 0.1j,
                     parallel=0):
        """3x3 composed from 6 scalar reference operators, 9 applies
        (SURVEY.md §8(c)): G_ii symmetric (auto-compressed), G_ij general."""
        ys = [np.zeros(int(np.prod(levels)), np.complex128) for _ in range(3)]
        for i in range(3):
            for j in range(i, 3):
                lags = oracle.dyadic_lags(levels, i, j, k, self_term)
                g = self.generator(levels, lags, SYM_SYMMETRIC if i == j else SYM_GENERAL)
                op = self.split(g)
                self.destroy_gen(g)
                ys[i] += self.apply(op, x3[j], parallel)
                if i != j:
                    ys[j] += self.apply(op, x3[i], parallel)
                self.destroy_op(op)
        return ys


def rel_l2(a, b) -> float:
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def max_rel(a, b) -> float:
    """Reference metric: max|a-b| / max|b| (proj/src/core/tensor.cpp:302-313)."""
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    s = np.max(np.abs(b)) if b.size else 0.0
    dm = np.max(np.abs(a - b)) if a.size else 0.0
    return float(dm / s) if s > 0 else float(dm)
