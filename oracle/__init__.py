"""FASQ CPU oracle -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over ``oracle/libfasq_oracle.so`` (built from
``oracle/fasq_oracle.c`` by :func:`build`).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2605_04084_b200``) never imports it, and it imports nothing from the
product path.

Every function cites the PAPER.md passage (``P:<line>``) it follows; the
readings of the paper it relies on are listed in DESIGN.md ("Readings").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fasq_oracle.c")
_LIB = os.path.join(_HERE, "libfasq_oracle.so")

# -ffp-contract=off: no a*b+c fusion (the pack is a fixed sequence of RN ops).
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-shared", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter"]


def build(force: bool = False) -> str:
    """Compiles the oracle shared library with gcc (idempotent)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + ".tmp%d" % os.getpid()
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        vp = ctypes.c_void_p
        L.fasq_ref_validate.argtypes = [i64, i64, i32, i32, i32]
        L.fasq_ref_validate16.argtypes = [i64, i64, i32, i32, i32]
        L.fasq_ref_index_bits.argtypes = [i32]
        L.fasq_ref_index_bits.restype = i32
        L.fasq_ref_pack16_range_ex.argtypes = [vp, i64, i64, i32, i32, i32, u64, i32, i32, i32, i64, i64, vp, vp,
                                               vp]
        L.fasq_ref_reconstruct16.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp]
        L.fasq_ref_pack_dim0_range.argtypes = [vp, i64, i64, i32, i32, i32, u64, i32, i32, i32, i64, i64, vp,
                                               vp, vp]
        L.fasq_ref_reconstruct_dim0.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp]
        L.fasq_ref_gemm_rows_dim0.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp, i64, i64, i64, vp]
        L.fasq_ref_gemm_rows16.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp, i64, i64, i64, vp]
        L.fasq_ref_pack_range.argtypes = [vp, i64, i64, i32, i32, i32, u64, i32, i64, i64, vp, vp, vp]
        L.fasq_ref_pack.argtypes = [vp, i64, i64, i32, i32, i32, u64, i32, vp, vp, vp]
        L.fasq_ref_pack_range_ex.argtypes = [vp, i64, i64, i32, i32, i32, u64, i32, i32, i32, i64, i64, vp, vp,
                                             vp]
        L.fasq_ref_lloyd_fp32.argtypes = [vp, i64, i64, i32, i32, i32, u64, i32, i64, vp, vp]
        L.fasq_ref_reconstruct.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp]
        L.fasq_ref_gemm_rows.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp, i64, i64, i64, vp]
        L.fasq_ref_f32_to_f16.argtypes = [ctypes.c_float]
        L.fasq_ref_f32_to_f16.restype = ctypes.c_uint16
        L.fasq_ref_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.fasq_ref_f16_to_f32.restype = ctypes.c_float
        L.fasq_ref_f32_to_f16_array.argtypes = [vp, vp, i64]
        L.fasq_ref_f16_to_f32_array.argtypes = [vp, vp, i64]
        L.fasq_ref_splitmix64_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        L.fasq_ref_splitmix64_next.restype = ctypes.c_uint64
        L.fasq_ref_num_threads.restype = ctypes.c_int
        L.fasq_ref_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__("oracle status %d" % code)
        self.code = code


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _bits16(W) -> np.ndarray:
    """fp16 array (or its uint16 bit pattern) -> contiguous uint16 bits."""
    W = np.asarray(W)
    if W.dtype == np.float16:
        W = W.view(np.uint16)
    assert W.dtype == np.uint16, W.dtype
    return np.ascontiguousarray(W)


def index_bits(C: int) -> int:
    """Eq. 4: bits of one index, ceil(log2 K_s)."""
    return int(lib().fasq_ref_index_bits(C))


def _indices(indices) -> tuple[np.ndarray, bool]:
    """A uint8 (C <= 256) or uint16 (C <= 1024, NEXT-2) index table and whether it is wide."""
    a = np.asarray(indices)
    if a.dtype == np.uint16:
        return np.ascontiguousarray(a), True
    return np.ascontiguousarray(a, dtype=np.uint8), False


def validate(F_out: int, F_in: int, d: int, C: int, group: int) -> int:
    """(a1) Eq. 2 partition checks; 0 = ok, else a status code."""
    return int(lib().fasq_ref_validate(F_out, F_in, d, C, group))


def set_threads(n: int) -> None:
    lib().fasq_ref_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().fasq_ref_num_threads())


def pack(W, d: int, C: int, group: int = 1, seed: int = 0, iters: int = 25,
         cb_range=None, init: int = 0, empty: int = 0):
    """Alg. 1: returns (codebooks fp16 [N_cb][C][d], indices u8
    [N_ss][F_out] -- uint16 when C > 256 --, iters_run int32 [N_cb]).  ``cb_range=(g0, g1)`` packs only
    codebooks g0..g1-1 (rows outside are left zero) -- codebooks are
    independent k-means problems (Alg. 1 "parallel for").
    init: 0 = seeded distinct sample (reading R3), 1 = exact-integer k-means++
    (reading R17); empty: 0 = an empty cluster keeps its centroid
    (R5), 1 = reseed from the farthest point (reading R18)."""
    Wb = _bits16(W)
    F_out, F_in = Wb.shape
    wide = C > 256   # NEXT-2: uint16 indices for C <= 1024 (Eq. 4, Table 2 2-512 / 2-1024)
    st = lib().fasq_ref_validate16(F_out, F_in, d, C, group) if wide else validate(F_out, F_in, d, C, group)
    if st:
        raise OracleError(st)
    N_ss = F_in // d
    N_cb = N_ss // group
    g0, g1 = (0, N_cb) if cb_range is None else cb_range
    cb = np.zeros((N_cb, C, d), np.uint16)
    idx = np.zeros((N_ss, F_out), np.uint16 if wide else np.uint8)
    its = np.zeros((N_cb,), np.int32)
    fn = lib().fasq_ref_pack16_range_ex if wide else lib().fasq_ref_pack_range_ex
    st = fn(_ptr(Wb), F_out, F_in, d, C, group, seed & (2**64 - 1), iters, init, empty, g0, g1, _ptr(cb),
            _ptr(idx), _ptr(its))
    if st:
        raise OracleError(st)
    return cb.view(np.float16), idx, its


def pack_dim0(W, d: int, C: int, group: int = 1, seed: int = 0, iters: int = 25, init: int = 0, empty: int = 0):
    """The paper's dim = 0 partition (Eq. 2 first case; its experiments):
    subspaces along the OUTPUT axis.  Returns (codebooks fp16 [N_cb][C][d], indices
    uint8 [N_ss = F_out/d][F_in], iters_run)."""
    Wb = _bits16(W)
    F_out, F_in = Wb.shape
    st = validate(F_in, F_out, d, C, group)          # dim = 0 is dim = 1 of W^T
    if st:
        raise OracleError(st)
    N_ss = F_out // d
    N_cb = N_ss // group
    cb = np.zeros((N_cb, C, d), np.uint16)
    idx = np.zeros((N_ss, F_in), np.uint8)
    its = np.zeros((N_cb,), np.int32)
    st = lib().fasq_ref_pack_dim0_range(_ptr(Wb), F_out, F_in, d, C, group, seed & (2**64 - 1), iters, init,
                                        empty, 0, N_cb, _ptr(cb), _ptr(idx), _ptr(its))
    if st:
        raise OracleError(st)
    return cb.view(np.float16), idx, its


def reconstruct_dim0(codebooks, indices, F_out: int, group: int = 1) -> np.ndarray:
    """dim = 0 reconstruction: W_hat[ss*d+e][j] = T_cluster[ss/group][T_index[ss][j]][e]."""
    cb = _bits16(codebooks)
    idx = np.ascontiguousarray(indices, dtype=np.uint8)
    N_cb, C, d = cb.shape
    N_ss, F_in = idx.shape
    out = np.zeros((F_out, F_in), np.uint16)
    st = lib().fasq_ref_reconstruct_dim0(_ptr(cb), _ptr(idx), F_out, F_in, d, C, group, _ptr(out))
    if st:
        raise OracleError(st)
    return out.view(np.float16)


def gemm_dim0(codebooks, indices, X, group: int = 1, rows=None) -> np.ndarray:
    """y = W_hat . x in fp64 with the dim = 0 reconstruction (F_out = N_ss * d)."""
    cb = _bits16(codebooks)
    idx = np.ascontiguousarray(indices, dtype=np.uint8)
    Xb = _bits16(X)
    if Xb.ndim == 1:
        Xb = Xb[None, :]
    Xb = np.ascontiguousarray(Xb)
    N_cb, C, d = cb.shape
    N_ss, F_in = idx.shape
    F_out = N_ss * d
    M = Xb.shape[0]
    j0, j1 = (0, F_out) if rows is None else rows
    Y = np.zeros((M, j1 - j0), np.float64)
    st = lib().fasq_ref_gemm_rows_dim0(_ptr(cb), _ptr(idx), F_out, F_in, d, C, group, _ptr(Xb), M, j0, j1,
                                       _ptr(Y))
    if st:
        raise OracleError(st)
    return Y


def lloyd_fp32(W, d: int, C: int, group: int, seed: int, iters: int, g: int):
    """Init + Lloyd for codebook g without finalisation (test hook):
    returns (centroids fp32 [C][d], assignment int32 [group*F_out], passes)."""
    Wb = _bits16(W)
    F_out, F_in = Wb.shape
    cent = np.zeros((C, d), np.float32)
    asg = np.zeros((group * F_out,), np.int32)
    r = lib().fasq_ref_lloyd_fp32(_ptr(Wb), F_out, F_in, d, C, group, seed & (2**64 - 1),
                                  iters, g, _ptr(cent), _ptr(asg))
    if r < 0:
        raise OracleError(r)
    return cent, asg, int(r)


def reconstruct(codebooks, indices, F_in: int, group: int = 1) -> np.ndarray:
    """Naive reconstruction: W_hat fp16 [F_out][F_in]."""
    cb = _bits16(codebooks)
    idx, wide = _indices(indices)
    N_cb, C, d = cb.shape
    N_ss, F_out = idx.shape
    out = np.zeros((F_out, F_in), np.uint16)
    fn = lib().fasq_ref_reconstruct16 if wide else lib().fasq_ref_reconstruct
    st = fn(_ptr(cb), _ptr(idx), F_out, F_in, d, C, group, _ptr(out))
    if st:
        raise OracleError(st)
    return out.view(np.float16)


def gemm(codebooks, indices, X, group: int = 1, rows=None) -> np.ndarray:
    """Reconstruct-then-multiply in fp64 (Eq. 3): Y [M][F_out]
    (or [M][j1-j0] for ``rows=(j0, j1)``)."""
    cb = _bits16(codebooks)
    idx, wide = _indices(indices)
    Xb = _bits16(X)
    if Xb.ndim == 1:
        Xb = Xb[None, :]
    Xb = np.ascontiguousarray(Xb)
    N_cb, C, d = cb.shape
    N_ss, F_out = idx.shape
    M, F_in = Xb.shape
    j0, j1 = (0, F_out) if rows is None else rows
    Y = np.zeros((M, j1 - j0), np.float64)
    fn = lib().fasq_ref_gemm_rows16 if wide else lib().fasq_ref_gemm_rows
    st = fn(_ptr(cb), _ptr(idx), F_out, F_in, d, C, group, _ptr(Xb), M, j0, j1, _ptr(Y))
    if st:
        raise OracleError(st)
    return Y


def gemv(codebooks, indices, x, group: int = 1, rows=None) -> np.ndarray:
    """Decode product y = W_hat . x for a batch x [B][F_in] (Alg. 2's math)."""
    return gemm(codebooks, indices, x, group=group, rows=rows)


def f32_to_f16_bits(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty(a.shape, np.uint16)
    lib().fasq_ref_f32_to_f16_array(_ptr(a), _ptr(out), a.size)
    return out


def f16_bits_to_f32(h) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    out = np.empty(h.shape, np.float32)
    lib().fasq_ref_f16_to_f32_array(_ptr(h), _ptr(out), h.size)
    return out


def splitmix64(seed: int, n: int):
    st = ctypes.c_uint64(seed & (2**64 - 1))
    return [int(lib().fasq_ref_splitmix64_next(ctypes.byref(st))) for _ in range(n)]
