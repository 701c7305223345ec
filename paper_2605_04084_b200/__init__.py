"""B200-native FASQ (arXiv 2605.04084): product-quantized linear layers.

Thin Python binding over the C-ABI library ``lib/libfasq.so`` (declared in
``include/fasq.h``): argument marshalling only.  Every compute step runs in the
library's sm_100a CUDA kernels; PyTorch supplies device memory, streams and
process groups.  There is no CPU fallback: if the library is missing this
module raises on import, and every compute call raises on a non-CUDA tensor.

Names follow the paper: d = SZ_ss (sub-vector size), C = K_s (codebook
cardinality), N_ss = F_in/d subspaces, T_cluster = codebooks, T_index = indices.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FASQ_LIB_PATH") or os.path.join(_PKG, "lib", "libfasq.so")   # override: A/B experiments only

FASQ_F16, FASQ_F32, FASQ_ACC_I64 = 0, 1, 2
GEMM_AUTO, GEMM_LUT, GEMM_EXPAND_TC = 0, 1, 2
FLAG_PDL = 1
FLAG_X_ACC = 2
ACC_SCALE = 2.0 ** 32   # FASQ_ACC_I64 units

_STATUS = {0: "FASQ_OK", -1: "FASQ_E_ARG", -2: "FASQ_E_NONDIVISIBLE", -3: "FASQ_E_CLUSTER_OVERFLOW",
           -4: "FASQ_E_NONFINITE", -5: "FASQ_E_SHAPE", -6: "FASQ_E_UNSUPPORTED", -7: "FASQ_E_CUDA",
           -8: "FASQ_E_OOM", -9: "FASQ_E_RANGE"}

# Every symbol include/fasq.h declares (checked by tests/test_abi.py).
EXPORTED = ["fasq_pack", "fasq_import", "fasq_import_ex", "fasq_export", "fasq_shard_rows", "fasq_layer_info_get",
            "fasq_free", "fasq_gemv", "fasq_gemv_ex", "fasq_gemv_grouped", "fasq_acc_convert",
            "fasq_chain_create", "fasq_chain_create_tp", "fasq_chain_ipc_handle", "fasq_chain_set_peers",
            "fasq_chain_set_peer_chains", "fasq_chain_run", "fasq_chain_output", "fasq_chain_trace",
            "fasq_chain_ctas", "fasq_chain_free", "fasq_chain_run_host", "fasq_chain_check",
            "fasq_chain_plan_ks", "fasq_gemv_host", "fasq_gemm", "fasq_gemm_grouped",
            "fasq_llama_create", "fasq_llama_ipc_handle", "fasq_llama_set_peers", "fasq_llama_set_peer_models",
            "fasq_llama_chain",
            "fasq_llama_kv_cache", "fasq_llama_reset", "fasq_llama_step", "fasq_llama_step_ex", "fasq_llama_tokens",
            "fasq_llama_step_host", "fasq_llama_step_io", "fasq_llama_prefill", "fasq_llama_logits", "fasq_llama_token_history", "fasq_llama_free",
            "fasq_last_launch_count", "fasq_status_string", "fasq_last_error_message",
            "fasq_abi_version", "fasq_set_allocator", "fasq_layer_distinct_centroids"]


LAYOUT_PACKED = 1   # FASQ_LAYOUT_PACKED: ceil(log2 C)-bit indices (NEXT-2)
LAYOUT_DIM0 = 2     # FASQ_LAYOUT_DIM0: output-axis subspaces (NEXT-4)


class FasqError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__("%s (%d)%s" % (_STATUS.get(code, "?"), code, (": " + msg) if msg else ""))
        self.code = code


class _PackParams(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("C", ctypes.c_int32), ("group", ctypes.c_int32),
                ("iters", ctypes.c_int32), ("seed", ctypes.c_uint64), ("init", ctypes.c_int32),
                ("empty", ctypes.c_int32), ("layout", ctypes.c_uint32)]


class GemvOpts(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_uint32), ("next_layers", ctypes.POINTER(ctypes.c_void_p)),
                ("n_next", ctypes.c_int32), ("zero_dev", ctypes.c_void_p), ("zero_bytes", ctypes.c_int64)]


class _ChainStep(ctypes.Structure):
    _fields_ = [("layers", ctypes.POINTER(ctypes.c_void_p)), ("n_layers", ctypes.c_int32),
                ("input_step", ctypes.c_int32), ("input_layer", ctypes.c_int32)]


class LlamaDesc(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("hidden", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float),
                ("max_T", ctypes.c_int32), ("pos_wrap", ctypes.c_int32), ("B", ctypes.c_int32),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("q", ctypes.POINTER(ctypes.c_void_p)), ("k", ctypes.POINTER(ctypes.c_void_p)),
                ("v", ctypes.POINTER(ctypes.c_void_p)), ("o", ctypes.POINTER(ctypes.c_void_p)),
                ("gate", ctypes.POINTER(ctypes.c_void_p)), ("up", ctypes.POINTER(ctypes.c_void_p)),
                ("down", ctypes.POINTER(ctypes.c_void_p)), ("attn_norm", ctypes.POINTER(ctypes.c_void_p)),
                ("mlp_norm", ctypes.POINTER(ctypes.c_void_p)), ("final_norm", ctypes.c_void_p),
                ("embed", ctypes.c_void_p), ("lm_head", ctypes.c_void_p), ("max_ctas", ctypes.c_int32)]


class LayerInfo(ctypes.Structure):
    _fields_ = [("F_out", ctypes.c_int64), ("F_in", ctypes.c_int64), ("d", ctypes.c_int32),
                ("C", ctypes.c_int32), ("group", ctypes.c_int32), ("N_ss", ctypes.c_int32),
                ("N_cb", ctypes.c_int32), ("row_offset", ctypes.c_int32),
                ("index_bytes", ctypes.c_int64), ("codebook_bytes", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("bits_per_weight", ctypes.c_double),
                ("eff_bits_W", ctypes.c_double), ("index_bits", ctypes.c_int32), ("layout", ctypes.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libfasq.so not built (%s); run `python -m paper_2605_04084_b200.build` "
                          "or __graft_entry__.build() -- there is no CPU fallback" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    pp = ctypes.POINTER(ctypes.c_void_p)
    L.fasq_pack.argtypes = [vp, i64, i64, ctypes.POINTER(_PackParams), vp, pp]
    L.fasq_import.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp, pp]
    L.fasq_import_ex.argtypes = [vp, vp, i64, i64, i32, i32, i32, u32, vp, pp]
    L.fasq_export.argtypes = [vp, vp, vp, vp]
    L.fasq_shard_rows.argtypes = [vp, i32, i32, vp, pp]
    L.fasq_layer_info_get.argtypes = [vp, ctypes.POINTER(LayerInfo)]
    L.fasq_free.argtypes = [vp]
    L.fasq_free.restype = None
    L.fasq_gemv.argtypes = [vp, vp, i32, vp, i32, vp]
    L.fasq_gemv_ex.argtypes = [vp, vp, i32, vp, i32, u32, vp]
    L.fasq_gemv_host.argtypes = [vp, vp, i32, vp, i32, vp]
    L.fasq_gemv_grouped.argtypes = [ctypes.POINTER(vp), i32, vp, i32, ctypes.POINTER(vp), i32,
                                    ctypes.POINTER(GemvOpts), vp]
    L.fasq_acc_convert.argtypes = [vp, i64, vp, i32, vp]
    L.fasq_chain_create.argtypes = [ctypes.POINTER(_ChainStep), i32, i32, vp, pp]
    L.fasq_chain_create_tp.argtypes = [ctypes.POINTER(_ChainStep), i32, i32, i32, i32, i32, vp, pp]
    L.fasq_chain_ipc_handle.argtypes = [vp, vp]
    L.fasq_chain_set_peers.argtypes = [vp, vp]
    L.fasq_chain_set_peer_chains.argtypes = [vp, ctypes.POINTER(vp)]
    L.fasq_chain_run.argtypes = [vp, vp, vp]
    L.fasq_chain_output.argtypes = [vp, i32, i32, vp, i32, vp]
    L.fasq_chain_trace.argtypes = [vp, vp]
    L.fasq_chain_ctas.argtypes = [vp]
    L.fasq_chain_free.argtypes = [vp]
    L.fasq_chain_free.restype = None
    L.fasq_chain_run_host.argtypes = [vp, vp, vp, i32, i32, i32, vp]
    L.fasq_chain_check.argtypes = [vp, vp]
    L.fasq_chain_plan_ks.argtypes = [ctypes.POINTER(i64), ctypes.POINTER(i64), i32, i32, i32, i32,
                                     ctypes.POINTER(i32)]
    L.fasq_llama_create.argtypes = [ctypes.POINTER(LlamaDesc), vp, pp]
    L.fasq_llama_ipc_handle.argtypes = [vp, vp]
    L.fasq_llama_set_peers.argtypes = [vp, vp]
    L.fasq_llama_set_peer_models.argtypes = [vp, ctypes.POINTER(vp)]
    L.fasq_llama_chain.argtypes = [vp]
    L.fasq_llama_chain.restype = vp
    L.fasq_llama_kv_cache.argtypes = [vp, i32, pp, pp]
    L.fasq_llama_reset.argtypes = [vp, ctypes.POINTER(i32), i32, vp]
    L.fasq_llama_step.argtypes = [vp, vp]
    L.fasq_llama_tokens.argtypes = [vp, vp, vp]
    L.fasq_llama_step_ex.argtypes = [vp, vp, i32]
    L.fasq_llama_step_host.argtypes = [vp, ctypes.POINTER(i32), vp]
    L.fasq_llama_step_io.argtypes = [vp, ctypes.POINTER(i32), i32, ctypes.POINTER(i32), vp]
    L.fasq_llama_prefill.argtypes = [vp, vp, i32, i32, vp]
    L.fasq_llama_logits.argtypes = [vp, i32, pp]
    L.fasq_llama_token_history.argtypes = [vp, vp, vp]
    L.fasq_llama_free.argtypes = [vp]
    L.fasq_llama_free.restype = None
    L.fasq_gemm.argtypes = [vp, vp, i64, vp, i32, i32, vp]
    L.fasq_gemm_grouped.argtypes = [vp, i32, vp, i64, vp, i32, i32, vp]
    L.fasq_gemm_grouped.restype = ctypes.c_int32
    L.fasq_set_allocator.argtypes = [vp, vp, vp]
    L.fasq_layer_distinct_centroids.argtypes = [vp, ctypes.POINTER(i64), vp]
    L.fasq_layer_distinct_centroids.restype = ctypes.c_int32
    L.fasq_set_allocator.restype = ctypes.c_int32
    L.fasq_status_string.restype = ctypes.c_char_p
    L.fasq_last_error_message.restype = ctypes.c_char_p
    for name in ("fasq_pack", "fasq_import", "fasq_export", "fasq_shard_rows", "fasq_layer_info_get",
                 "fasq_gemv", "fasq_gemv_ex", "fasq_gemv_grouped", "fasq_acc_convert", "fasq_gemv_host",
                 "fasq_chain_create", "fasq_chain_create_tp", "fasq_chain_ipc_handle", "fasq_chain_set_peers",
                 "fasq_chain_set_peer_chains", "fasq_chain_run", "fasq_chain_output", "fasq_chain_trace",
                 "fasq_chain_ctas", "fasq_gemm", "fasq_last_launch_count", "fasq_chain_run_host",
                 "fasq_chain_check", "fasq_chain_plan_ks", "fasq_llama_create", "fasq_llama_ipc_handle",
                 "fasq_llama_set_peers", "fasq_llama_kv_cache", "fasq_llama_reset", "fasq_llama_step",
                 "fasq_llama_tokens", "fasq_llama_step_ex", "fasq_llama_set_peer_models", "fasq_llama_step_host", "fasq_llama_logits", "fasq_llama_token_history",
                 "fasq_abi_version"):
        getattr(L, name).restype = ctypes.c_int32
    return L


lib = _load()


def _check(code: int):
    if code != 0:
        raise FasqError(code, (lib.fasq_last_error_message() or b"").decode())


def _stream(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _check_out(out: torch.Tensor, shape, dtypes=(torch.float16, torch.float32, torch.int64)):
    """Caller-supplied output buffers: CUDA, contiguous, exact shape, known dtype."""
    if not isinstance(out, torch.Tensor) or not out.is_cuda:
        raise TypeError("out must be a CUDA tensor")
    if out.dtype not in dtypes:
        raise TypeError("out dtype %s not in %s" % (out.dtype, dtypes))
    if tuple(out.shape) != tuple(shape) or not out.is_contiguous():
        raise FasqError(-5, "out must be contiguous %s, got %s" % (tuple(shape), tuple(out.shape)))


def _cuda(t: torch.Tensor, dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor (FASQ has no CPU path)" % name)
    if t.dtype != dtype:
        raise TypeError("%s must be %s, got %s" % (name, dtype, t.dtype))
    return t.contiguous()


def last_launch_count() -> int:
    """Kernel launches enqueued by the last compute call on this thread."""
    return int(lib.fasq_last_launch_count())


class Layer:
    """A product-quantized linear layer (y = W_hat . x) resident on one GPU."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        inf = LayerInfo()
        _check(lib.fasq_layer_info_get(self._h, ctypes.byref(inf)))
        self.info = inf.as_dict()
        self.F_out, self.F_in = inf.F_out, inf.F_in
        self.d, self.C, self.group = inf.d, inf.C, inf.group
        self.N_ss, self.N_cb = inf.N_ss, inf.N_cb
        self.index_bits = inf.index_bits   # 8, or ceil(log2 C) for a packed layer (NEXT-2)
        self.layout = inf.layout           # FASQ_LAYOUT_* bits
        self.dim0 = bool(inf.layout & LAYOUT_DIM0)

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib.fasq_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib.fasq_free(self._h)
        except Exception:
            pass

    def export(self, stream=None):
        """Logical arrays: (codebooks fp16 [N_cb][C][d], indices [N_ss][F_out] uint8, or
        int16 holding the uint16 values when C > 256)."""
        cb = torch.empty((self.N_cb, self.C, self.d), dtype=torch.float16, device="cuda")
        idx = torch.empty((self.N_ss, self.F_in if self.dim0 else self.F_out),
                          dtype=torch.uint8 if self.C <= 256 else torch.int16, device="cuda")
        _check(lib.fasq_export(self._h, cb.data_ptr(), idx.data_ptr(), _stream(stream)))
        return cb, idx

    def distinct_centroids(self, stream=None) -> int:
        """P:241 dedup: distinct fp16 centroids over all codebooks (dedup'd
        codebook bytes = this * d * 2)."""
        n = ctypes.c_int64()
        _check(lib.fasq_layer_distinct_centroids(self._h, ctypes.byref(n), _stream(stream)))
        return n.value

    def shard_rows(self, rank: int, world: int, stream=None) -> "Layer":
        out = ctypes.c_void_p()
        _check(lib.fasq_shard_rows(self._h, rank, world, _stream(stream), ctypes.byref(out)))
        return Layer(out.value)


def pack(W: torch.Tensor, d: int, C: int, group: int = 1, seed: int = 0, iters: int = 25,
         stream=None, init: int = 0, empty: int = 0, packed: bool = False, dim0: bool = False) -> Layer:
    """Alg. 1 on the GPU: k-means per codebook -> Layer.  ``packed``
    (implied for C > 256): ceil(log2 C)-bit packed index storage (Eq. 4, NEXT-2).
    ``dim0``: the paper's dim = 0 partition (subspaces along the output axis,
    P:444; NEXT-4)."""
    W = _cuda(W, torch.float16, "W")
    prm = _PackParams(d, C, group, iters, seed & (2**64 - 1), init, empty,
                      (LAYOUT_PACKED if packed else 0) | (LAYOUT_DIM0 if dim0 else 0))
    out = ctypes.c_void_p()
    _check(lib.fasq_pack(W.data_ptr(), W.shape[0], W.shape[1], ctypes.byref(prm), _stream(stream),
                         ctypes.byref(out)))
    return Layer(out.value)


def import_layer(codebooks: torch.Tensor, indices: torch.Tensor, F_in: int, group: int = 1,
                 stream=None, packed: bool | None = None, dim0: bool = False) -> Layer:
    """Layer from logical codebooks fp16 [N_cb][C][d] + indices [N_ss][F_out]
    (uint8 for C <= 256, int16/uint16 bits above).  ``packed`` (default: C > 256)
    stores ceil(log2 C)-bit indices (Eq. 4, NEXT-2).  ``dim0``: indices are
    [N_ss = F_out/d][F_in] of the paper's dim = 0 partition (NEXT-4)."""
    cb = _cuda(codebooks, torch.float16, "codebooks")
    N_cb, C, d = cb.shape
    wide = C > 256
    if isinstance(indices, torch.Tensor) and indices.dtype in (torch.int16, torch.uint16):
        indices = indices.view(torch.int16)
    idx = _cuda(indices, torch.int16 if wide else torch.uint8, "indices")
    if dim0:
        N_ss, F_in_idx = idx.shape
        if F_in_idx != F_in:
            raise FasqError(-5, "dim0 indices must be [F_out/d][F_in]")
        F_out = N_ss * d
    else:
        N_ss, F_out = idx.shape
    if packed is None:
        packed = wide
    layout = (LAYOUT_PACKED if packed else 0) | (LAYOUT_DIM0 if dim0 else 0)
    out = ctypes.c_void_p()
    _check(lib.fasq_import_ex(cb.data_ptr(), idx.data_ptr(), F_out, F_in, d, C, group, layout,
                              _stream(stream), ctypes.byref(out)))
    return Layer(out.value)


def gemv(layer: Layer, x: torch.Tensor, out: torch.Tensor | None = None,
         out_dtype: torch.dtype = torch.float32, flags: int = 0, stream=None) -> torch.Tensor:
    """Decode GEMV (Eq. 3 / Alg. 2): x fp16 [B][F_in] (B <= 8) -> y [B][F_out]."""
    x = _cuda(x, torch.float16, "x")
    if x.dim() == 1:
        x = x.unsqueeze(0)
    B = x.shape[0]
    if x.shape[1] != layer.F_in:
        raise FasqError(-5, "x has %d columns, layer F_in=%d" % (x.shape[1], layer.F_in))
    if out is None:
        out = torch.empty((B, layer.F_out), dtype=out_dtype, device=x.device)
    _check_out(out, (B, layer.F_out), (torch.float16, torch.float32))
    yt = FASQ_F32 if out.dtype == torch.float32 else FASQ_F16
    _check(lib.fasq_gemv_ex(layer.handle, x.data_ptr(), B, out.data_ptr(), yt, flags, _stream(stream)))
    return out


def gemv_grouped(layers, x: torch.Tensor, outs=None, out_dtype: torch.dtype = torch.float32,
                 flags: int = 0, next_layers=None, zero: torch.Tensor | None = None, stream=None):
    """One launch for up to 4 layers sharing x (e.g. q/k/v): returns [y_l].

    ``out_dtype=torch.int64`` selects FASQ_ACC_I64 outputs (added into
    caller-zeroed ``outs``); an int64 ``x`` is read as FASQ_ACC_I64.
    ``next_layers``: layers of the next launch in a decode chain (L2 warm-up
    hint).  ``zero``: a device tensor to zero during the launch."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("x must be a CUDA tensor (FASQ has no CPU path)")
    if x.dtype == torch.int64:
        flags |= FLAG_X_ACC
    elif x.dtype != torch.float16:
        raise TypeError("x must be fp16 or int64 (FASQ_ACC_I64)")
    x = x.contiguous()
    if x.dim() == 1:
        x = x.unsqueeze(0)
    B = x.shape[0]
    n = len(layers)
    if outs is None:
        outs = [torch.zeros((B, L.F_out), dtype=out_dtype, device=x.device) for L in layers]
    dt = outs[0].dtype
    yt = FASQ_F32 if dt == torch.float32 else FASQ_F16 if dt == torch.float16 else FASQ_ACC_I64
    hs = (ctypes.c_void_p * n)(*[L.handle.value for L in layers])
    ys = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
    nn = len(next_layers) if next_layers else 0
    nx = (ctypes.c_void_p * max(nn, 1))(*([L.handle.value for L in next_layers] if nn else [None]))
    opts = GemvOpts(flags, nx if nn else None, nn, zero.data_ptr() if zero is not None else None,
                    zero.numel() * zero.element_size() if zero is not None else 0)
    _check(lib.fasq_gemv_grouped(hs, n, x.data_ptr(), B, ys, yt, ctypes.byref(opts), _stream(stream)))
    return outs


def acc_convert(acc: torch.Tensor, out: torch.Tensor | None = None, out_dtype=torch.float16, stream=None):
    """FASQ_ACC_I64 -> fp16/fp32."""
    acc = _cuda(acc, torch.int64, "acc")
    if out is None:
        out = torch.empty(acc.shape, dtype=out_dtype, device=acc.device)
    yt = FASQ_F32 if out.dtype == torch.float32 else FASQ_F16
    _check(lib.fasq_acc_convert(acc.data_ptr(), acc.numel(), out.data_ptr(), yt, _stream(stream)))
    return out


class Chain:
    """Persistent decode-chain executor (fasq_chain_*): a list of steps, each
    ``(layers, input)`` with ``input = None`` (the external x) or
    ``(step, layer)`` (an earlier step's output)."""

    def __init__(self, steps, B: int = 1, stream=None, world: int = 1, rank: int = 0, max_ctas: int = 0):
        self._keep = []
        arr = (_ChainStep * len(steps))()
        for i, (layers, src) in enumerate(steps):
            hs = (ctypes.c_void_p * len(layers))(*[L.handle.value for L in layers])
            self._keep.append((hs, list(layers)))
            arr[i].layers = hs
            arr[i].n_layers = len(layers)
            arr[i].input_step, arr[i].input_layer = (-1, 0) if src is None else src
        out = ctypes.c_void_p()
        _check(lib.fasq_chain_create_tp(arr, len(steps), B, world, rank, max_ctas, _stream(stream),
                                        ctypes.byref(out)))
        self._h = out
        self.B = B
        self.world, self.rank = world, rank
        self.steps = [(list(l), s) for (l, s) in steps]
        self.n_steps = len(self.steps)

    @property
    def in_features(self) -> int:
        for layers, src in self.steps:
            if src is None:
                return layers[0].F_in
        raise ValueError("chain has no external-input step")

    def run(self, x: torch.Tensor, stream=None):
        x = _cuda(x, torch.float16, "x")
        if x.dim() == 1:
            x = x.unsqueeze(0)
        if tuple(x.shape) != (self.B, self.in_features):
            raise FasqError(-5, "x must be [%d][%d], got %s" % (self.B, self.in_features, tuple(x.shape)))
        _check(lib.fasq_chain_run(self._h, x.data_ptr(), _stream(stream)))

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor, step: int, layer: int = 0, stream=None):
        """End to end with HOST buffers (H2D of x, the chain, conversion, D2H of y)."""
        if x_host.is_cuda or y_host.is_cuda:
            raise TypeError("run_host takes host tensors")
        if x_host.dtype != torch.float16 or tuple(x_host.shape) != (self.B, self.in_features):
            raise FasqError(-5, "x_host must be fp16 [%d][%d]" % (self.B, self.in_features))
        width = self.steps[step][0][layer].F_out * self.world
        if tuple(y_host.shape) != (self.B, width) or y_host.dtype not in (torch.float16, torch.float32):
            raise FasqError(-5, "y_host must be fp16/fp32 [%d][%d]" % (self.B, width))
        if not (x_host.is_contiguous() and y_host.is_contiguous()):
            raise ValueError("host buffers must be contiguous")
        yt = FASQ_F32 if y_host.dtype == torch.float32 else FASQ_F16
        _check(lib.fasq_chain_run_host(self._h, x_host.data_ptr(), y_host.data_ptr(), step, layer, yt,
                                       _stream(stream)))
        return y_host

    def check(self, stream=None):
        """Raises FasqError(FASQ_E_RANGE) if a run since the last check had an
        out-of-range counted partial (synchronises the stream)."""
        _check(lib.fasq_chain_check(self._h, _stream(stream)))

    def ipc_handle(self) -> bytes:
        """64-byte cudaIpcMemHandle of this chain's arena (exchange across ranks)."""
        buf = ctypes.create_string_buffer(64)
        _check(lib.fasq_chain_ipc_handle(self._h, buf))
        return buf.raw

    def set_peers(self, handles):
        """handles: list of every rank's ipc_handle() (rank order)."""
        blob = b"".join(handles)
        if len(blob) != 64 * self.world:
            raise ValueError("need world x 64-byte handles")
        _check(lib.fasq_chain_set_peers(self._h, ctypes.create_string_buffer(blob, len(blob))))

    def set_peer_chains(self, chains):
        """In-process ranks: chains[r] is rank r's Chain (including self)."""
        arr = (ctypes.c_void_p * len(chains))(*[c._h.value for c in chains])
        _check(lib.fasq_chain_set_peer_chains(self._h, arr))

    def output(self, step: int, layer: int = 0, out: torch.Tensor | None = None,
               out_dtype=torch.float16, stream=None) -> torch.Tensor:
        F_out = self.steps[step][0][layer].F_out * self.world
        if out is None:
            out = torch.empty((self.B, F_out), dtype=out_dtype, device="cuda")
        _check_out(out, (self.B, F_out))
        dt = out.dtype
        yt = FASQ_F32 if dt == torch.float32 else FASQ_F16 if dt == torch.float16 else FASQ_ACC_I64
        _check(lib.fasq_chain_output(self._h, step, layer, out.data_ptr(), yt, _stream(stream)))
        return out

    @property
    def ctas(self) -> int:
        return int(lib.fasq_chain_ctas(self._h))

    def trace(self, buf: torch.Tensor | None):
        """Diagnostics: record %globaltimer stamps into ``buf`` (int64
        [steps][ctas][4]) on every later run; None turns it off."""
        if buf is not None:
            if buf.dtype != torch.int64 or not buf.is_cuda or buf.numel() < self.n_steps * self.ctas * 4:
                raise ValueError("trace buffer: cuda int64 [steps][ctas][4]")
        self._trace_buf = buf
        _check(lib.fasq_chain_trace(self._h, None if buf is None else buf.data_ptr()))

    def free(self):
        if self._h and getattr(self, "_owned", True):
            lib.fasq_chain_free(self._h)
        self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            if getattr(self, "_h", None) and getattr(self, "_owned", True):
                lib.fasq_chain_free(self._h)
        except Exception:
            pass


def gemv_host(layer: Layer, x_host: torch.Tensor, y_host: torch.Tensor, stream=None) -> torch.Tensor:
    """End-to-end GEMV with HOST buffers (H2D of x, kernels, D2H of y inside)."""
    if x_host.is_cuda or y_host.is_cuda:
        raise TypeError("gemv_host takes host tensors")
    yt = FASQ_F32 if y_host.dtype == torch.float32 else FASQ_F16
    _check(lib.fasq_gemv_host(layer.handle, x_host.data_ptr(), x_host.shape[0], y_host.data_ptr(), yt,
                              _stream(stream)))
    return y_host


def gemm(layer: Layer, X: torch.Tensor, out: torch.Tensor | None = None,
         out_dtype: torch.dtype = torch.float32, algo: int = GEMM_AUTO, stream=None) -> torch.Tensor:
    """Prefill GEMM (Alg. 3's math): X fp16 [M][F_in] -> Y [M][F_out]."""
    X = _cuda(X, torch.float16, "X")
    M = X.shape[0]
    if X.shape[1] != layer.F_in:
        raise FasqError(-5, "X has %d columns, layer F_in=%d" % (X.shape[1], layer.F_in))
    if out is None:
        out = torch.empty((M, layer.F_out), dtype=out_dtype, device=X.device)
    _check_out(out, (M, layer.F_out), (torch.float16, torch.float32))
    yt = FASQ_F32 if out.dtype == torch.float32 else FASQ_F16
    _check(lib.fasq_gemm(layer.handle, X.data_ptr(), M, out.data_ptr(), yt, algo, _stream(stream)))
    return out


def gemm_grouped(layers, X: torch.Tensor, outs=None, out_dtype: torch.dtype = torch.float32, algo: int = GEMM_AUTO,
                 stream=None):
    """fasq_gemm_grouped: the prefill GEMMs of layers sharing X (q / k / v,
    gate / up) -- one EXPAND launch over all their row tiles when each would run
    EXPAND on its own.  Returns the list of Y [M][F_out_l]."""
    X = _cuda(X, torch.float16, "X")
    M = X.shape[0]
    for L in layers:
        if X.shape[1] != L.F_in:
            raise FasqError(-5, "X has %d columns, layer F_in=%d" % (X.shape[1], L.F_in))
    if outs is None:
        outs = [torch.empty((M, L.F_out), dtype=out_dtype, device=X.device) for L in layers]
    for L, o in zip(layers, outs):
        _check_out(o, (M, L.F_out), (torch.float16, torch.float32))
    if len({o.dtype for o in outs}) != 1:
        raise FasqError(-1, "outs must share one dtype")
    yt = FASQ_F32 if outs[0].dtype == torch.float32 else FASQ_F16
    n = len(layers)
    hs = (ctypes.c_void_p * n)(*[L.handle.value for L in layers])
    ys = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
    _check(lib.fasq_gemm_grouped(hs, n, X.data_ptr(), M, ys, yt, algo, _stream(stream)))
    return outs


# ---- device memory through torch (fasq_set_allocator) -------------------------
_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


def _torch_alloc(ctx, nbytes, stream):
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
    except Exception:   # OOM etc.: the library reports FASQ_E_OOM
        return None


def _torch_free(ctx, ptr, stream):
    torch.cuda.caching_allocator_delete(ptr)


_TORCH_HOOKS = (_ALLOC_FN(_torch_alloc), _FREE_FN(_torch_free))   # kept alive for the process


def use_torch_allocator(on: bool = True):
    """Route every device buffer libfasq owns (layers, chains, KV caches, per-
    call split-K workspaces, pack scratch) through torch's caching allocator
    (north_star: PyTorch for device memory), or back to CUDA's stream-ordered
    allocator with on=False.  Tensor-parallel chain arenas stay cudaMalloc
    allocations (CUDA IPC)."""
    if on:
        _check(lib.fasq_set_allocator(ctypes.cast(_TORCH_HOOKS[0], ctypes.c_void_p),
                                      ctypes.cast(_TORCH_HOOKS[1], ctypes.c_void_p), None))
    else:
        _check(lib.fasq_set_allocator(None, None, None))


def plan_ks(shapes, nctas: int = 148, d: int = 2, B: int = 1):
    """Host-only query of the chain planner: K-split count per layer of one
    grouped step; shapes = [(F_out, F_in)]."""
    n = len(shapes)
    fo = (ctypes.c_int64 * n)(*[s[0] for s in shapes])
    ng = (ctypes.c_int64 * n)(*[-(-(s[1] // d) // 32) for s in shapes])
    ks = (ctypes.c_int32 * n)()
    _check(lib.fasq_chain_plan_ks(fo, ng, n, nctas, d, B, ks))
    return list(ks)


class Llama:
    """Whole-model greedy decode (fasq_llama_*): a Llama-shaped decoder whose
    every linear layer is a FASQ Layer.  ``layers`` is a list (n_layers) of
    dicts with keys q, k, v, o, gate, up, down (Layer, this rank's shard) and
    attn_norm, mlp_norm (fp16 CUDA tensors [hidden]).  Chain step numbering:
    0 = h0 (embedding); block l: 1+5l q/k/v, 2+5l attention output, 3+5l h
    after the attention residual, 4+5l gate/up, 5+5l h after the MLP residual."""

    def __init__(self, layers, final_norm, embed, lm_head, n_heads, n_kv_heads, head_dim, vocab,
                 rms_eps=1e-5, rope_theta=500000.0, max_T=2048, pos_wrap=0, B=1, world=1, rank=0,
                 max_ctas=0, stream=None):
        self._keep = [final_norm, embed, lm_head, layers]
        n = len(layers)
        hidden = embed.shape[1]
        for t, name in ((final_norm, "final_norm"), (embed, "embed"), (lm_head, "lm_head")):
            _cuda(t, torch.float16, name)
            if not t.is_contiguous():
                raise ValueError(name + " must be contiguous")
        if tuple(embed.shape) != (vocab, hidden) or tuple(lm_head.shape) != (vocab // world, hidden):
            raise FasqError(-5, "embed must be [vocab][hidden] and lm_head [vocab/world][hidden]")

        def arr(key):
            a = (ctypes.c_void_p * n)()
            for i, L in enumerate(layers):
                v = L[key]
                if isinstance(v, Layer):
                    a[i] = v.handle.value
                else:
                    _cuda(v, torch.float16, key)
                    if tuple(v.shape) != (hidden,) or not v.is_contiguous():
                        raise FasqError(-5, "%s[%d] must be fp16 [%d]" % (key, i, hidden))
                    a[i] = v.data_ptr()
            self._keep.append(a)
            return a
        ffn = layers[0]["gate"].F_out * world
        self.desc = LlamaDesc(n, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab, rms_eps, rope_theta, max_T,
                              pos_wrap, B, world, rank, arr("q"), arr("k"), arr("v"), arr("o"), arr("gate"),
                              arr("up"), arr("down"), arr("attn_norm"), arr("mlp_norm"), final_norm.data_ptr(),
                              embed.data_ptr(), lm_head.data_ptr(), max_ctas)
        out = ctypes.c_void_p()
        _check(lib.fasq_llama_create(ctypes.byref(self.desc), _stream(stream), ctypes.byref(out)))
        self._h = out
        self.B, self.world, self.rank = B, world, rank
        self.n_layers, self.hidden, self.vocab, self.max_T = n, hidden, vocab, max_T
        self.n_kv_local, self.head_dim = n_kv_heads // world, head_dim
        # a non-owning view of the model's chain (fasq_chain_output etc.)
        self.chain = Chain.__new__(Chain)
        self.chain._h = ctypes.c_void_p(lib.fasq_llama_chain(self._h))
        self.chain._owned = False
        self.chain.n_steps = 1 + 5 * n
        self.chain.B, self.chain.world, self.chain.rank = B, world, rank
        self._logits = None

    def kv_cache(self, layer: int):
        """(K, V) fp16 views [B][n_kv/world][max_T][head_dim] of a layer's cache."""
        kp, vp = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib.fasq_llama_kv_cache(self._h, layer, ctypes.byref(kp), ctypes.byref(vp)))
        shape = (self.B, self.n_kv_local, self.max_T, self.head_dim)
        return _wrap_dev(kp.value, shape, torch.float16), _wrap_dev(vp.value, shape, torch.float16)

    def reset(self, tokens, pos: int, stream=None):
        arr = (ctypes.c_int32 * self.B)(*[int(t) for t in tokens])
        _check(lib.fasq_llama_reset(self._h, arr, pos, _stream(stream)))

    def step(self, stream=None):
        _check(lib.fasq_llama_step(self._h, _stream(stream)))

    def step_part(self, part: int, stream=None):
        """part 1: the chain kernel of a step, 2: its lm_head kernel (per-kernel timing)."""
        _check(lib.fasq_llama_step_ex(self._h, _stream(stream), part))

    def tokens(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self.B,), dtype=torch.int32, device="cuda")
        _check_out(out, (self.B,), (torch.int32,))
        _check(lib.fasq_llama_tokens(self._h, out.data_ptr(), _stream(stream)))
        return out

    def step_host(self, stream=None):
        """One step end to end; returns the chosen tokens (host list)."""
        arr = (ctypes.c_int32 * self.B)()
        _check(lib.fasq_llama_step_host(self._h, arr, _stream(stream)))
        return list(arr)

    def prefill(self, tokens, pos0: int = 0, stream=None):
        """fasq_llama_prefill: run the prompt `tokens` (device int32 tensor or
        list) at positions pos0.. through the whole model; the next step()
        decodes the greedy continuation."""
        if not isinstance(tokens, torch.Tensor):
            tokens = torch.tensor(tokens, dtype=torch.int32, device="cuda")
        t = _cuda(tokens, torch.int32, "tokens")
        _check(lib.fasq_llama_prefill(self._h, t.data_ptr(), t.numel(), pos0, _stream(stream)))

    def step_io(self, tokens, pos: int = -1, stream=None):
        """fasq_llama_step_io: decode `tokens` (host list of B ints) at `pos`
        (-1: the current position) and return the chosen tokens; one sync."""
        tin = (ctypes.c_int32 * self.B)(*tokens)
        tout = (ctypes.c_int32 * self.B)()
        _check(lib.fasq_llama_step_io(self._h, tin, pos, tout, _stream(stream)))
        return list(tout)

    def enable_logits(self, on: bool = True):
        p = ctypes.c_void_p()
        _check(lib.fasq_llama_logits(self._h, 1 if on else 0, ctypes.byref(p)))
        self._logits = _wrap_dev(p.value, (self.B, self.vocab // self.world), torch.float32) if on else None
        return self._logits

    def token_history(self, stream=None) -> torch.Tensor:
        out = torch.empty((self.B, self.max_T), dtype=torch.int32, device="cuda")
        _check(lib.fasq_llama_token_history(self._h, out.data_ptr(), _stream(stream)))
        return out

    def output(self, step: int, layer: int = 0, out_dtype=torch.float32, width: int | None = None, stream=None):
        """Chain output (see the class docstring for the step numbering)."""
        if width is None:
            width = self._width(step, layer)
        out = torch.empty((self.B, width), dtype=out_dtype, device="cuda")
        yt = FASQ_F32 if out_dtype == torch.float32 else FASQ_F16 if out_dtype == torch.float16 else FASQ_ACC_I64
        _check(lib.fasq_chain_output(self.chain._h, step, layer, out.data_ptr(), yt, _stream(stream)))
        return out

    def _width(self, step, layer):
        if step == 0:
            return self.hidden
        k = (step - 1) % 5
        L = self._keep[3][(step - 1) // 5]
        if k == 0:
            return (L["q"], L["k"], L["v"])[layer].F_out
        if k == 1:
            return L["q"].F_out
        if k == 3:
            return L["gate"].F_out
        return self.hidden

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(lib.fasq_llama_ipc_handle(self._h, buf))
        return buf.raw

    def set_peer_models(self, models):
        """In-process ranks (tests): models[r] is rank r's Llama (including self)."""
        arr = (ctypes.c_void_p * len(models))(*[m._h.value for m in models])
        _check(lib.fasq_llama_set_peer_models(self._h, arr))

    def set_peers(self, handles):
        blob = b"".join(handles)
        if len(blob) != 64 * self.world:
            raise ValueError("need world x 64-byte handles")
        _check(lib.fasq_llama_set_peers(self._h, ctypes.create_string_buffer(blob, len(blob))))

    def free(self):
        if self._h:
            lib.fasq_llama_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib.fasq_llama_free(self._h)
        except Exception:
            pass


def _wrap_dev(ptr: int, shape, dtype) -> torch.Tensor:
    """A torch view of library-owned device memory (valid while its owner lives)."""
    n = 1
    for v in shape:
        n *= v
    es = torch.empty((), dtype=dtype).element_size()

    class _A:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": {torch.float16: "<f2", torch.float32: "<f4",
                                                                       torch.int32: "<i4"}[dtype],
                                    "data": (ptr, False), "version": 2}
    t = torch.as_tensor(_A(), device="cuda")
    assert t.numel() * es == n * es
    return t
