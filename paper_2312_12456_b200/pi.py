"""Thin ctypes binding over libpi.so (include/pi.h).  Argument marshalling only.

Every step of the hot path runs in libpi's sm_100a kernels; this module only
turns torch tensors into device pointers and status codes into exceptions.
There is no fallback: if libpi.so is missing or cannot be loaded, importing
this module raises.

Function names mirror the C ABI: pi_layer_create, pi_predict, pi_compact,
pi_sparse_ffn, pi_layer_forward, pi_layer_forward_host, pi_stack_forward,
pi_partition.  ``Layer`` is a convenience owner of a pi_layer handle.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpi.so")

PI_OK = 0
STATUS = {0: "PI_OK", 1: "PI_ERR_INVALID_ARGUMENT", 2: "PI_ERR_SHAPE", 3: "PI_ERR_INDEX",
          4: "PI_ERR_ALIGNMENT", 5: "PI_ERR_UNSUPPORTED", 6: "PI_ERR_CUDA", 7: "PI_ERR_OUT_OF_MEMORY"}
PI_DT_F16, PI_DT_BF16 = 0, 1
PI_ACT_RELU, PI_ACT_REGLU = 0, 1
PI_PRED_RELU, PI_PRED_LINEAR = 0, 1
PI_FFN_16, PI_FFN_Q4 = 0, 1
PI_FLAG_INPUT_RMSNORM = 1
PI_FLAG_MULTI_KERNEL = 2
PI_MAX_BATCH = 32

EXPORTS = ("pi_version", "pi_last_error", "pi_layer_create", "pi_layer_destroy", "pi_layer_get_info",
           "pi_predict", "pi_compact", "pi_sparse_ffn", "pi_layer_forward", "pi_layer_forward_host",
           "pi_stack_forward", "pi_stack_forward_host", "pi_partition", "pi_layer_set_trace",
           "pi_stack_create", "pi_stack_destroy", "pi_stack_run", "pi_stack_run_host", "pi_place_ilp",
           "pi_group_create", "pi_group_destroy", "pi_group_run")


class PiError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class LayerDesc(ctypes.Structure):
    _fields_ = [("layer_id", ctypes.c_int32), ("d", ctypes.c_int32), ("m_total", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("m_local", ctypes.c_int32),
                ("neuron_ids", ctypes.POINTER(ctypes.c_int32)),
                ("dtype", ctypes.c_int), ("act", ctypes.c_int), ("pred_act", ctypes.c_int),
                ("w_up", ctypes.c_void_p), ("w_gate", ctypes.c_void_p), ("w_down", ctypes.c_void_p),
                ("b_up", ctypes.c_void_p), ("b_down", ctypes.c_void_p), ("p_w1", ctypes.c_void_p),
                ("p_b1", ctypes.c_void_p), ("p_w2", ctypes.c_void_p), ("p_b2", ctypes.c_void_p),
                ("logit_threshold", ctypes.c_float), ("max_batch", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("neuron_freq", ctypes.POINTER(ctypes.c_float)),
                ("hot_freq", ctypes.c_float), ("hot_cap", ctypes.c_int32), ("spec_freq", ctypes.c_float),
                ("spec_cap", ctypes.c_int32), ("ffn_format", ctypes.c_int),
                ("w_up_scale", ctypes.c_void_p), ("w_gate_scale", ctypes.c_void_p),
                ("w_down_scale", ctypes.c_void_p)]


class LayerInfo(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("m_local", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("max_batch", ctypes.c_int32), ("mask_words", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("act", ctypes.c_int32), ("pred_act", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("num_sms", ctypes.c_int32), ("weight_bytes", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_int64), ("launches_per_forward", ctypes.c_int32),
                ("ffn_format", ctypes.c_int32), ("n_spec", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libpi.so not found at {LIB_PATH}; build it with `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, P = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER
    lib.pi_version.restype = ctypes.c_char_p
    lib.pi_last_error.restype = ctypes.c_char_p
    lib.pi_layer_create.argtypes = [P(LayerDesc), vp, P(vp)]
    lib.pi_layer_destroy.argtypes = [vp]
    lib.pi_layer_get_info.argtypes = [vp, P(LayerInfo)]
    lib.pi_predict.argtypes = [vp, vp, i32, vp, vp, vp]
    lib.pi_compact.argtypes = [vp, vp, i32, vp, vp, vp]
    lib.pi_sparse_ffn.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp]
    lib.pi_layer_forward.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp]
    lib.pi_layer_forward_host.argtypes = [vp, vp, i32, vp, vp]
    lib.pi_stack_forward.argtypes = [P(vp), i32, vp, i32, vp, vp, vp]
    lib.pi_stack_forward_host.argtypes = [P(vp), i32, vp, i32, vp, vp]
    lib.pi_partition.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    lib.pi_layer_set_trace.argtypes = [vp, vp]
    lib.pi_stack_create.argtypes = [P(vp), i32, P(vp)]
    lib.pi_stack_destroy.argtypes = [vp]
    lib.pi_stack_run.argtypes = [vp, vp, i32, vp, vp, vp]
    lib.pi_stack_run_host.argtypes = [vp, vp, i32, vp, vp]
    lib.pi_group_create.argtypes = [P(vp), i32, i32, i32, ctypes.c_uint32, P(vp)]
    lib.pi_group_destroy.argtypes = [vp]
    lib.pi_group_run.argtypes = [vp, vp, i32, vp, vp, vp]
    dbl = ctypes.c_double
    lib.pi_place_ilp.argtypes = [vp, i32, i32, vp, i32, dbl, dbl, dbl, dbl, vp, vp, ctypes.POINTER(dbl)]
    for name in EXPORTS:
        if name not in ("pi_version", "pi_last_error"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


_lib = _load()


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int):
    if status != PI_OK:
        raise PiError(status, _lib.pi_last_error().decode())


def pi_version() -> str:
    return _lib.pi_version().decode()


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


_DT = {torch.float16: PI_DT_F16, torch.bfloat16: PI_DT_BF16}


class Layer:
    """Owns one pi_layer handle (the library copies and repacks the weights)."""

    def __init__(self, w, neuron_ids: Optional[Sequence[int]] = None, max_batch: int = 1, flags: int = 0,
                 layer_id: int = 0, threshold: Optional[float] = None, pred_act: Optional[str] = None,
                 own_b_down: bool = True, stream=None, neuron_freq=None, hot_freq: float = 0.9,
                 hot_cap: int = 0, q4=None, spec_freq: float = 0.0, spec_cap: int = 1 << 30):
        """w: gen.LayerWeights (16-bit global tensors).  q4: optional gen.Q4Weights -- the FFN
        then runs on INT4 neuron rows (PI_FFN_Q4); w still supplies the predictor and biases."""
        self.handle = None
        dt = w.w_up.dtype
        if dt not in _DT:
            raise ValueError(f"weight dtype {dt} not supported")
        m_total, d = w.w_up.shape
        r = w.p_w1.shape[0]
        ids = None
        m_local = m_total
        if neuron_ids is not None:
            self._ids = np.ascontiguousarray(np.asarray(neuron_ids, dtype=np.int32))
            ids = self._ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            m_local = len(self._ids)
        thr = w.threshold if threshold is None else threshold
        freq_p = None
        if neuron_freq is not None:
            self._freq = np.ascontiguousarray(np.asarray(neuron_freq, dtype=np.float32))
            assert self._freq.shape[0] == m_total
            freq_p = self._freq.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        pa = (pred_act or getattr(w, "pred_act", "relu"))
        if q4 is None:
            mats = (_ptr(w.w_up), _ptr(w.w_gate), _ptr(w.w_down))
            q4p = (PI_FFN_16, None, None, None)
        else:
            mats = (_ptr(q4.up_codes), _ptr(q4.gate_codes), _ptr(q4.down_codes))
            q4p = (PI_FFN_Q4, _ptr(q4.up_scales), _ptr(q4.gate_scales), _ptr(q4.down_scales))
        desc = LayerDesc(layer_id, d, m_total, r, m_local, ids, _DT[dt],
                         PI_ACT_REGLU if w.act == "reglu" else PI_ACT_RELU,
                         PI_PRED_RELU if pa == "relu" else PI_PRED_LINEAR,
                         *mats, _ptr(w.b_up),
                         _ptr(w.b_down) if own_b_down else None, _ptr(w.p_w1), _ptr(w.p_b1), _ptr(w.p_w2),
                         _ptr(w.p_b2), float(thr), int(max_batch), int(flags), freq_p, float(hot_freq),
                         int(hot_cap), float(spec_freq), int(spec_cap), *q4p)
        h = ctypes.c_void_p()
        s = _stream(stream)
        _check(_lib.pi_layer_create(ctypes.byref(desc), s, ctypes.byref(h)))
        self.handle = h
        # create is asynchronous on `s`; the caller's tensors must outlive the repack
        torch.cuda.current_stream().synchronize() if stream is None else torch.cuda.synchronize()
        info = LayerInfo()
        _check(_lib.pi_layer_get_info(self.handle, ctypes.byref(info)))
        self.info = info
        self.d, self.m_local, self.rank, self.words = info.d, info.m_local, info.rank, info.mask_words
        self.max_batch = info.max_batch

    def close(self):
        if self.handle is not None:
            _lib.pi_layer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- the ABI calls (argument marshalling only) ---
    def predict(self, x, mask, logits=None, stream=None):
        _check(_lib.pi_predict(self.handle, _ptr(x), x.shape[0], _ptr(mask), _ptr(logits), _stream(stream)))

    def compact(self, mask, B, ids, n_active, stream=None):
        _check(_lib.pi_compact(self.handle, _ptr(mask), int(B), _ptr(ids), _ptr(n_active), _stream(stream)))

    def sparse_ffn(self, x, ids, n_active, mask, y, stream=None):
        _check(_lib.pi_sparse_ffn(self.handle, _ptr(x), x.shape[0], _ptr(ids), _ptr(n_active), _ptr(mask),
                                  _ptr(y), _stream(stream)))

    def forward(self, x, y, mask_out=None, ids_out=None, n_out=None, stream=None):
        _check(_lib.pi_layer_forward(self.handle, _ptr(x), x.shape[0], _ptr(y), _ptr(mask_out), _ptr(ids_out),
                                     _ptr(n_out), _stream(stream)))

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None):
        assert not x_host.is_cuda and not y_host.is_cuda
        assert x_host.dtype == torch.float32 and y_host.dtype == torch.float32
        _check(_lib.pi_layer_forward_host(self.handle, x_host.data_ptr(), x_host.shape[0], y_host.data_ptr(),
                                          _stream(stream)))

    def set_trace(self, buf: Optional[torch.Tensor]):
        """Phase timestamps of the fused kernel into buf (int64 [num_sms * 256], include/pi.h);
        None = off."""
        if buf is not None and (buf.dtype != torch.int64 or buf.numel() < self.info.num_sms * 256):
            raise ValueError(f"trace buffer must be int64 with >= {self.info.num_sms * 256} elements")
        _check(_lib.pi_layer_set_trace(self.handle, _ptr(buf)))

    # --- buffers sized for this layer ---
    def new_mask(self, B, device="cuda"):
        return torch.zeros(B, self.words, dtype=torch.int32, device=device)

    def new_ids(self, device="cuda"):
        return torch.zeros(max(1, self.m_local), dtype=torch.int32, device=device)


pi_predict = Layer.predict
pi_compact = Layer.compact
pi_sparse_ffn = Layer.sparse_ffn
pi_layer_forward = Layer.forward
pi_layer_forward_host = Layer.forward_host


def pi_layer_create(w, **kw) -> Layer:
    return Layer(w, **kw)


def handles(layers: Sequence[Layer]):
    """ctypes array of the layers' handles (build once, reuse per step)."""
    return (ctypes.c_void_p * len(layers))(*[L.handle for L in layers])


def pi_stack_forward(layers, x, y, n_active_out=None, stream=None):
    arr = layers if isinstance(layers, ctypes.Array) else handles(layers)
    _check(_lib.pi_stack_forward(arr, len(arr), _ptr(x), x.shape[0], _ptr(y), _ptr(n_active_out),
                                 _stream(stream)))


def pi_stack_forward_host(layers, x_host: torch.Tensor, y_host: torch.Tensor, stream=None):
    arr = layers if isinstance(layers, ctypes.Array) else handles(layers)
    assert not x_host.is_cuda and not y_host.is_cuda
    _check(_lib.pi_stack_forward_host(arr, len(arr), x_host.data_ptr(), x_host.shape[0], y_host.data_ptr(),
                                      _stream(stream)))


class StackHandle:
    """Owns a pi_stack (one persistent launch per decode step for all layers)."""

    def __init__(self, layers: Sequence[Layer]):
        self.layers = list(layers)       # keep the layers alive while the stack exists
        arr = handles(self.layers)
        h = ctypes.c_void_p()
        _check(_lib.pi_stack_create(arr, len(arr), ctypes.byref(h)))
        self.handle = h

    def run(self, x, y, n_active_out=None, stream=None):
        _check(_lib.pi_stack_run(self.handle, _ptr(x), x.shape[0], _ptr(y), _ptr(n_active_out), _stream(stream)))

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None):
        assert not x_host.is_cuda and not y_host.is_cuda
        _check(_lib.pi_stack_run_host(self.handle, x_host.data_ptr(), x_host.shape[0], y_host.data_ptr(),
                                      _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) is not None:
            _lib.pi_stack_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GroupHandle:
    """Owns a pi_group: n_groups independent stacks of n_layers layers in ONE persistent launch,
    group_ctas CTAs per group (include/pi.h).  x, y: [n_groups, 1, d] device fp32."""

    def __init__(self, groups: Sequence[Sequence[Layer]], group_ctas: int, flags: int = 0):
        self.layers = [L for g in groups for L in g]
        self.n_groups, self.n_layers = len(groups), len(groups[0])
        assert all(len(g) == self.n_layers for g in groups)
        arr = handles(self.layers)
        h = ctypes.c_void_p()
        _check(_lib.pi_group_create(arr, self.n_groups, self.n_layers, group_ctas, flags, ctypes.byref(h)))
        self.handle = h
        self.group_ctas = group_ctas

    def run(self, x, y, n_active_out=None, stream=None):
        assert x.shape[0] == self.n_groups and y.shape[0] == self.n_groups
        _check(_lib.pi_group_run(self.handle, _ptr(x), x.shape[1], _ptr(y), _ptr(n_active_out), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) is not None:
            _lib.pi_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PI_GROUP_DEFER_AFTER_REDUCTION = 1
PI_GROUP_DEFER_AFTER_BARRIER = 2
pi_group_create = GroupHandle
pi_group_run = GroupHandle.run
pi_stack_create = StackHandle
pi_stack_run = StackHandle.run
pi_stack_run_host = StackHandle.run_host


def pi_partition(freq, n_shards: int, granule: int = 1):
    """Returns (owner[m], shard_ids[m], shard_offsets[G+1]) as int32 numpy arrays."""
    f = np.ascontiguousarray(np.asarray(freq, dtype=np.float32))
    m = f.shape[0]
    owner = np.zeros(m, np.int32)
    ids = np.zeros(m, np.int32)
    off = np.zeros(n_shards + 1 if n_shards > 0 else 1, np.int32)
    _check(_lib.pi_partition(f.ctypes.data, m, int(n_shards), int(granule), owner.ctypes.data, ids.ctypes.data,
                             off.ctypes.data))
    return owner, ids, off


def pi_place_ilp(freq_layers, neuron_bytes, granule: int, mcap_fast: float, bw_fast: float, bw_slow: float,
                 t_sync: float):
    """The paper's placement ILP (Eqs. 1-8), exact.  freq_layers [L, m]; neuron_bytes [L].
    Returns (fast uint8 [L, m], fast_count int32 [L], objective float)."""
    f = np.ascontiguousarray(np.asarray(freq_layers, dtype=np.float32))
    L, m = f.shape
    nbytes = np.ascontiguousarray(np.asarray(neuron_bytes, dtype=np.float64))
    fast = np.zeros((L, m), np.uint8)
    cnt = np.zeros(L, np.int32)
    obj = ctypes.c_double()
    _check(_lib.pi_place_ilp(f.ctypes.data, L, m, nbytes.ctypes.data, int(granule), float(mcap_fast), float(bw_fast),
                             float(bw_slow), float(t_sync), fast.ctypes.data, cnt.ctypes.data, ctypes.byref(obj)))
    return fast, cnt, obj.value


def mask_words(m: int) -> int:
    return (m + 31) // 32


__all__ = ["Layer", "PiError", "pi_version", "pi_layer_create", "pi_predict", "pi_compact", "pi_sparse_ffn",
           "pi_layer_forward", "pi_layer_forward_host", "pi_stack_forward", "pi_partition", "math"]
