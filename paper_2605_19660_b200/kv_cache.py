"""Host-side mirror of the reference KvCache API over the C-ABI library.

Reference interface (C++): oscar::KvCache (kv_cache.hpp:61-123),
oscar::PipelineConfig (kv_cache.hpp:19-32), decode_step / attention
(pipeline.hpp:43-68).  This module binds include/oscar_kv.h with ctypes; it
holds no compute of its own.  Device tensors are passed as raw pointers
(torch is used only to own device memory).  If the CUDA library
(liboscar_b200.so) is missing, importing this module raises -- there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSCAR_LIB") or os.path.join(HERE, "liboscar_b200.so")  # OSCAR_LIB: A/B builds

METHODS = {"fp": 0, "kivi": 1, "rotate-only": 2, "scale-only": 3, "oscar": 4}
SCALINGS = {"l2": 0, "rsqrt": 1, "max": 2, "mean-abs": 3}
R, D, G = 128, 128, 32


class _Config(ctypes.Structure):
    _fields_ = [
        ("method", ctypes.c_int32),
        ("bits", ctypes.c_int32),
        ("group_size", ctypes.c_int64),
        ("residual_len", ctypes.c_int64),
        ("scaling", ctypes.c_int32),
        ("rotate_v", ctypes.c_int32),
        ("head_dim", ctypes.c_int64),
        ("heads", ctypes.c_int64),
    ]


class _MemReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "packed_tokens", "residual_tokens", "packed_k_payload_bits", "packed_v_payload_bits",
        "residual_k_payload_bits", "residual_v_payload_bits", "k_norm_bits", "param_bits")] + [
        ("effective_bits_per_value", ctypes.c_double),
        ("device_hot_bytes", ctypes.c_int64),
        ("device_total_bytes", ctypes.c_int64),
    ]


_P = ctypes.c_void_p


class _Export(ctypes.Structure):
    _fields_ = [(n, _P) for n in (
        "k_payload", "v_payload", "k_delta", "k_constant", "v_delta", "v_constant", "k_zp", "v_zp",
        "k_raw", "v_raw", "k_norms", "k_residual", "k_norms_residual", "v_residual")]


PEER_MAX, PEER_STRIDE = 8, 132


class _PeerPlan(ctypes.Structure):
    """oscar_peer_plan (include/oscar_kv.h)."""

    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("rows", ctypes.c_int64),
                ("recv", _P * PEER_MAX)]


_lib = None


def lib():
    """Load liboscar_b200.so (fails loudly: the product has no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.oscar_last_error.restype = ctypes.c_char_p
        L.oscar_kv_config_validate.argtypes = [ctypes.POINTER(_Config)]
        L.oscar_kv_create.argtypes = [ctypes.POINTER(_Config), ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
        L.oscar_kv_destroy.argtypes = [_P]
        L.oscar_kv_append.argtypes = [_P, _P, _P, ctypes.c_int64, _P]
        L.oscar_kv_decode_step.argtypes = [_P, _P, _P, _P, _P, _P, _P]
        L.oscar_kv_attend.argtypes = [_P, _P, _P, _P, _P]
        L.oscar_kv_decode_step_logits.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P]
        L.oscar_kv_logits.argtypes = [_P, _P, _P, _P, _P]
        L.oscar_kv_decode_step_many.argtypes = [ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P]
        L.oscar_kv_decode_step_host.argtypes = [_P, _P, _P, _P, _P, _P, _P]
        L.oscar_kv_append_k.argtypes = [_P, _P, _P, ctypes.c_int64, _P]
        L.oscar_kv_append_v.argtypes = [_P, _P, ctypes.c_int64, _P]
        L.oscar_kv_decode_step_f64.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P]
        L.oscar_kv_stats_v.argtypes = [_P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.oscar_kvc1_read_config.argtypes = [ctypes.c_char_p, ctypes.POINTER(_Config), ctypes.POINTER(ctypes.c_int64)]
        L.oscar_kv_stats.argtypes = [_P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int64)]
        L.oscar_kv_memory_report.argtypes = [_P, ctypes.POINTER(_MemReport)]
        L.oscar_kv_export.argtypes = [_P, ctypes.c_int64, ctypes.POINTER(_Export)]
        L.oscar_kv_dump.argtypes = [_P, ctypes.c_int64, ctypes.c_char_p]
        L.oscar_kv_load.argtypes = [_P, ctypes.c_int64, ctypes.c_char_p]
        L.oscar_kv_materialize.argtypes = [_P, ctypes.c_int64, _P, _P]
        L.oscar_lse_merge.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P, _P, _P]
        L.oscar_kv_last_launch_count.argtypes = [_P]
        L.oscar_kv_status.argtypes = [_P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]
        L.oscar_peer_area_bytes.restype = ctypes.c_int64
        L.oscar_peer_area_bytes.argtypes = [ctypes.c_int32, ctypes.c_int64]
        L.oscar_kv_attend_publish.argtypes = [_P, _P, _P, _P, ctypes.POINTER(_PeerPlan), ctypes.c_uint32, _P]
        L.oscar_peer_publish_empty.argtypes = [ctypes.POINTER(_PeerPlan), ctypes.c_uint32, _P]
        L.oscar_peer_merge.argtypes = [ctypes.POINTER(_PeerPlan), ctypes.c_uint32, _P, _P, _P, _P]
        L.oscar_ipc_alloc.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(_P), _P]
        L.oscar_ipc_open.argtypes = [_P, ctypes.c_int32, ctypes.POINTER(_P)]
        L.oscar_ipc_close.argtypes = [_P]
        L.oscar_ipc_free.argtypes = [_P]
        _lib = L
    return _lib


# every entry point declared in include/oscar_kv.h
C_ABI_SYMBOLS = [
    "oscar_last_error", "oscar_kv_config_validate", "oscar_kv_create", "oscar_kv_destroy", "oscar_kv_append",
    "oscar_kv_decode_step", "oscar_kv_decode_step_many", "oscar_kv_attend", "oscar_kv_decode_step_host", "oscar_kv_stats",
    "oscar_kv_memory_report", "oscar_kv_export", "oscar_kv_dump", "oscar_kv_load", "oscar_kv_materialize", "oscar_lse_merge",
    "oscar_kv_last_launch_count", "oscar_peer_area_bytes", "oscar_kv_attend_publish", "oscar_peer_publish_empty",
    "oscar_peer_merge", "oscar_ipc_alloc", "oscar_ipc_open", "oscar_ipc_close", "oscar_ipc_free",
    "oscar_kv_status", "oscar_kv_decode_step_logits", "oscar_kv_logits",
    "oscar_kv_append_k", "oscar_kv_append_v", "oscar_kv_decode_step_f64", "oscar_kv_stats_v", "oscar_kvc1_read_config",
]


def _check(rc: int):
    if rc != 0:
        msg = lib().oscar_last_error().decode()
        # reference exception types: invalid_argument / logic_error / runtime_error
        raise {1: ValueError, 2: RuntimeError}.get(rc, OSError)(msg)


@dataclass
class PipelineConfig:
    """oscar::PipelineConfig (kv_cache.hpp:19-32) + the value-rotation mode."""

    method: str = "oscar"
    bits: int = 2
    group_size: int = 32
    residual_len: int = 128
    scaling: str = "l2"
    head_dim: int = 128
    heads: int = 1
    rotate_v: bool = False

    def _c(self) -> _Config:
        return _Config(METHODS[self.method], self.bits, self.group_size, self.residual_len, SCALINGS[self.scaling],
                       int(self.rotate_v), self.head_dim, self.heads)

    def rotates(self):
        return self.method in ("rotate-only", "oscar")

    def scales(self):
        return self.method in ("scale-only", "oscar")

    def quantizes(self):
        return self.method != "fp" and self.bits != 0

    def validate(self):
        c = self._c()
        _check(lib().oscar_kv_config_validate(ctypes.byref(c)))


def _ptr(t) -> int:
    if t is None:
        return None
    return t.data_ptr()


def _dev_of(t, name: str) -> int:
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor, got {type(t).__name__}")
    return t.device.index


def _need(t, name: str, device: int, dtype: str, shape=None, numel=None):
    """The C-ABI takes raw device pointers and cannot check what they point to:
    verify device, dtype, contiguity and shape here (a wrong batch or head
    count would read/write out of bounds on the device; a strided view would
    silently build a wrong cache)."""
    import torch

    if t is None:
        raise ValueError(f"{name}: tensor required")
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.device.index != device:
        raise ValueError(f"{name}: expected a CUDA tensor on cuda:{device}, got "
                         f"{getattr(t, 'device', type(t).__name__)}")
    want = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dtype]
    if t.dtype != want:
        raise ValueError(f"{name}: expected {want}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous (pass .contiguous())")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: expected {numel} elements, got {t.numel()}")
    return t


def _stream(stream):
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return stream


class KvCache:
    """Device KV cache for `batch` sequences x cfg.heads KV heads (one writer)."""

    def __init__(self, cfg: PipelineConfig, batch: int, q_heads: int, max_tokens: int, device: int = 0,
                 keep_exact: bool = True):
        self.cfg = cfg
        self.B, self.Hq, self.H, self.max_tokens, self.device = batch, q_heads, cfg.heads, max_tokens, device
        self._c = cfg._c()
        h = _P()
        _check(lib().oscar_kv_create(ctypes.byref(self._c), batch, q_heads, max_tokens, device, int(keep_exact),
                                     ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().oscar_kv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- buffer_quant_k + buffer_quant_v (kv_cache.cpp:194-292), raw inputs ----
    def buffer_quant(self, k, v, stream=None):
        """k, v: bf16 CUDA tensors [B, S, H, d] (raw keys; values pre-rotated
        unless cfg.rotate_v)."""
        n = 0 if k is None else k.shape[1]
        if n > 0:
            shp = (self.B, n, self.H, D)
            _need(k, "buffer_quant k", self.device, "bf16", shp)
            _need(v, "buffer_quant v", self.device, "bf16", shp)
        _check(lib().oscar_kv_append(self._h, _ptr(k), _ptr(v), n, _stream(stream)))

    append = buffer_quant

    # ---- the reference's own call shapes: fp64 rows (kv_cache.hpp:80-84) ------------
    def buffer_quant_k(self, k_t, norms, stream=None):
        """KvCache::buffer_quant_k (kv_cache.cpp:194-249): k_t fp64 CUDA tensor
        [B, n, H, d] of ALREADY transformed keys K_u, norms fp64 [B, n, H]."""
        n = k_t.shape[1]
        _need(k_t, "buffer_quant_k k_t", self.device, "f64", (self.B, n, self.H, D))
        _need(norms, "buffer_quant_k norms", self.device, "f64", (self.B, n, self.H))
        _check(lib().oscar_kv_append_k(self._h, _ptr(k_t), _ptr(norms), n, _stream(stream)))

    def buffer_quant_v(self, v, stream=None):
        """KvCache::buffer_quant_v (kv_cache.cpp:251-292): v fp64 [B, n, H, d], stored as given."""
        n = v.shape[1]
        _need(v, "buffer_quant_v v", self.device, "f64", (self.B, n, self.H, D))
        _check(lib().oscar_kv_append_v(self._h, _ptr(v), n, _stream(stream)))

    def decode_step_f64(self, q, k_t, norms, v, out=None, lse=None, stream=None):
        """decode_step with the current token in the reference's form: q bf16 [B, Hq, d],
        k_t fp64 [B, H, d], norms fp64 [B, H], v fp64 [B, H, d]."""
        import torch

        _need(q, "q", self.device, "bf16", (self.B, self.Hq, D))
        _need(k_t, "k_t", self.device, "f64", (self.B, self.H, D))
        _need(norms, "norms", self.device, "f64", (self.B, self.H))
        _need(v, "v", self.device, "f64", (self.B, self.H, D))
        if out is None:
            out = torch.empty((self.B, self.Hq, D), dtype=torch.float32, device=q.device)
        self._check_out(out, lse)
        _check(lib().oscar_kv_decode_step_f64(self._h, _ptr(q), _ptr(k_t), _ptr(norms), _ptr(v), _ptr(out),
                                              _ptr(lse), _stream(stream)))
        return out

    @property
    def v_tokens(self):
        """(v_packed, v_residual): the value stream's counters (fp64 form)."""
        p, r = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().oscar_kv_stats_v(self._h, ctypes.byref(p), ctypes.byref(r)))
        return p.value, r.value

    # ---- decode_step body (pipeline.cpp:292-323) --------------------------------
    def decode_step(self, q, k, v, out=None, lse=None, stream=None, logits=None):
        """logits: optional fp32 [B, Hq, total_tokens + 1] that receives
        StepOutput.logits (pipeline.hpp:54-58) of this step."""
        import torch

        self._check_step(q, k, v)
        if out is None:
            out = torch.empty((self.B, self.Hq, D), dtype=torch.float32, device=q.device)
        self._check_out(out, lse)
        if logits is None:
            _check(lib().oscar_kv_decode_step(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse),
                                              _stream(stream)))
        else:
            _need(logits, "logits", self.device, "f32", numel=self.B * self.Hq * (self.total_tokens + 1))
            _check(lib().oscar_kv_decode_step_logits(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse),
                                                     _ptr(logits), _stream(stream)))
        return out

    def logits(self, q, k=None, out=None, stream=None):
        """Attention logits q.k/sqrt(d) (natural units) of every query head over
        the cache contents (+ the current token k): fp32 [B, Hq, S]."""
        import torch

        self._check_step(q)
        if k is not None:
            _need(k, "k", self.device, "bf16", (self.B, self.H, D))
        n = self.total_tokens + (1 if k is not None else 0)
        if out is None:
            out = torch.empty((self.B, self.Hq, n), dtype=torch.float32, device=q.device)
        _need(out, "logits", self.device, "f32", numel=self.B * self.Hq * n)
        _check(lib().oscar_kv_logits(self._h, _ptr(q), _ptr(k), _ptr(out), _stream(stream)))
        return out

    def _check_step(self, q, k=None, v=None):
        _need(q, "q", self.device, "bf16", (self.B, self.Hq, D))
        if k is not None or v is not None:
            _need(k, "k", self.device, "bf16", (self.B, self.H, D))
            _need(v, "v", self.device, "bf16", (self.B, self.H, D))

    def _check_out(self, out, lse):
        _need(out, "out", self.device, "f32", numel=self.B * self.Hq * D)
        if lse is not None:
            _need(lse, "lse", self.device, "f32", numel=self.B * self.Hq)

    def attend(self, q, out=None, lse=None, stream=None):
        import torch

        if out is None:
            out = torch.empty((self.B, self.Hq, D), dtype=torch.float32, device=q.device)
        if lse is None:
            lse = torch.empty((self.B, self.Hq), dtype=torch.float32, device=q.device)
        self._check_step(q)
        self._check_out(out, lse)
        _check(lib().oscar_kv_attend(self._h, _ptr(q), _ptr(out), _ptr(lse), _stream(stream)))
        return out, lse

    def attend_publish(self, q, plan: "PeerPlan", epoch: int, k=None, v=None, stream=None):
        """attend (k = v = None) or decode_step whose rows are published to every
        rank of `plan` (fused sequence-shard exchange) instead of returned."""
        self._check_step(q, k, v)
        _check(lib().oscar_kv_attend_publish(self._h, _ptr(q), _ptr(k), _ptr(v), ctypes.byref(plan.c), epoch,
                                             _stream(stream)))

    def decode_step_host(self, q: np.ndarray, k: np.ndarray, v: np.ndarray, out: np.ndarray, lse=None,
                         stream=None):
        """HOST buffers (uint16 bf16 bit patterns for q/k/v, fp32 out)."""
        _check(lib().oscar_kv_decode_step_host(
            self._h, q.ctypes.data, k.ctypes.data, v.ctypes.data, out.ctypes.data,
            None if lse is None else lse.ctypes.data, _stream(stream)))
        return out

    # ---- counters (kv_cache.hpp:67-71) ---------------------------------------------
    def _stats(self):
        p, r, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().oscar_kv_stats(self._h, ctypes.byref(p), ctypes.byref(r), ctypes.byref(f)))
        return p.value, r.value, f.value

    @property
    def packed_tokens(self):
        return self._stats()[0]

    @property
    def residual_tokens(self):
        return self._stats()[1]

    @property
    def total_tokens(self):
        p, r, _ = self._stats()
        return p + r

    @property
    def flush_count(self):
        return self._stats()[2]

    def status(self, clear: bool = False) -> dict:
        """Device-side flags of the quantize/append kernels (oscar_kv_status)."""
        f = ctypes.c_int32()
        _check(lib().oscar_kv_status(self._h, ctypes.byref(f), int(clear)))
        return {"fp16_overflow": bool(f.value & 1), "nonfinite_input": bool(f.value & 2), "raw": f.value}

    def last_launch_count(self) -> int:
        return lib().oscar_kv_last_launch_count(self._h)

    def memory_report(self) -> dict:
        m = _MemReport()
        _check(lib().oscar_kv_memory_report(self._h, ctypes.byref(m)))
        return {n: getattr(m, n) for n, _ in _MemReport._fields_}

    # ---- reference-layout views (parity / checkpoint) -----------------------------
    def export(self, b: int = 0) -> dict:
        """Sequence b in the reference's own layout (see oscar_kv_export)."""
        packed, r, flushes = self._stats()
        H, nb, bits = self.H, packed // R, (self.cfg.bits if self.cfg.quantizes() else 0)
        kp, vp = D * (R // G), R * (D // G)
        arr = {}
        if bits == 2:
            arr["k_payload"] = np.zeros((H, nb, R * D // 8), np.uint16)
            arr["v_payload"] = np.zeros((H, nb, R * D // 8), np.uint16)
        elif bits == 4:
            arr["k_payload"] = np.zeros((H, nb, R * D), np.uint16)
            arr["v_payload"] = np.zeros((H, nb, R * D), np.uint16)
        if bits:
            for kind, n in (("k", kp), ("v", vp)):
                arr[f"{kind}_delta"] = np.zeros((H, nb, n))
                arr[f"{kind}_constant"] = np.zeros((H, nb, n))
                arr[f"{kind}_zp"] = np.zeros((H, nb, n), np.int64)
        else:
            arr["k_raw"] = np.zeros((H, nb, R * D))
            arr["v_raw"] = np.zeros((H, nb, R * D))
        arr["k_norms"] = np.zeros((H, packed))
        arr["k_residual"] = np.zeros((r, H, D))
        arr["k_norms_residual"] = np.zeros(r * H)
        arr["v_residual"] = np.zeros((r, H, D))
        ex = _Export(**{n: (a.ctypes.data if a.size else None) for n, a in arr.items()})
        _check(lib().oscar_kv_export(self._h, b, ctypes.byref(ex)))
        arr.update(packed=packed, residual=r, flushes=flushes, bits=bits)
        return arr

    def dump(self, b: int, path: str):
        """KvCache::dump (kv_cache.cpp:469-507) for sequence b."""
        _check(lib().oscar_kv_dump(self._h, b, path.encode()))

    def load(self, b: int, path: str):
        """KvCache::load (kv_cache.cpp:509-549) into sequence b."""
        _check(lib().oscar_kv_load(self._h, b, path.encode()))

    @classmethod
    def from_kvc1(cls, path: str, q_heads: int, max_tokens: int | None = None, device: int = 0) -> "KvCache":
        """static KvCache::load(path) (kv_cache.hpp:95): a one-sequence cache with
        the file's config, holding the file's contents."""
        cfg, tokens = read_kvc1_config(path)
        c = cls(cfg, batch=1, q_heads=q_heads, max_tokens=max_tokens or tokens + cfg.residual_len, device=device)
        c.load(0, path)
        return c

    def materialize(self, b: int = 0):
        """materialize_k / materialize_v (kv_cache.cpp:327-381) of sequence b."""
        n = self.total_tokens
        k = np.zeros((n, self.H, D))
        v = np.zeros((n, self.H, D))
        _check(lib().oscar_kv_materialize(self._h, b, k.ctypes.data, v.ctypes.data))
        return k, v


class DecodeBatch:
    """decode_step over several caches (e.g. every layer of a model step) in
    one C-ABI call (oscar_kv_decode_step_many).  Pointer arrays are built once
    for fixed q/k/v/out buffers; call run() each step after filling them."""

    def __init__(self, caches, qs, ks, vs, outs, lses=None):
        n = len(caches)
        if not all(len(x) == n for x in (qs, ks, vs, outs)) or (lses is not None and len(lses) != n):
            raise ValueError("DecodeBatch: one q/k/v/out (and lse) per cache")
        for i, c in enumerate(caches):
            c._check_step(qs[i], ks[i], vs[i])
            c._check_out(outs[i], None if lses is None else lses[i])
        arr = ctypes.c_void_p * n
        self.n = n
        self._keep = (caches, qs, ks, vs, outs, lses)
        self.h = arr(*[c._h.value for c in caches])
        self.q = arr(*[_ptr(x) for x in qs])
        self.k = arr(*[_ptr(x) for x in ks])
        self.v = arr(*[_ptr(x) for x in vs])
        self.o = arr(*[_ptr(x) for x in outs])
        self.l = arr(*[_ptr(x) for x in lses]) if lses is not None else None

    def run(self, stream=None):
        _check(lib().oscar_kv_decode_step_many(self.n, self.h, self.q, self.k, self.v, self.o, self.l,
                                               _stream(stream)))


def lse_merge(outs, lses, out=None, lse_out=None, stream=None):
    """Merge P partial attentions: outs [P, rows, d], lses [P, rows] (device)."""
    import torch

    dev = _dev_of(outs, "outs")
    P, rows, d = outs.shape
    _need(outs, "outs", dev, "f32")
    _need(lses, "lses", dev, "f32", (P, rows))
    if out is not None:
        _need(out, "out", dev, "f32", numel=rows * d)
    if lse_out is not None:
        _need(lse_out, "lse_out", dev, "f32", numel=rows)
    if out is None:
        out = torch.empty((rows, d), dtype=torch.float32, device=outs.device)
    _check(lib().oscar_lse_merge(_ptr(outs), _ptr(lses), P, rows, d, _ptr(out), _ptr(lse_out), _stream(stream)))
    return out


# ----------------------------------------------------------------------------- peer exchange (C5)
def peer_area_bytes(world: int, rows: int) -> int:
    """Bytes of one rank's receive area: uint64 (epoch << 32 | fp32) words [2][world][rows][132]."""
    n = lib().oscar_peer_area_bytes(world, rows)
    if n < 0:
        raise ValueError(f"bad peer area shape world={world} rows={rows}")
    return int(n)


class PeerPlan:
    """oscar_peer_plan over receive areas given as device addresses (one per
    rank, as mapped in this process)."""

    def __init__(self, world: int, rank: int, rows: int, areas):
        if len(areas) != world:
            raise ValueError("one receive area per rank")
        self.world, self.rank, self.rows = world, rank, rows
        self.c = _PeerPlan(world, rank, rows)
        for p, a in enumerate(areas):
            self.c.recv[p] = int(a)


def peer_publish_empty(plan: PeerPlan, epoch: int, stream=None):
    _check(lib().oscar_peer_publish_empty(ctypes.byref(plan.c), epoch, _stream(stream)))


def peer_merge(plan: PeerPlan, epoch: int, out, lse=None, status=None, stream=None):
    """Wait for every rank's rows of `epoch` and merge -> out [rows, 128] (device).
    status: optional device int32 tensor, set to 1 (and the rows to NaN) if a
    peer does not publish within ~5 s."""
    dev = _dev_of(out, "out")
    _need(out, "out", dev, "f32", numel=plan.rows * D)
    if lse is not None:
        _need(lse, "lse", dev, "f32", numel=plan.rows)
    if status is not None:
        import torch

        if status.dtype != torch.int32 or not status.is_cuda:
            raise ValueError("status: expected a CUDA int32 tensor")
    _check(lib().oscar_peer_merge(ctypes.byref(plan.c), epoch, _ptr(out), _ptr(lse), _ptr(status),
                                  _stream(stream)))
    return out


def ipc_alloc(nbytes: int, device: int = 0) -> tuple[int, bytes]:
    """Zeroed device allocation + its 64-byte CUDA IPC handle."""
    p = _P()
    h = ctypes.create_string_buffer(64)
    _check(lib().oscar_ipc_alloc(nbytes, device, ctypes.byref(p), h))
    return p.value, h.raw


def ipc_open(handle: bytes, device: int = 0) -> int:
    p = _P()
    _check(lib().oscar_ipc_open(ctypes.create_string_buffer(handle, 64), device, ctypes.byref(p)))
    return p.value


def ipc_close(ptr: int):
    _check(lib().oscar_ipc_close(_P(ptr)))


def ipc_free(ptr: int):
    _check(lib().oscar_ipc_free(_P(ptr)))


def read_kvc1_config(path: str):
    """(PipelineConfig, tokens) of a KVC1 file's manifest (oscar_kvc1_read_config)."""
    c = _Config()
    n = ctypes.c_int64()
    _check(lib().oscar_kvc1_read_config(path.encode(), ctypes.byref(c), ctypes.byref(n)))
    inv_m = {v: k for k, v in METHODS.items()}
    inv_s = {v: k for k, v in SCALINGS.items()}
    cfg = PipelineConfig(method=inv_m[c.method], bits=c.bits, group_size=c.group_size, residual_len=c.residual_len,
                         scaling=inv_s[c.scaling], head_dim=c.head_dim, heads=c.heads, rotate_v=bool(c.rotate_v))
    return cfg, n.value
