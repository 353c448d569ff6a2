"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes bindings to the two CPU checkers:

* ``Ref``  -- the UNMODIFIED reference library compiled from
  /root/reference/proj/src by oracle/Makefile into ``oracle/_ref`` (the real
  reference, driven through its own C++ API via ``ref_shim.cpp``);
* ``Port`` -- our plain-C restatement ``oracle/oscar_oracle.c``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module.  The product path (``paper_2605_19660_b200``) never does.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "liboscar_ref.so")
PORT_SO = os.path.join(HERE, "_build", "liboscar_oracle.so")

METHODS = {"fp": 0, "kivi": 1, "rotate-only": 2, "scale-only": 3, "oscar": 4}
SCALINGS = {"l2": 0, "rsqrt": 1, "max": 2, "mean-abs": 3}

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u16p = ctypes.POINTER(ctypes.c_uint16)


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


def build(with_ref: bool = True) -> None:
    """Build the checkers (make -C oracle).  _ref needs /root/reference."""
    import subprocess

    targets = ["port"]
    if with_ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_use_threads(n: int) -> int:
    """Run the compiled reference's OpenMP regions on n threads (all host
    cores for the CPU baseline); returns the thread count in effect."""
    return int(Ref.lib().ref_set_num_threads(int(n)))


# --------------------------------------------------------------------------
@dataclass
class ExportedCache:
    """A cache in the reference's own layout (kv_cache.hpp:38-43, 104-122)."""

    bits: int
    H: int
    d: int
    R: int
    G: int
    packed_tokens: int
    residual_tokens: int
    flush_count: int
    # per head: list of blocks; each block: dict(delta, zp, constant, codes | raw)
    k_blocks: list = field(default_factory=list)
    v_blocks: list = field(default_factory=list)
    k_norms: list = field(default_factory=list)  # per head fp64 [packed]
    k_residual: np.ndarray | None = None  # [r, H, d] fp64
    k_norms_residual: np.ndarray | None = None  # [r*H]
    v_residual: np.ndarray | None = None


def parse_kvc1(path: str) -> ExportedCache:
    """Parse a KVC1 dump (kv_cache.cpp:469-507, README.md:123-130)."""
    with open(path, "rb") as f:
        manifest = json.loads(f.readline())
        body = f.read()
    off = 0

    def take(dtype, n):
        nonlocal off
        a = np.frombuffer(body, dtype=dtype, count=n, offset=off).copy()
        off += a.nbytes
        return a

    H, d, R, G, bits = manifest["H"], manifest["d_h"], manifest["R"], manifest["G"], manifest["b"]

    def read_blocks(sizes):
        out = []
        for s in sizes:
            n = s["params"]
            p = take(np.uint8, 24 * n).reshape(n, 24) if n else np.zeros((0, 24), np.uint8)
            blk = {
                "delta": p[:, 0:8].copy().view(np.float64).reshape(-1),
                "zp": p[:, 8:16].copy().view(np.int64).reshape(-1),
                "constant": p[:, 16:24].copy().view(np.float64).reshape(-1),
                "words": take(np.uint16, s["words"]),
                "packed_count": s["packed_count"],
                "codes": take(np.uint16, s["codes"]),
                "raw": take(np.float64, s["raw"]),
            }
            out.append(blk)
        return out

    ec = ExportedCache(bits, H, d, R, G, manifest["S_packed"], manifest["residual_tokens"],
                       manifest["flush_count"])
    for h in range(H):
        ec.k_blocks.append(read_blocks(manifest["k_blocks"][h]))
        ec.k_norms.append(take(np.float64, manifest["S_packed"]))
    r = manifest["residual_tokens"]
    ec.k_residual = take(np.float64, r * H * d).reshape(r, H, d)
    ec.k_norms_residual = take(np.float64, r * H)
    for h in range(H):
        ec.v_blocks.append(read_blocks(manifest["v_blocks"][h]))
    rv = manifest["v_residual_tokens"]
    ec.v_residual = take(np.float64, rv * H * d).reshape(rv, H, d)
    assert off == len(body), "trailing bytes in KVC1 dump"
    for blocks in ec.k_blocks + ec.v_blocks:
        for b in blocks:
            if bits == 2 and b["words"].size:
                b["codes"] = unpack_2bit_np(b["words"], b["packed_count"])
    return ec


def unpack_2bit_np(words: np.ndarray, n: int) -> np.ndarray:
    i = np.arange(n)
    return ((words[i // 8] >> (2 * (i % 8))) & 3).astype(np.uint16)


def pack_2bit_np(codes: np.ndarray) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint16)
    n = codes.size
    words = np.zeros((n + 7) // 8, dtype=np.uint16)
    i = np.arange(n)
    np.bitwise_or.at(words, i // 8, (codes.astype(np.uint16) << (2 * (i % 8)).astype(np.uint16)))
    return words


# --------------------------------------------------------------------------
class _Lib:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            cls._lib = ctypes.CDLL(cls.SO)
            cls._setup(cls._lib)
        return cls._lib


class Ref(_Lib):
    """The compiled reference (oracle/_ref/liboscar_ref.so)."""

    SO = REF_SO

    @staticmethod
    def _setup(L):
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_cache_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_void_p)]
        L.ref_cache_destroy.argtypes = [ctypes.c_void_p]
        L.ref_cache_append.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int64]
        L.ref_cache_stats.argtypes = [ctypes.c_void_p, _i64p]
        L.ref_cache_memory_report.argtypes = [ctypes.c_void_p, _i64p, _dp]
        L.ref_cache_dump.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.ref_cache_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.ref_cache_materialize.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.ref_decode_step.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_int64, _dp, ctypes.c_int]
        L.ref_decode_step_logits.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_int64, _dp, _dp,
                                             ctypes.c_int]
        L.ref_cache_buffer_quant_k.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int64]
        L.ref_cache_buffer_quant_v.argtypes = [ctypes.c_void_p, _dp, ctypes.c_int64]
        L.ref_decode_step_f64.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp, ctypes.c_int64, _dp, ctypes.c_int]
        L.ref_crit7_inputs.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, _dp, _dp, _dp, _dp, _dp]
        L.ref_simulate_fidelity.argtypes = [ctypes.c_int64, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                            _dp, _dp, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                            _i64p]
        L.ref_preprocess.argtypes = [ctypes.c_int64, ctypes.c_int64, _dp, _dp, _dp, _dp]
        L.ref_fht.argtypes = [_dp, ctypes.c_int64]
        L.ref_token_scale.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                      _dp, _dp, _i64p]
        L.ref_quant_params.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp, _i64p, _dp]
        L.ref_pack_2bit.argtypes = [_u16p, ctypes.c_int64, _u16p]
        L.ref_attention.argtypes = [_dp, ctypes.c_int64, _dp, _dp, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, _dp]
        L.ref_num_threads.restype = ctypes.c_int
        L.ref_set_num_threads.restype = ctypes.c_int
        L.ref_set_num_threads.argtypes = [ctypes.c_int]

    @classmethod
    def check(cls, rc):
        if rc != 0:
            msg = cls.lib().ref_last_error().decode()
            raise {1: ValueError, 2: RuntimeError}.get(rc, OSError)(msg)


class RefCache:
    """reference KvCache + apply_method transforms, via ref_shim.cpp."""

    def __init__(self, method="oscar", bits=2, G=32, R=128, scaling="l2", d=128, H=1,
                 rotate_v=False, _handle=None):
        L = Ref.lib()
        self.H, self.d = H, d
        if _handle is not None:
            self.h = _handle
            return
        h = ctypes.c_void_p()
        Ref.check(L.ref_cache_create(METHODS[method], bits, G, R, SCALINGS[scaling], d, H,
                                     int(rotate_v), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            Ref.lib().ref_cache_destroy(self.h)
            self.h = None

    def append(self, xk: np.ndarray, xv: np.ndarray):
        xk = np.ascontiguousarray(xk, dtype=np.float64)
        xv = np.ascontiguousarray(xv, dtype=np.float64)
        Ref.check(Ref.lib().ref_cache_append(self.h, _ptr(xk), _ptr(xv), xk.shape[0]))

    def buffer_quant_k(self, k_t: np.ndarray, norms: np.ndarray):
        """KvCache::buffer_quant_k(K_u [S,H,d], norms [S*H]) -- the reference's own call."""
        k_t = np.ascontiguousarray(k_t, dtype=np.float64)
        norms = np.ascontiguousarray(norms, dtype=np.float64).reshape(-1)
        Ref.check(Ref.lib().ref_cache_buffer_quant_k(self.h, _ptr(k_t), _ptr(norms), k_t.shape[0]))

    def buffer_quant_v(self, v: np.ndarray):
        v = np.ascontiguousarray(v, dtype=np.float64)
        Ref.check(Ref.lib().ref_cache_buffer_quant_v(self.h, _ptr(v), v.shape[0]))

    def decode_step_f64(self, q_raw, k_t, norms, v, g, append=True):
        """decode_step with the current token in the cache's form (tr.k [H,d], tr.norms [H], xv [H,d])."""
        q = np.ascontiguousarray(q_raw, np.float64)
        kt = np.ascontiguousarray(k_t, np.float64)
        nr = np.ascontiguousarray(norms, np.float64).reshape(-1)
        vv = np.ascontiguousarray(v, np.float64)
        out = np.zeros((self.H * g, self.d))
        Ref.check(Ref.lib().ref_decode_step_f64(self.h, _ptr(q), _ptr(kt), _ptr(nr), _ptr(vv), g, _ptr(out),
                                                int(append)))
        return out

    def stats(self):
        out = np.zeros(4, np.int64)
        Ref.lib().ref_cache_stats(self.h, _ptr(out, _i64p))
        return dict(packed=int(out[0]), residual=int(out[1]), total=int(out[2]), flushes=int(out[3]))

    def memory_report(self):
        out = np.zeros(8, np.int64)
        eff = ctypes.c_double()
        Ref.lib().ref_cache_memory_report(self.h, _ptr(out, _i64p), ctypes.byref(eff))
        keys = ["packed_tokens", "residual_tokens", "packed_k_payload_bits", "packed_v_payload_bits",
                "residual_k_payload_bits", "residual_v_payload_bits", "k_norm_bits", "param_bits"]
        r = {k: int(v) for k, v in zip(keys, out)}
        r["effective_bits_per_value"] = eff.value
        return r

    def dump(self, path: str):
        Ref.check(Ref.lib().ref_cache_dump(self.h, path.encode()))

    @classmethod
    def load(cls, path: str, H: int, d: int) -> "RefCache":
        h = ctypes.c_void_p()
        Ref.check(Ref.lib().ref_cache_load(path.encode(), ctypes.byref(h)))
        return cls(H=H, d=d, _handle=h)

    def export(self, tmpdir: str) -> ExportedCache:
        path = os.path.join(tmpdir, f"ref_{id(self)}.kvc1")
        self.dump(path)
        try:
            return parse_kvc1(path)
        finally:
            os.remove(path)

    def materialize(self):
        n = self.stats()["total"]
        k = np.zeros((n, self.H, self.d))
        v = np.zeros((n, self.H, self.d))
        Ref.check(Ref.lib().ref_cache_materialize(self.h, _ptr(k), _ptr(v)))
        return k, v

    def decode_step(self, q_raw, k_raw, v_raw, g, append=True):
        q = np.ascontiguousarray(q_raw, np.float64)
        k = np.ascontiguousarray(k_raw, np.float64)
        v = np.ascontiguousarray(v_raw, np.float64)
        out = np.zeros((self.H * g, self.d))
        Ref.check(Ref.lib().ref_decode_step(self.h, _ptr(q), _ptr(k), _ptr(v), g, _ptr(out), int(append)))
        return out


    def decode_step_logits(self, q_raw, k_raw, v_raw, g, append=True):
        """decode_step + StepOutput.logits [Hq, total + 1] (natural units)."""
        q = np.ascontiguousarray(q_raw, np.float64)
        k = np.ascontiguousarray(k_raw, np.float64)
        v = np.ascontiguousarray(v_raw, np.float64)
        total = self.stats()["total"] + 1
        out = np.zeros((self.H * g, self.d))
        lg = np.zeros((self.H * g, total))
        Ref.check(Ref.lib().ref_decode_step_logits(self.h, _ptr(q), _ptr(k), _ptr(v), g, _ptr(out), _ptr(lg),
                                                   int(append)))
        return out, lg


MEMORY_FIELDS = ["packed_tokens", "residual_tokens", "packed_k_payload_bits", "packed_v_payload_bits",
                 "residual_k_payload_bits", "residual_v_payload_bits", "k_norm_bits", "param_bits"]


def ref_crit7_inputs(seed: int, S: int = 256, Dn: int = 64, heads: int = 4, d_h: int = 128):
    """Acceptance criterion 7's inputs for `seed` (acceptance_main.cpp:282-312):
    generate(TniSpec) hidden rows [(S+Dn), heads*d_h] and the make_sim_stub
    weights (w_q, w_k, w_v, w_o), all from the compiled reference."""
    dm = heads * d_h
    hidden = np.zeros((S + Dn, dm))
    w = [np.zeros((dm, dm)) for _ in range(4)]
    Ref.check(Ref.lib().ref_crit7_inputs(seed, S, Dn, heads, d_h, _ptr(hidden), *[_ptr(x) for x in w]))
    return hidden, w


def ref_simulate_fidelity(hidden, S: int, weights, method: str, bits: int = 2, heads: int = 4, d_h: int = 128,
                          scaling: str = "l2") -> dict:
    """The reference's simulate_fidelity (pipeline.cpp:359-408) on these inputs."""
    hidden = np.ascontiguousarray(hidden, np.float64)
    Dn = hidden.shape[0] - S
    ws = [np.ascontiguousarray(x, np.float64) for x in weights]
    o6 = np.zeros(6)
    m8 = np.zeros(8, np.int64)
    Ref.check(Ref.lib().ref_simulate_fidelity(heads, d_h, _ptr(hidden), S, Dn, *[_ptr(x) for x in ws],
                                              METHODS[method], bits, SCALINGS[scaling], _ptr(o6), _ptr(m8, _i64p)))
    mem = {k: int(v) for k, v in zip(MEMORY_FIELDS, m8)}
    mem["effective_bits_per_value"] = float(o6[5])
    return {"output_mse": float(o6[0]), "logit_mse": float(o6[1]), "prefill_output_mse": float(o6[2]),
            "flushes": int(o6[3]), "decode_steps": int(o6[4]), "memory": mem}


def ref_preprocess(w_v, w_o, heads: int = 4, d_h: int = 128):
    """preprocess (pipeline.cpp:38-78): folded (W_V, W_O)."""
    wv = np.ascontiguousarray(w_v, np.float64)
    wo = np.ascontiguousarray(w_o, np.float64)
    a, b = np.zeros_like(wv), np.zeros_like(wo)
    Ref.check(Ref.lib().ref_preprocess(heads, d_h, _ptr(wv), _ptr(wo), _ptr(a), _ptr(b)))
    return a, b


def ref_fht(v: np.ndarray) -> np.ndarray:
    v = np.array(v, dtype=np.float64)
    Ref.check(Ref.lib().ref_fht(_ptr(v), v.size))
    return v


def ref_apply_k(x: np.ndarray, method="oscar", scaling="l2"):
    """apply_method's key half (pipeline.cpp:224-236) by the compiled reference:
    x [S, H, d] fp64 -> (K_u [S, H, d], norms [S*H])."""
    x = np.array(x, dtype=np.float64)
    rot = method in ("rotate-only", "oscar")
    sc = method in ("scale-only", "oscar")
    if rot:
        x = np.stack([np.stack([ref_fht(x[t, h]) for h in range(x.shape[1])]) for t in range(x.shape[0])])
    if sc:
        ku, nr, _ = ref_token_scale(x, scaling)
        return ku, nr
    return x, np.ones(x.shape[0] * x.shape[1])


def ref_token_scale(x: np.ndarray, scaling="l2"):
    x = np.ascontiguousarray(x, np.float64)
    S, H, d = x.shape
    sc = np.zeros_like(x)
    nr = np.zeros(S * H)
    deg = ctypes.c_int64()
    Ref.check(Ref.lib().ref_token_scale(_ptr(x), S, H, d, SCALINGS[scaling], _ptr(sc), _ptr(nr),
                                        ctypes.byref(deg)))
    return sc, nr, deg.value


def ref_quant_params(x, bits):
    x = np.ascontiguousarray(x, np.float64)
    dl, c = ctypes.c_double(), ctypes.c_double()
    zp = ctypes.c_int64()
    Ref.check(Ref.lib().ref_quant_params(_ptr(x), x.size, bits, ctypes.byref(dl), ctypes.byref(zp),
                                         ctypes.byref(c)))
    return dl.value, zp.value, c.value


def ref_pack_2bit(codes):
    codes = np.ascontiguousarray(codes, np.uint16)
    words = np.zeros((codes.size + 7) // 8, np.uint16)
    Ref.check(Ref.lib().ref_pack_2bit(_ptr(codes, _u16p), codes.size, _ptr(words, _u16p)))
    return words


def ref_attention(q, k, v):
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    Tq, H, d = q.shape
    out = np.zeros_like(q)
    Ref.check(Ref.lib().ref_attention(_ptr(q), Tq, _ptr(k), _ptr(v), k.shape[0], H, d, _ptr(out)))
    return out


# --------------------------------------------------------------------------
class Port(_Lib):
    """Our C restatement (oracle/_build/liboscar_oracle.so)."""

    SO = PORT_SO

    @staticmethod
    def _setup(L):
        L.oo_fht.argtypes = [_dp, ctypes.c_int64]
        L.oo_fast_rsqrt.argtypes = [ctypes.c_double]
        L.oo_fast_rsqrt.restype = ctypes.c_double
        L.oo_token_scale.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _dp, _dp]
        L.oo_token_scale.restype = ctypes.c_int64
        L.oo_quant_params.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp, _i64p, _dp]
        L.oo_quantize_one.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
        L.oo_quantize_one.restype = ctypes.c_uint16
        L.oo_dequantize_one.argtypes = [ctypes.c_uint16, ctypes.c_double, ctypes.c_int64, ctypes.c_double]
        L.oo_dequantize_one.restype = ctypes.c_double
        L.oo_pack_2bit.argtypes = [_u16p, ctypes.c_int64, _u16p]
        L.oo_unpack_2bit.argtypes = [_u16p, ctypes.c_int64, _u16p]
        L.oo_attention.argtypes = [_dp, ctypes.c_int64, _dp, _dp, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int64, _dp]
        L.oo_cache_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        L.oo_cache_create.restype = ctypes.c_void_p
        L.oo_cache_destroy.argtypes = [ctypes.c_void_p]
        L.oo_cache_append.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int64]
        L.oo_cache_stats.argtypes = [ctypes.c_void_p, _i64p]
        L.oo_cache_num_blocks.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64]
        L.oo_cache_num_blocks.restype = ctypes.c_int64
        L.oo_cache_block.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _u16p,
                                     _dp, _i64p, _dp, _dp]
        L.oo_cache_block.restype = ctypes.c_int64
        L.oo_cache_k_norms.argtypes = [ctypes.c_void_p, ctypes.c_int64, _dp]
        L.oo_cache_residual.argtypes = [ctypes.c_void_p, _dp, _dp, _dp]
        L.oo_cache_materialize.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.oo_decode_step.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_int64, _dp, ctypes.c_int]


class PortCache:
    """C restatement of KvCache + apply_method (oscar_oracle.c)."""

    def __init__(self, method="oscar", bits=2, G=32, R=128, scaling="l2", d=128, H=1, rotate_v=False):
        L = Port.lib()
        self.h = L.oo_cache_create(METHODS[method], bits, G, R, SCALINGS[scaling], d, H, int(rotate_v))
        if not self.h:
            raise ValueError("oracle: invalid config")
        self.H, self.d, self.R, self.G, self.bits = H, d, R, G, bits
        self.quantizes = method != "fp" and bits != 0

    def __del__(self):
        if getattr(self, "h", None):
            Port.lib().oo_cache_destroy(self.h)
            self.h = None

    def append(self, xk, xv):
        xk = np.ascontiguousarray(xk, np.float64)
        xv = np.ascontiguousarray(xv, np.float64)
        rc = Port.lib().oo_cache_append(self.h, _ptr(xk), _ptr(xv), xk.shape[0])
        if rc:
            raise RuntimeError("residual window overflow")

    def stats(self):
        out = np.zeros(4, np.int64)
        Port.lib().oo_cache_stats(self.h, _ptr(out, _i64p))
        return dict(packed=int(out[0]), residual=int(out[1]), total=int(out[2]), flushes=int(out[3]))

    def export(self) -> ExportedCache:
        L = Port.lib()
        st = self.stats()
        H, d, R, G = self.H, self.d, self.R, self.G
        ec = ExportedCache(self.bits, H, d, R, G, st["packed"], st["residual"], st["flushes"])
        for is_v, dst in ((0, ec.k_blocks), (1, ec.v_blocks)):
            for h in range(H):
                blocks = []
                for b in range(L.oo_cache_num_blocks(self.h, is_v, h)):
                    npar = (R // G) * d if not is_v else R * (d // G)
                    codes = np.zeros(R * d, np.uint16)
                    dl = np.zeros(npar)
                    zp = np.zeros(npar, np.int64)
                    cst = np.zeros(npar)
                    raw = np.zeros(R * d)
                    n = L.oo_cache_block(self.h, is_v, h, b, _ptr(codes, _u16p), _ptr(dl), _ptr(zp, _i64p),
                                         _ptr(cst), _ptr(raw))
                    if n:
                        blocks.append(dict(codes=codes, delta=dl, zp=zp, constant=cst, raw=np.zeros(0)))
                    else:
                        blocks.append(dict(codes=np.zeros(0, np.uint16), delta=np.zeros(0),
                                           zp=np.zeros(0, np.int64), constant=np.zeros(0), raw=raw))
                dst.append(blocks)
        for h in range(H):
            n = np.zeros(st["packed"])
            L.oo_cache_k_norms(self.h, h, _ptr(n))
            ec.k_norms.append(n)
        r = st["residual"]
        kr = np.zeros((r, H, d))
        kn = np.zeros(r * H)
        vr = np.zeros((r, H, d))
        L.oo_cache_residual(self.h, _ptr(kr), _ptr(kn), _ptr(vr))
        ec.k_residual, ec.k_norms_residual, ec.v_residual = kr, kn, vr
        return ec

    def materialize(self):
        n = self.stats()["total"]
        k = np.zeros((n, self.H, self.d))
        v = np.zeros((n, self.H, self.d))
        Port.lib().oo_cache_materialize(self.h, _ptr(k), _ptr(v))
        return k, v

    def decode_step(self, q_raw, k_raw, v_raw, g, append=True):
        q = np.ascontiguousarray(q_raw, np.float64)
        k = np.ascontiguousarray(k_raw, np.float64)
        v = np.ascontiguousarray(v_raw, np.float64)
        out = np.zeros((self.H * g, self.d))
        rc = Port.lib().oo_decode_step(self.h, _ptr(q), _ptr(k), _ptr(v), g, _ptr(out), int(append))
        if rc:
            raise RuntimeError("residual window overflow")
        return out


def port_fht(v):
    v = np.array(v, dtype=np.float64)
    Port.lib().oo_fht(_ptr(v), v.size)
    return v


def port_token_scale(x, scaling="l2"):
    x = np.ascontiguousarray(x, np.float64)
    S, H, d = x.shape
    sc = np.zeros_like(x)
    nr = np.zeros(S * H)
    deg = Port.lib().oo_token_scale(_ptr(x), S, H, d, SCALINGS[scaling], _ptr(sc), _ptr(nr))
    return sc, nr, deg


def port_quant_params(x, bits):
    x = np.ascontiguousarray(x, np.float64)
    dl, c = ctypes.c_double(), ctypes.c_double()
    zp = ctypes.c_int64()
    Port.lib().oo_quant_params(_ptr(x), x.size, bits, ctypes.byref(dl), ctypes.byref(zp), ctypes.byref(c))
    return dl.value, zp.value, c.value


def port_pack_2bit(codes):
    codes = np.ascontiguousarray(codes, np.uint16)
    words = np.zeros((codes.size + 7) // 8, np.uint16)
    Port.lib().oo_pack_2bit(_ptr(codes, _u16p), codes.size, _ptr(words, _u16p))
    return words


def port_attention(q, k, v):
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    Tq, H, d = q.shape
    out = np.zeros_like(q)
    Port.lib().oo_attention(_ptr(q), Tq, _ptr(k), _ptr(v), k.shape[0], H, d, _ptr(out))
    return out


def caches_equal(a: ExportedCache, b: ExportedCache, check_words: bool = True) -> list:
    """Bit-exact comparison of two exported caches; returns a list of mismatches."""
    errs = []
    for name in ("packed_tokens", "residual_tokens", "flush_count"):
        if getattr(a, name) != getattr(b, name):
            errs.append(f"{name}: {getattr(a, name)} != {getattr(b, name)}")
    for kind in ("k_blocks", "v_blocks"):
        A, B = getattr(a, kind), getattr(b, kind)
        for h in range(len(A)):
            if len(A[h]) != len(B[h]):
                errs.append(f"{kind}[{h}] block count {len(A[h])} != {len(B[h])}")
                continue
            for i, (x, y) in enumerate(zip(A[h], B[h])):
                for f in ("codes", "delta", "zp", "constant", "raw"):
                    xa, ya = np.asarray(x[f]), np.asarray(y[f])
                    if xa.shape != ya.shape or not np.array_equal(xa.view(np.uint8), ya.view(np.uint8)):
                        n = int(np.sum(xa != ya)) if xa.shape == ya.shape else -1
                        errs.append(f"{kind}[{h}][{i}].{f} differs ({n} entries)")
    for h in range(len(a.k_norms)):
        if not np.array_equal(a.k_norms[h].view(np.uint8), b.k_norms[h].view(np.uint8)):
            errs.append(f"k_norms[{h}] differ")
    for f in ("k_residual", "k_norms_residual", "v_residual"):
        x, y = getattr(a, f), getattr(b, f)
        if x.shape != y.shape or not np.array_equal(x.view(np.uint8), y.view(np.uint8)):
            errs.append(f"{f} differs")
    return errs
