"""The C++ host wrapper (include/oscar_kv.hpp) driven by a compiled C++ program
on the GPU -- the call shape a reference-side caller uses:
oscar_b200::KvCache create -> buffer_quant (prefill) -> decode_step x N
(crossing a flush) -> dump -> a second KvCache load -> decode_step, with the
reference's exception types on misuse.  The program's inputs come from a
fixed LCG that this test reproduces in numpy; its outputs and KVC1 dump are
checked against the compiled reference (oracle/_ref)."""
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200.synthetic import bf16_bits_to_f64

from gpu_util import log_err, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_19660_b200")
H, G_, S, STEPS = 2, 4, 380, 6  # 256 packed + 124 window; step 4 fills the window -> flush

PROGRAM = r"""
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "oscar_kv.hpp"

static uint64_t st = 0x9E3779B97F4A7C15ull;
static uint16_t next_bf16(float scale) {  // LCG -> uniform(-2,2)*scale -> bf16 (RNE)
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    float f = ((float)(st >> 40) / 16777216.0f - 0.5f) * 4.0f * scale;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static void *to_dev(const std::vector<uint16_t> &h) {
    void *d = nullptr;
    cudaMalloc(&d, h.size() * 2);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    return d;
}

int main(int argc, char **argv) {
    const int64_t H = @H@, Hq = @HQ@, S = @S@, STEPS = @STEPS@, D = 128;
    const char *dir = argv[1];
    oscar_b200::PipelineConfig pc;
    pc.heads = H;
    pc.bits = 2;
    pc.validate();
    oscar_b200::KvCache cache(pc, /*batch=*/1, Hq, S + STEPS + 8, /*device=*/0);
    // inputs: keys (channels 0-3 offset by +-18 like the TNI recipe), values, queries
    std::vector<uint16_t> k((S + STEPS) * H * D), v((S + STEPS) * H * D), q(STEPS * Hq * D);
    for (int64_t i = 0; i < (S + STEPS) * H * D; ++i) {
        k[i] = next_bf16((i % D) < 4 ? 9.0f : 1.0f);
        v[i] = next_bf16(1.0f);
    }
    for (auto &x : q) x = next_bf16(1.0f);
    void *dk = to_dev(k), *dv = to_dev(v), *dq = to_dev(q);
    float *dout = nullptr;
    cudaMalloc(&dout, Hq * D * 4);
    cache.buffer_quant(dk, dv, S);
    std::vector<float> outs(STEPS * Hq * D);
    for (int64_t t = 0; t < STEPS; ++t) {
        const int64_t off = (S + t) * H * D * 2;  // bytes
        cache.decode_step((char *)dq + t * Hq * D * 2, (char *)dk + off, (char *)dv + off, dout);
        cudaMemcpy(outs.data() + t * Hq * D, dout, Hq * D * 4, cudaMemcpyDeviceToHost);
    }
    std::printf("tokens %lld packed %lld residual %lld flushes %lld\n", (long long)cache.total_tokens(),
                (long long)cache.packed_tokens(), (long long)cache.residual_tokens(), (long long)cache.flush_count());
    std::string dump = std::string(dir) + "/cpp.kvc1";
    cache.dump(0, dump);
    // reload into a second cache and attend the same query: identical output
    oscar_b200::KvCache again(pc, 1, Hq, S + STEPS + 8, 0);
    again.load(0, dump);
    std::vector<float> o1(Hq * D), o2(Hq * D);
    cache.attend(dq, dout, nullptr);
    cudaMemcpy(o1.data(), dout, Hq * D * 4, cudaMemcpyDeviceToHost);
    again.attend(dq, dout, nullptr);
    cudaMemcpy(o2.data(), dout, Hq * D * 4, cudaMemcpyDeviceToHost);
    const bool same = std::memcmp(o1.data(), o2.data(), o1.size() * 4) == 0;
    auto mr = again.memory_report();
    // misuse -> the reference's exception types
    int caught = 0;
    try { oscar_b200::KvCache bad(pc, 1, Hq + 1, 16, 0); } catch (const std::invalid_argument &) { ++caught; }
    try { again.load(0, std::string(dir) + "/missing.kvc1"); } catch (const std::runtime_error &) { ++caught; }
    FILE *f = std::fopen((std::string(dir) + "/outs.bin").c_str(), "wb");
    std::fwrite(outs.data(), 4, outs.size(), f);
    std::fclose(f);
    std::printf("reload_same %d caught %d effbits %.4f\n", same ? 1 : 0, caught, mr.effective_bits_per_value);
    return 0;
}
"""


def program() -> str:
    return (PROGRAM.replace("@HQ@", str(H * G_)).replace("@H@", str(H)).replace("@STEPS@", str(STEPS))
            .replace("@S@", str(S)))


def _lcg_inputs():
    st = 0x9E3779B97F4A7C15
    M = (1 << 64) - 1

    def nxt(scale):
        nonlocal st
        st = (st * 6364136223846793005 + 1442695040888963407) & M
        f = np.float32((np.float32(st >> 40) / np.float32(16777216.0) - np.float32(0.5)) * np.float32(4.0) *
                       np.float32(scale))
        u = int(np.array([f], np.float32).view(np.uint32)[0])
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFFFFFF
        return u >> 16

    D = 128
    n = (S + STEPS) * H * D
    kb = np.zeros(n, np.uint16)
    vb = np.zeros(n, np.uint16)
    for i in range(n):
        kb[i] = nxt(9.0 if (i % D) < 4 else 1.0)
        vb[i] = nxt(1.0)
    qb = np.array([nxt(1.0) for _ in range(STEPS * H * G_ * D)], np.uint16)
    return (bf16_bits_to_f64(kb).reshape(S + STEPS, H, D), bf16_bits_to_f64(vb).reshape(S + STEPS, H, D),
            bf16_bits_to_f64(qb).reshape(STEPS, H * G_, D))


def test_cpp_program_drives_the_device_cache():
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "prog.cpp")
        with open(src, "w") as f:
            f.write(program())
        exe = os.path.join(td, "prog")
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                        src, "-o", exe, "-L", LIBDIR, "-loscar_b200", f"-Wl,-rpath,{LIBDIR}",
                        "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
        r = subprocess.run([exe, td], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        lines = r.stdout.split("\n")
        assert lines[0] == f"tokens {S + STEPS} packed 384 residual 2 flushes 1", r.stdout
        assert lines[1].startswith("reload_same 1 caught 2"), r.stdout
        outs = np.fromfile(os.path.join(td, "outs.bin"), np.float32).reshape(STEPS, H * G_, 128)
        k, v, q = _lcg_inputs()
        ref = ob.RefCache(H=H, bits=2)
        ref.append(k[:S], v[:S])
        for t in range(STEPS):
            o = ref.decode_step(q[t], k[S + t], v[S + t], G_, append=True)
            err = rel_err(outs[t].astype(np.float64), o)
            log_err(f"cpp_wrapper[H=2,g=4,S={S + t}]", err)
            assert err <= 5e-3, (t, err)
        theirs = os.path.join(td, "ref.kvc1")
        ref.dump(theirs)
        assert open(os.path.join(td, "cpp.kvc1"), "rb").read() == open(theirs, "rb").read()


PROGRAM_F64 = r"""
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include "oscar_kv.hpp"

static uint64_t st = 0x2545F4914F6CDD1Dull;
static double next_f64(double scale) {  // LCG -> uniform(-2, 2) * scale, exact in fp64
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return ((double)(st >> 11) * 0x1p-53 - 0.5) * 4.0 * scale;
}

int main(int argc, char **argv) {
    const int64_t H = 2, D = 128, S = 300, Hq = 8;
    const std::string dir = argv[1];
    oscar_b200::PipelineConfig pc;
    pc.heads = H;
    pc.bits = 2;
    // the reference's calls, the reference's types: Tensor3 K_u + norms, Tensor3 V
    oscar_b200::Tensor3 kt(S, H, D), v(S, H, D);
    std::vector<double> norms(S * H);
    for (int64_t t = 0; t < S; ++t)
        for (int64_t h = 0; h < H; ++h) {
            for (int64_t c = 0; c < D; ++c) kt.at(t, h, c) = next_f64(c < 4 ? 8.0 : 1.0);
            for (int64_t c = 0; c < D; ++c) v.at(t, h, c) = next_f64(1.0);
            norms[t * H + h] = 2.0 + next_f64(0.25);
        }
    oscar_b200::KvCache cache(pc, /*batch=*/1, Hq, S + 64, 0);
    cache.buffer_quant_k(kt, norms);
    cache.buffer_quant_v(v);
    cache.dump(0, dir + "/f64.kvc1");
    // static KvCache::load: config from the file
    oscar_b200::KvCache loaded = oscar_b200::KvCache::load(dir + "/f64.kvc1", Hq);
    const oscar_b200::Tensor3 mk = loaded.materialize_k(), mv = loaded.materialize_v();
    FILE *f = std::fopen((dir + "/mat.bin").c_str(), "wb");
    std::fwrite(mk.data.data(), 8, mk.data.size(), f);
    std::fwrite(mv.data.data(), 8, mv.data.size(), f);
    std::fclose(f);
    int caught = 0;
    oscar_b200::KvCache two(pc, /*batch=*/2, Hq, 64, 0);
    try { two.buffer_quant_k(kt, norms); } catch (const std::invalid_argument &) { ++caught; }
    try { cache.buffer_quant(nullptr, nullptr, 0); } catch (const std::logic_error &) { ++caught; }  // form mix
    std::printf("packed %lld residual %lld loaded %lld %lld caught %d\n", (long long)cache.packed_tokens(),
                (long long)cache.residual_tokens(), (long long)loaded.packed_tokens(),
                (long long)loaded.residual_tokens(), caught);
    return 0;
}
"""


def _lcg_f64(S, H, D=128):
    st = 0x2545F4914F6CDD1D
    M = (1 << 64) - 1

    def nxt(scale):
        nonlocal st
        st = (st * 6364136223846793005 + 1442695040888963407) & M
        return (float(st >> 11) * 2.0 ** -53 - 0.5) * 4.0 * scale

    kt = np.zeros((S, H, D))
    v = np.zeros((S, H, D))
    nr = np.zeros(S * H)
    for t in range(S):
        for h in range(H):
            for c in range(D):
                kt[t, h, c] = nxt(8.0 if c < 4 else 1.0)
            for c in range(D):
                v[t, h, c] = nxt(1.0)
            nr[t * H + h] = 2.0 + nxt(0.25)
    return kt, nr, v


def test_cpp_reference_call_shapes():
    """buffer_quant_k(Tensor3 K_u, norms) / buffer_quant_v(Tensor3) from host fp64
    rows, static KvCache::load(path) and Tensor3 materialize_k / materialize_v
    through the C++ wrapper: the dump is the reference's dump byte for byte and
    the materialised rows are the reference's materialize_k / _v exactly."""
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    S, H = 300, 2
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "prog.cpp")
        with open(src, "w") as f:
            f.write(PROGRAM_F64)
        exe = os.path.join(td, "prog")
        subprocess.run(["g++", "-std=c++17", "-O1", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
                        src, "-o", exe, "-L", LIBDIR, "-loscar_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
        r = subprocess.run([exe, td], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.strip() == "packed 256 residual 44 loaded 256 44 caught 2", r.stdout
        kt, nr, v = _lcg_f64(S, H)
        ref = ob.RefCache(H=H, bits=2)
        ref.buffer_quant_k(kt, nr)
        ref.buffer_quant_v(v)
        theirs = os.path.join(td, "ref.kvc1")
        ref.dump(theirs)
        assert open(os.path.join(td, "f64.kvc1"), "rb").read() == open(theirs, "rb").read()
        mat = np.fromfile(os.path.join(td, "mat.bin"), np.float64).reshape(2, S, H, 128)
        rk, rv = ref.materialize()
        assert np.array_equal(mat[0], rk) and np.array_equal(mat[1], rv)
