// peer.cu -- receive side of the fused sequence-shard exchange (peer.cuh):
// one warp per (sequence, query head) row waits for every rank's row of this
// epoch in the local receive area (flag-in-word: each 8-byte word carries its
// epoch) and merges the partial softmaxes
// (O_r, LSE_r) -> (sum_r e^(LSE_r - M) O_r / sum_r e^(LSE_r - M), M + ln sum).
// The exchanged payload is the C5 message of SURVEY.md §8(d): 14,448 B per
// rank per layer (28 rows x 516 B; 29.6 KB on the wire with the epochs), i.e.
// latency-bound; one 32-thread block per row keeps the wait + merge to a
// single short launch.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "kernels.h"
#include "peer.cuh"

namespace osk {

namespace {

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void peer_merge_kernel(const PeerPlan p, uint32_t epoch, float *out, float *lse_out, int *status) {
    const int64_t row = blockIdx.x;
    const int lane = threadIdx.x;
    const uint64_t *recv = p.recv[p.rank];
    // every lane polls the words it reads (flag-in-word, peer.cuh): lane src < world the
    // LSE word of rank src, every lane its 4 channel words of every rank
    bool ok = true;
    uint64_t t0 = 0;
    auto expired = [&]() {  // a peer never published: fail loudly after ~5 s, don't hang
        if (t0 == 0) t0 = globaltimer_ns();
        __nanosleep(32);
        return globaltimer_ns() - t0 > 5000000000ull;
    };
    float my_l = -CUDART_INF_F;
    if (lane < p.world) {
        const uint64_t *w = recv + peer_slot(p, epoch, lane, row) * PEER_STRIDE + 128;
        uint64_t v = ld_volatile_u64(w);
        while ((uint32_t)(v >> 32) != epoch && ok) {
            if (expired()) ok = false;
            v = ld_volatile_u64(w);
        }
        my_l = __uint_as_float((uint32_t)v);
    }
    float M = my_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
    float L = 0.f;
    for (int src = 0; src < p.world; ++src) {
        const uint64_t *r = recv + peer_slot(p, epoch, src, row) * PEER_STRIDE + lane * 4;
        uint64_t a, b, c, d;
        ld_volatile_v2_u64(r, a, b);
        ld_volatile_v2_u64(r + 2, c, d);
        while (ok && ((uint32_t)(a >> 32) != epoch || (uint32_t)(b >> 32) != epoch ||
                      (uint32_t)(c >> 32) != epoch || (uint32_t)(d >> 32) != epoch)) {
            if (expired()) ok = false;
            ld_volatile_v2_u64(r, a, b);
            ld_volatile_v2_u64(r + 2, c, d);
        }
        const float l = __shfl_sync(0xffffffffu, my_l, src);
        const float w = (l == -CUDART_INF_F) ? 0.f : __expf(l - M);
        O.x += __uint_as_float((uint32_t)a) * w;
        O.y += __uint_as_float((uint32_t)b) * w;
        O.z += __uint_as_float((uint32_t)c) * w;
        O.w += __uint_as_float((uint32_t)d) * w;
        L += w;
    }
    if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0 && status) atomicExch(status, 1);
        reinterpret_cast<float4 *>(out + row * 128)[lane] = make_float4(CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F,
                                                                          CUDART_NAN_F);
        if (lse_out && lane == 0) lse_out[row] = CUDART_NAN_F;
        return;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    reinterpret_cast<float4 *>(out + row * 128)[lane] = make_float4(O.x * inv, O.y * inv, O.z * inv, O.w * inv);
    if (lse_out && lane == 0) lse_out[row] = L > 0.f ? M + __logf(L) : -CUDART_INF_F;
}

__global__ void peer_publish_empty_kernel(const PeerPlan p, uint32_t epoch) {
    peer_publish_row(p, epoch, blockIdx.x, make_float4(0.f, 0.f, 0.f, 0.f), -CUDART_INF_F, threadIdx.x);
}

}  // namespace

cudaError_t launch_peer_merge(const PeerPlan &p, uint32_t epoch, float *out, float *lse, int *status,
                              cudaStream_t st) {
    if (p.rows <= 0) return cudaSuccess;
    peer_merge_kernel<<<(unsigned)p.rows, 32, 0, st>>>(p, epoch, out, lse, status);
    return cudaGetLastError();
}

cudaError_t launch_peer_publish_empty(const PeerPlan &p, uint32_t epoch, cudaStream_t st) {
    if (p.rows <= 0) return cudaSuccess;
    peer_publish_empty_kernel<<<(unsigned)p.rows, 32, 0, st>>>(p, epoch);
    return cudaGetLastError();
}

}  // namespace osk
