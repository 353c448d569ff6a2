// peer.cu -- receive side of the fused sequence-shard exchange (peer.cuh):
// one warp per (sequence, query head) row waits for every rank's row of this
// epoch in the local receive area and merges the partial softmaxes
// (O_r, LSE_r) -> (sum_r e^(LSE_r - M) O_r / sum_r e^(LSE_r - M), M + ln sum).
// The exchanged bytes are the C5 message of SURVEY.md §8(d): 14,448 B per
// rank per layer (28 rows x 516 B), i.e. latency-bound; one 32-thread block
// per row keeps the wait + merge to a single short launch.
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
    const float *recv = p.recv[p.rank];
    const uint32_t *flags = p.flags[p.rank];
    // lane src polls rank src's flag (acquire, system scope); the warp barrier then
    // orders every lane's reads after those acquires; the rows are read from L2
    // (__ldcg: never a stale L1 line of an earlier epoch)
    bool ok = true;
    if (lane < p.world) {
        const uint32_t *f = flags + peer_slot(p, epoch, lane, row);
        if (ld_acquire_sys_u32(f) != epoch) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_sys_u32(f) != epoch) {
                __nanosleep(64);
                if (globaltimer_ns() - t0 > 5000000000ull) {  // a peer never published: fail loudly, don't hang
                    ok = false;
                    break;
                }
            }
        }
    }
    if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0 && status) atomicExch(status, 1);
        reinterpret_cast<float4 *>(out + row * 128)[lane] = make_float4(CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F,
                                                                          CUDART_NAN_F);
        if (lse_out && lane == 0) lse_out[row] = CUDART_NAN_F;
        return;
    }
    __syncwarp();  // memory ordering: the acquires above happen before every lane's reads below
    // lane src < world holds rank src's LSE
    const float my_l = lane < p.world ? __ldcg(recv + peer_slot(p, epoch, lane, row) * PEER_STRIDE + 128)
                                      : -CUDART_INF_F;
    float M = my_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
    float L = 0.f;
    for (int src = 0; src < p.world; ++src) {
        const float *r = recv + peer_slot(p, epoch, src, row) * PEER_STRIDE;
        const float l = __shfl_sync(0xffffffffu, my_l, src);
        const float w = (l == -CUDART_INF_F) ? 0.f : __expf(l - M);
        const float4 v = __ldcg(reinterpret_cast<const float4 *>(r) + lane);
        O.x += v.x * w;
        O.y += v.y * w;
        O.z += v.z * w;
        O.w += v.w * w;
        L += w;
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
