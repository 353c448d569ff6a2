// peer.cuh -- device side of the fused sequence-shard exchange (C5,
// SURVEY.md §8(e)): the attention kernel's final merge publishes each
// normalised row (O[128], LSE) of this rank straight into every rank's
// receive area over NVLink peer memory, then raises a per-row epoch flag;
// peer_merge_kernel (peer.cu) on each rank waits for the flags and merges
// the rows.  Replaces the NCCL all-gather + lse_merge of the baseline path.
//
// Memory ordering: every lane stores its 16 B of the row and fences at system
// scope, the warp synchronises, and one lane stores the flags with
// st.release.sys; the reader acquires the flag (system scope) before reading.
// Double-buffered by epoch parity: a rank cannot publish epoch e+2 before
// every rank has merged epoch e (its own merge of e+1 needs their e+1 rows,
// published after their merge of e), so parity slots are never overwritten
// while being read.
#pragma once
#include <stdint.h>

#include "kernels.h"

namespace osk {

__device__ __forceinline__ void st_release_sys_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// row slot of rank `src` for epoch parity in a receive area
__device__ __forceinline__ int64_t peer_slot(const PeerPlan &p, uint32_t epoch, int src, int64_t row) {
    return (((int64_t)(epoch & 1u) * p.world + src) * p.rows + row);
}

// one warp: lane holds channels 4*lane..4*lane+3 of the normalised row
__device__ __forceinline__ void peer_publish_row(const PeerPlan &p, uint32_t epoch, int64_t row, float4 o,
                                                 float lse, int lane) {
    const int64_t slot = peer_slot(p, epoch, p.rank, row);
    for (int dst = 0; dst < p.world; ++dst) {
        float *base = p.recv[dst] + slot * PEER_STRIDE;
        *reinterpret_cast<float4 *>(base + lane * 4) = o;
        if (lane == 0) base[128] = lse;
    }
    __threadfence_system();  // each lane's row stores are performed before ...
    __syncwarp();            // ... the warp reconverges and lane 0 raises the flags with release
                             // semantics (cumulative over the stores ordered before the barrier)
    if (lane == 0)
        for (int dst = 0; dst < p.world; ++dst) st_release_sys_u32(p.flags[dst] + slot, epoch);
}

}  // namespace osk
