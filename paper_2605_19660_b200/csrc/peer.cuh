// peer.cuh -- device side of the fused sequence-shard exchange (C5,
// SURVEY.md §8(e)): the attention kernel's final merge publishes each
// normalised row (O[128], LSE) of this rank straight into every rank's
// receive area over NVLink peer memory; peer_merge_kernel (peer.cu) on each
// rank waits for the rows and merges them.  Replaces the NCCL all-gather +
// lse_merge of the baseline path.
//
// Flag-in-word protocol (no memory fences): every 8-byte word of a row is
// (epoch << 32 | fp32 bits), written with single-copy-atomic 64-bit stores
// (two per 16-byte vector store, each element atomic); the reader polls the
// words it needs until their epoch matches, so a word is never read before
// its own payload arrived.  A system-scope fence per row (the previous
// "data, fence.sys, release flag" form) cost ~6 us per fence; this costs two
// 16-byte stores per lane per destination.  Double-buffered by epoch parity:
// a rank cannot publish epoch e+2 before every rank has merged epoch e (its
// own merge of e+1 needs their e+1 rows, published after their merge of e),
// so parity slots are never overwritten while being read.
#pragma once
#include <stdint.h>

#include "kernels.h"

namespace osk {

__device__ __forceinline__ void st_volatile_v2_u64(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_volatile_v2_u64(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ll_word(float x, uint32_t epoch) {
    return ((uint64_t)epoch << 32) | (uint64_t)__float_as_uint(x);
}

// row slot of rank `src` for epoch parity in a receive area (in 8-byte words: * PEER_STRIDE)
__device__ __forceinline__ int64_t peer_slot(const PeerPlan &p, uint32_t epoch, int src, int64_t row) {
    return (((int64_t)(epoch & 1u) * p.world + src) * p.rows + row);
}

// one warp: lane holds channels 4*lane..4*lane+3 of the normalised row
__device__ __forceinline__ void peer_publish_row(const PeerPlan &p, uint32_t epoch, int64_t row, float4 o,
                                                 float lse, int lane) {
    const int64_t slot = peer_slot(p, epoch, p.rank, row);
    const uint64_t w0 = ll_word(o.x, epoch), w1 = ll_word(o.y, epoch), w2 = ll_word(o.z, epoch),
                   w3 = ll_word(o.w, epoch), wl = ll_word(lse, epoch);
    for (int dst = 0; dst < p.world; ++dst) {
        uint64_t *base = p.recv[dst] + slot * PEER_STRIDE;
        st_volatile_v2_u64(base + lane * 4, w0, w1);
        st_volatile_v2_u64(base + lane * 4 + 2, w2, w3);
        if (lane == 0) st_volatile_v2_u64(base + 128, wl, wl);
    }
}

}  // namespace osk
