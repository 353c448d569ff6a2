// split.h -- the stream-K split of the decode-attention work, shared by the
// kernel and the host.
//
// The flattened (sequence*KV-head, pipeline unit) space of `total` units is cut
// into `ncta` contiguous CTA ranges.  Every (b, kv head) segment a CTA touches
// costs a fixed overhead (q fragments, the warp partials, a share of the
// merges) on top of its units, so the split is even in a VIRTUAL space in
// which each segment is preceded by `seg_cost` virtual units:
//   v(u) = bh * (nb + cost + tail) + cost + (u - bh * nb)   (bh = u / nb)
//   CTA c covers virtual [B_c, B_{c+1}), B_c = c * V / ncta, V = (nb + cost + tail) * BH
// `tail` virtual units after each segment charge its owner for the residual
// tiles; cost = tail = 0 is the plain even split.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define OSK_SPLIT_HD __host__ __device__ __forceinline__
#else
#define OSK_SPLIT_HD inline
#endif

namespace osk {

struct Split {
    int64_t nb;      // units per (b, kv head)
    int64_t BH;
    int64_t ncta;
    int64_t cost;    // virtual units before each segment (segment overhead)
    int64_t tail;    // virtual units after each segment (its residual-window tiles)
    OSK_SPLIT_HD int64_t span() const { return nb + cost + tail; }
    OSK_SPLIT_HD int64_t total() const { return nb * BH; }
    OSK_SPLIT_HD int64_t vtotal() const { return span() * BH; }
    // first unit u with v(u) >= B
    OSK_SPLIT_HD int64_t unit_at(int64_t B) const {
        if (B >= vtotal()) return total();
        const int64_t bh = B / span();
        int64_t off = B - bh * span() - cost;
        off = off < 0 ? 0 : off;
        return off >= nb ? (bh + 1) * nb : bh * nb + off;  // inside the tail zone: next segment
    }
    OSK_SPLIT_HD int64_t begin(int64_t c) const { return unit_at(c * vtotal() / ncta); }
    OSK_SPLIT_HD int64_t end(int64_t c) const { return unit_at((c + 1) * vtotal() / ncta); }
    // CTA whose range holds unit u
    OSK_SPLIT_HD int64_t cta_of(int64_t u) const {
        const int64_t bh = u / nb;
        const int64_t v = bh * span() + cost + (u - bh * nb);
        return ((v + 1) * ncta - 1) / vtotal();
    }
};

}  // namespace osk
