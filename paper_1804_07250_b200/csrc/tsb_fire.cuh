// Warp-cooperative heat-bath coins shared by the domino and lozenge sweep
// kernels (sm_100a).
#pragma once

#include "tsb_internal.cuh"

namespace tsb {

// Heat-bath coins of a warp's rotateable active vertices, load-balanced.
// Each lane owns WPL (1 or 2) words (bits `ra`, `rb` rotateable, rb = 0 when
// WPL = 1; `ia`, `ib`: the site
// fires iff (u < p) equals this bit -- domino state 3, lozenge ROT_LOW).
// Site index = r * side + 32 * word + bit, word = wa - WPL * lane + WPL * lane'.
// The warp's sites are queued in shared memory and dealt round-robin to the
// lanes, two independent splitmix64 chains per lane per iteration, so a word
// full of rotateable sites no longer serialises its lane (dense mixed states).
// A site moves 3 -> 12 when u < p_up and 12 -> 3 otherwise
// (_kernels.py:49-55, sweeps.py:102-110); a lozenge star moves to the high
// state when u < p (lozenge.py:575-597).  Only rotateable sites are drawn and
// counter-based draws make the skipping exact.
template <int TM, int WPL = 2>
__device__ __forceinline__ uint2 warp_fire_body(uint32_t ra, uint32_t rb, uint32_t ia, uint32_t ib, uint16_t *queue,
                                        uint32_t *fres, const uint64_t *__restrict__ seedinfo,
                                        const uint64_t *__restrict__ tgrid, uint64_t t, int side, int z, int r,
                                        int wa, uint64_t step) {
    const int lane = threadIdx.x & 31;
    const int cnt = __popc(ra) + __popc(rb);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int pos = incl - cnt;
    // job = is3 << 11 | lane << 6 | word << 5 | bit
    for (uint32_t m = ra; m; m &= m - 1) {
        const int b = __ffs(m) - 1;
        queue[pos++] = (uint16_t)((((ia >> b) & 1u) << 11) | (lane << 6) | b);
    }
    for (uint32_t m = rb; m; m &= m - 1) {
        const int b = __ffs(m) - 1;
        queue[pos++] = (uint16_t)((((ib >> b) & 1u) << 11) | (lane << 6) | 32 | b);
    }
    fres[2 * lane] = 0u;
    fres[2 * lane + 1] = 0u;
    // pad the queue to a multiple of 32 with copies of job 0: a duplicate
    // coin sets the same fire bit again (idempotent), and every round of the
    // loop below then runs two independent splitmix chains per lane without
    // a divergent tail (lanes of a warp issue together, so the padding costs
    // no issue slots)
    const int padded = (total + 31) & ~31;
    __syncwarp();
    if (lane < padded - total) queue[total + lane] = queue[0];
    __syncwarp();
    const uint64_t salt = (step + 1ull) * kGold;
    // site index i = r * side + column, column = 32 * (wa of lane 0) + col,
    // col = 32 * WPL * lane' + 32 * word + bit (the job's low bits); the site
    // key's argument base + (i + 1) * G = kb + col * G
    const uint64_t row_idx = (uint64_t)r * (uint64_t)side + (uint64_t)(int64_t)((wa - WPL * lane) * 32);
    const uint64_t kb = seedinfo[2 * z] + (row_idx + 1ull) * kGold;
    auto col_of = [](uint32_t q) -> uint32_t {
        return WPL == 2 ? (q & 2047u) : (((q >> 6) & 31u) * (32u * WPL) + (q & 63u));
    };
    // below(x, col): the draw's u < p for the site in column col
    auto deal = [&](auto below) {
        int j = lane;
        for (; j + 32 < padded; j += 64) {
            const uint32_t q0 = queue[j], q1 = queue[j + 32];
            const uint32_t c0 = col_of(q0), c1 = col_of(q1);
            // two independent chains for ILP
            const uint64_t x0 = mix64(mix64(kb + (uint64_t)c0 * kGold) + salt);
            const uint64_t x1 = mix64(mix64(kb + (uint64_t)c1 * kGold) + salt);
            const bool f0 = below(x0, c0) == (bool)(q0 >> 11), f1 = below(x1, c1) == (bool)(q1 >> 11);
            // fire word of (lane', word) = fres[2 * lane' + word] (WPL = 1: word 0 only)
            if (f0) atomicOr(&fres[(q0 >> 5) & 63u], 1u << (q0 & 31u));
            if (f1) atomicOr(&fres[(q1 >> 5) & 63u], 1u << (q1 & 31u));
        }
        if (j < padded) {
            const uint32_t q0 = queue[j], c0 = col_of(q0);
            const uint64_t x0 = mix64(mix64(kb + (uint64_t)c0 * kGold) + salt);
            if (below(x0, c0) == (bool)(q0 >> 11)) atomicOr(&fres[(q0 >> 5) & 63u], 1u << (q0 & 31u));
        }
    };
    if (TM == 0 && t == (1ull << 52)) {
        // p = 1/2 (uniform weights): (x >> 11) < 2^52 iff bit 63 of x is 0,
        // which the compiler reads off the last multiply (no final xorshift
        // or 64-bit compare)
        deal([](uint64_t x, uint32_t) { return (int32_t)(uint32_t)(x >> 32) >= 0; });
    } else {
        deal([&](uint64_t x, uint32_t c) {
            const uint64_t tt = TM == 2 ? __ldg(tgrid + row_idx + c) : t;
            return (x >> 11) < tt;
        });
    }
    __syncwarp();
    return make_uint2(fres[2 * lane], fres[2 * lane + 1]);
}

// The call form: a separate function keeps the domino multi-sweep kernels
// within their 40-register budget (inlined: T_max +1 %, C4 +13 %), while the
// lozenge and CFTP pair kernels inline the body (C2 -1.3 %, C5 +4 %).
template <int TM, int WPL = 2>
__device__ __noinline__ uint2 warp_fire(uint32_t ra, uint32_t rb, uint32_t ia, uint32_t ib, uint16_t *queue,
                                        uint32_t *fres, const uint64_t *__restrict__ seedinfo,
                                        const uint64_t *__restrict__ tgrid, uint64_t t, int side, int z, int r,
                                        int wa, uint64_t step) {
    return warp_fire_body<TM, WPL>(ra, rb, ia, ib, queue, fres, seedinfo, tgrid, t, side, z, r, wa, step);
}

}  // namespace tsb
