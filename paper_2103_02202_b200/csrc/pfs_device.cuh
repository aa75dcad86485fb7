// Device helpers shared by the frame kernels (pfs_kernels.cu, pfs_colkernel.cu):
// the Philox4x32-10 generator, the coin-row and noise-draw schedules of
// DESIGN.md §4, Pauli patterns, mbarrier / bulk-copy (TMA) primitives and the
// 32x32 warp bit transpose.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pfs_internal.h"

#ifndef PFS_PROFILE
#define PFS_PROFILE 0
#endif

namespace pfs {

// ---------------------------------------------------------------- Philox
__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                              uint32_t& c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
}


// Coin rows come in windows of 128: coin row e of word w of
// global tile g is word (e >> 5) & 3 of Philox(((e >> 7) << 5) | (e & 31), w, g,
// DOMAIN_COIN), so one block serves rows e0, e0+32, e0+64, e0+96 of one word
// (e0 = "coin group" k: ((k >> 5) << 7) | (k & 31)).  coin_group fills o[r] with
// the word of row e0 + 32 r (injected mode: loaded, rows outside [lo, hi) skipped).
__device__ __forceinline__ uint32_t coin_row0(uint32_t k) { return ((k >> 5) << 7) | (k & 31u); }

template <int W>
__device__ __forceinline__ void coin_group(const KParams& kp, uint32_t k, uint32_t w, uint32_t g,
                                           int64_t tile, uint32_t lo, uint32_t hi, uint32_t o[4]) {
    if (kp.coins != nullptr) {
        const uint32_t e0 = coin_row0(k);
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const uint32_t e = e0 + 32u * r;
            o[r] = (e >= lo && e < hi) ? __ldg(kp.coins + (int64_t)e * kp.inject_words + tile * W + w) : 0u;
        }
        return;
    }
#if PFS_PROFILE
    if (kp.debug_skip & 4) { o[0] = o[1] = o[2] = o[3] = 0u; return; }
#endif
    uint32_t c0 = k, c1 = w, c2 = g, c3 = DOMAIN_COIN;
    philox4x32_10(c0, c1, c2, c3, (uint32_t)kp.seed, (uint32_t)(kp.seed >> 32));
    o[0] = c0; o[1] = c1; o[2] = c2; o[3] = c3;
}

// coin groups covering coin rows [lo, hi): k in [k0, k1), k0 a multiple of 32
__device__ __forceinline__ uint32_t coin_k0(uint32_t lo) { return (lo >> 7) << 5; }
__device__ __forceinline__ uint32_t coin_k1(uint32_t hi) { return ((hi + 127u) >> 7) << 5; }
__device__ __forceinline__ bool coin_group_live(uint32_t k, uint32_t lo, uint32_t hi) {
    const uint32_t e0 = coin_row0(k);
    return e0 + 96u >= lo && e0 < hi;
}


__device__ __forceinline__ void pattern_of(uint32_t ch, uint32_t pick, uint32_t& xm, uint32_t& zm) {
    switch (ch) {
        case CH_XERR: xm = 1; zm = 0; return;
        case CH_YERR: xm = 1; zm = 1; return;
        case CH_ZERR: xm = 0; zm = 1; return;
        case CH_DEP1: xm = (pick <= 1u) ? 1u : 0u; zm = (pick >= 1u) ? 1u : 0u; return;
        default: {
            const uint32_t code = pick + 1u;  // DEPOLARIZE2 codes 1..15 (gates.py:354-360)
            xm = (code & 1u) | (((code >> 2) & 1u) << 1);
            zm = ((code >> 1) & 1u) | (((code >> 3) & 1u) << 1);
        }
    }
}

// Noise draws.  A chunk is L = 2^lg consecutive trials of the
// op (trials past the op's end are virtual and dropped).  Philox block j of
// chunk r has counter (j, r, g, DOMAIN_NOISE | ordinal):
//   block 0        : w0,w1 -> 64-bit uniform for the Binomial(L, p) count,
//                    w2,w3 -> word pair 0;
//   block b >= 1   : word pairs 2b-1 (w0,w1) and 2b (w2,w3).
// Hit h of attempt a uses pair a*NZ_MAX_LIST + h: position = top lg bits of the
// first word (exactly uniform), Pauli pick = mulhi(second word, npat).  All
// positions are redrawn (next attempt) while any two coincide.  Counts above
// NZ_MAX_LIST (~1e-6 per chunk) use selection sampling with block 2^31 + i per
// trial, as does p == 1.  In the common case a chunk costs one Philox block.
__device__ __forceinline__ void noise_block(uint32_t j, uint32_t r, uint32_t g, uint32_t ordinal,
                                            uint64_t seed, uint32_t& w0, uint32_t& w1, uint32_t& w2,
                                            uint32_t& w3) {
    w0 = j; w1 = r; w2 = g; w3 = DOMAIN_NOISE | ordinal;
    philox4x32_10(w0, w1, w2, w3, (uint32_t)seed, (uint32_t)(seed >> 32));
}

template <typename Emit>
__device__ __forceinline__ void noise_chunk(const KParams& kp, const NoiseParam& np, uint32_t ordinal,
                                            uint32_t r, uint32_t g, uint32_t* sl, int ss, Emit emit) {
    const uint32_t L = np.L;
    const uint32_t lg = 31u - __clz(L);
    const uint32_t base = r * L;
    const uint32_t valid = (r + 1 == np.nchunks) ? np.last_len : L;  // real trials in this chunk
    uint32_t w0, w1, w2, w3;
    if (np.flags & NZ_ALL) {
        for (uint32_t i = 0; i < valid; i++) {
            noise_block(0x80000000u + i, r, g, ordinal, kp.seed, w0, w1, w2, w3);
            emit(base + i, np.npat > 1 ? __umulhi(w2, np.npat) : 0u);
        }
        return;
    }
    const unsigned long long* tab = reinterpret_cast<const unsigned long long*>(kp.noise_tab) + np.tab_full;
    noise_block(0u, r, g, ordinal, kp.seed, w0, w1, w2, w3);
    const uint64_t u = ((uint64_t)w1 << 32) | w0;
    uint32_t count = 0;
    while (count < np.len_full && u >= __ldg(tab + count)) count++;
    if (count == 0) return;
    const uint32_t sh = 32u - lg;
    if (count == 1) {  // the common case: block 0 already holds the hit
        const uint32_t pos = lg ? (w2 >> sh) : 0u;
        if (pos < valid) emit(base + pos, np.npat > 1 ? __umulhi(w3, np.npat) : 0u);
        return;
    }
    if (count <= NZ_MAX_LIST) {
        for (uint32_t attempt = 0;; attempt++) {
            bool dup = false;
            uint32_t blk = 0xFFFFFFFFu;
            for (uint32_t h = 0; h < count; h++) {
                const uint32_t k = attempt * NZ_MAX_LIST + h;
                uint32_t a, b;
                if (k == 0) { a = w2; b = w3; }
                else {
                    const uint32_t need = (k + 1) >> 1;
                    if (need != blk) { noise_block(need, r, g, ordinal, kp.seed, w0, w1, w2, w3); blk = need; }
                    if (k & 1u) { a = w0; b = w1; } else { a = w2; b = w3; }
                }
                const uint32_t pos = lg ? (a >> sh) : 0u;
                for (uint32_t q = 0; q < h; q++) dup |= (sl[q * ss] >> 4) == pos;
                sl[h * ss] = (pos << 4) | (np.npat > 1 ? __umulhi(b, np.npat) : 0u);
            }
            if (!dup) break;
            // block 0's pair must be recomputed for nothing: attempts > 0 never use pair 0
        }
        for (uint32_t h = 0; h < count; h++) {
            const uint32_t e = sl[h * ss];
            if ((e >> 4) < valid) emit(base + (e >> 4), e & 15u);
        }
    } else {
        uint32_t needed = count;
        for (uint32_t i = 0; needed > 0; i++) {
            noise_block(0x80000000u + i, r, g, ordinal, kp.seed, w0, w1, w2, w3);
            if (__umul64hi(((uint64_t)w1 << 32) | w0, (uint64_t)(L - i)) < needed) {
                if (i < valid) emit(base + i, np.npat > 1 ? __umulhi(w2, np.npat) : 0u);
                needed--;
            }
        }
    }
}


// ---------------------------------------------------------------- TMA staging
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(mbar)), "r"(count) : "memory");
}
// one elected thread: expect `bytes` and start a bulk global->shared copy that
// completes the transaction on `mbar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_addr(mbar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(mbar)) : "memory");
}
// wait with a suspend-time hint: the waiting warp sleeps instead of spinning
// on the issue slots its neighbours need
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* mbar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_addr(mbar)), "r"(parity), "r"(1000000u) : "memory");
    }
}

// wait polling with a nanosleep backoff (a lone producer thread whose latency
// does not matter: the slot ring is normally full)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* mbar, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_addr(mbar)), "r"(parity) : "memory");
        if (done) return;
        __nanosleep(256);
    }
}


__device__ __forceinline__ uint32_t transpose32_lane(uint32_t v, int lane) {
    // lane l holds row l (bit b = column b); afterwards lane l holds column l.
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint32_t mlo = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                           : j == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, v, j);
        if (lane & j) v = (v & ~mlo) | ((other >> j) & mlo);
        else v = (v & mlo) | ((other & mlo) << j);
    }
    return v;
}

// Dead coin rows (compiler pass 2b): rows of coin group k that some gate can
// read.  init_live_rows: the initial z rows 0..n-1; collapse_rows also loads
// the (qubit, slot) operands of an M / MR / R op's rows, flags stripped.
__device__ __forceinline__ uint32_t init_live_rows(const KParams& kp, uint32_t k, uint32_t n) {
    uint32_t live = 0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const uint32_t e = coin_row0(k) + 32u * r;
        if (e < n && !((__ldg(kp.init_dead + (e >> 5)) >> (e & 31u)) & 1u)) live |= 1u << r;
    }
    return live;
}

__device__ __forceinline__ uint32_t collapse_rows(const uint32_t* tg, uint32_t kind, uint32_t k, uint32_t lo,
                                                  uint32_t hi, uint2 qsv[4]) {
    uint32_t live = 0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const uint32_t e = coin_row0(k) + 32u * r;
        qsv[r] = make_uint2(0u, NO_SLOT);
        if (e < lo || e >= hi) continue;
        const uint32_t rel = e - lo;
        if (kind == K_R) qsv[r].x = tg[rel];
        else if (kind == K_M || (rel & 1u))
            qsv[r] = reinterpret_cast<const uint2*>(tg)[kind == K_MR ? rel >> 1 : rel];
        else continue;  // an MR's measure coin row: never applied
        if (!(qsv[r].x & COIN_DEAD)) live |= 1u << r;
        qsv[r].x &= ~COIN_DEAD;
    }
    return live;
}

// One noise op's draws for word g (DESIGN.md §4 with T = 32), warp-cooperative:
// lane l draws chunk r0 + l's Binomial count from Philox block 0; the warp's
// hits are compacted across lanes (prefix sum) and each lane produces one hit
// position per round.  A chunk whose positions collide, or whose count exceeds
// NZ_MAX_LIST, is redrawn serially by noise_chunk — so the hits are exactly
// noise_chunk's for every chunk.  wscr: 32 NZ_MAX_LIST words of per-warp shared scratch.
template <typename Apply>
__device__ __forceinline__ void noise_op_warp(const KParams& kp, const NoiseParam& np, uint32_t ordinal,
                                              uint32_t g, uint32_t* wscr, uint32_t* sl, int lane,
                                              Apply apply) {
    if (np.flags & NZ_ALL) {
        for (uint32_t r = (uint32_t)lane; r < np.nchunks; r += 32)
            noise_chunk(kp, np, ordinal, r, g, sl, 1, apply);
        return;
    }
    const uint32_t L = np.L;
    const uint32_t lg = 31u - __clz(L);
    const uint32_t sh = 32u - lg;
    const unsigned long long* tab = reinterpret_cast<const unsigned long long*>(kp.noise_tab) + np.tab_full;
    const uint32_t len = np.len_full;
    const unsigned long long t0 = len > 0 ? __ldg(tab) : 0ull;
    const unsigned long long t1 = len > 1 ? __ldg(tab + 1) : 0ull;
    for (uint32_t r0 = 0; r0 < np.nchunks; r0 += 32) {
        const uint32_t r = r0 + (uint32_t)lane;
        const bool valid = r < np.nchunks;
        uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0, count = 0;
        if (valid) {
            noise_block(0u, r, g, ordinal, kp.seed, w0, w1, w2, w3);
            const unsigned long long uu = ((unsigned long long)w1 << 32) | w0;
            if (len > 0 && uu >= t0) {
                count = 1;
                if (len > 1 && uu >= t1) {
                    count = 2;
                    while (count < len && uu >= __ldg(tab + count)) count++;
                }
            }
        }
        const bool big = count > (uint32_t)NZ_MAX_LIST;
        const uint32_t c = big ? 0u : count;
        uint32_t pre = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pre, d);
            if (lane >= d) pre += v;
        }
        const uint32_t H = __shfl_sync(0xFFFFFFFFu, pre, 31);
        if (H == 0 && !__any_sync(0xFFFFFFFFu, big)) continue;
        const uint32_t excl = pre - c;
        for (uint32_t j0 = 0; j0 < H; j0 += 32) {
            const uint32_t j = j0 + (uint32_t)lane;
            uint32_t lo = 0;  // owner chunk: smallest lane q with pre[q] > j
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t pv = __shfl_sync(0xFFFFFFFFu, pre, (int)(lo + st - 1));
                if (pv <= j) lo += st;
            }
            const uint32_t owner = lo > 31u ? 31u : lo;
            const uint32_t oexcl = __shfl_sync(0xFFFFFFFFu, excl, (int)owner);
            uint32_t x = __shfl_sync(0xFFFFFFFFu, w2, (int)owner);
            uint32_t y = __shfl_sync(0xFFFFFFFFu, w3, (int)owner);
            if (j < H) {
                const uint32_t h = j - oexcl;
                if (h > 0) {
                    uint32_t b0, b1, b2, b3;
                    noise_block((h + 1) >> 1, r0 + owner, g, ordinal, kp.seed, b0, b1, b2, b3);
                    x = (h & 1u) ? b0 : b2;
                    y = (h & 1u) ? b1 : b3;
                }
                const uint32_t pos = lg ? (x >> sh) : 0u;
                wscr[j] = (pos << 4) | (np.npat > 1 ? __umulhi(y, np.npat) : 0u);
            }
        }
        __syncwarp();
        bool dup = false;
        for (uint32_t h = 1; h < c; h++)
            for (uint32_t q = 0; q < h; q++) dup |= (wscr[excl + h] >> 4) == (wscr[excl + q] >> 4);
        if (dup || big) {
            noise_chunk(kp, np, ordinal, r, g, sl, 1, apply);  // rare: serial redraw
        } else {
            const uint32_t vlen = (r + 1 == np.nchunks) ? np.last_len : L;
            for (uint32_t h = 0; h < c; h++) {
                const uint32_t e = wscr[excl + h];
                if ((e >> 4) < vlen) apply(r * L + (e >> 4), e & 15u);
            }
        }
        __syncwarp();
    }
}

}  // namespace pfs
