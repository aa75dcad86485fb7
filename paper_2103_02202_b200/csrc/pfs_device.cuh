// Device helpers shared by the frame kernel (pfs_kernels.cu) and the
// error-model kernel (pfs_demkernel.cu): the Philox4x32-10 generator, the
// coin-row and noise-chunk schedules of DESIGN.md §4, Pauli patterns and the
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
// The 10 rounds inline (the hottest draw site uses this directly) ...
__device__ __forceinline__ void philox_rounds(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                              uint32_t k1) {
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
// ... and out of line: one copy serves the other call sites (code size)
static __device__ __noinline__ uint4 philox4x32_10_block(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                  uint32_t k1) {
    philox_rounds(c0, c1, c2, c3, k0, k1);
    return make_uint4(c0, c1, c2, c3);
}
__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                              uint32_t& c3, uint32_t k0, uint32_t k1) {
    const uint4 o = philox4x32_10_block(c0, c1, c2, c3, k0, k1);
    c0 = o.x; c1 = o.y; c2 = o.z; c3 = o.w;
}

// The RNG key of one global tile: the counters carry the low 32
// bits of the global tile index g; the high bits are folded into the key
// (k1 ^= g_hi * 0x9E3779B9, a bijection of g_hi), so every tile of a 64-bit
// shot range has its own stream and g < 2^32 keeps the plain (seed) key.
struct TileKey {
    uint32_t k0, k1, g;
};
__device__ __forceinline__ TileKey tile_key(uint64_t seed, uint64_t g64) {
    TileKey t;
    t.k0 = (uint32_t)seed;
    t.k1 = (uint32_t)(seed >> 32) ^ ((uint32_t)(g64 >> 32) * 0x9E3779B9u);
    t.g = (uint32_t)g64;
    return t;
}

// Collapse coins (FrameBatch.__init__, M, R, MR z rows; stabsim/frame_sim.py:
// 36-39, 74-90): word w of coin row e in tile g is word (w & 3) of
// Philox(e, w >> 2, g, DOMAIN_COIN) — one block serves four consecutive words
// (128 shots) of one row.
__device__ __forceinline__ void coin_block(const TileKey& tk, uint32_t e, uint32_t wq, uint32_t o[4]) {
    uint32_t c0 = e, c1 = wq, c2 = tk.g, c3 = DOMAIN_COIN;
    philox4x32_10(c0, c1, c2, c3, tk.k0, tk.k1);
    o[0] = c0; o[1] = c1; o[2] = c2; o[3] = c3;
}

__device__ __forceinline__ void pattern_of(uint32_t ch, uint32_t pick, uint32_t& xm, uint32_t& zm) {
    switch (ch) {
        case CH_XERR: xm = 1; zm = 0; return;
        case CH_YERR: xm = 1; zm = 1; return;
        case CH_ZERR: xm = 0; zm = 1; return;
        case CH_DEP1: xm = (pick <= 1u) ? 1u : 0u; zm = (pick >= 1u) ? 1u : 0u; return;
        default: {
            const uint32_t code = pick + 1u;  // DEPOLARIZE2 codes 1..15 (stabsim/gates.py:98-104)
            xm = (code & 1u) | (((code >> 2) & 1u) << 1);
            zm = ((code >> 1) & 1u) | (((code >> 3) & 1u) << 1);
        }
    }
}

// Noise draws.  An instruction's trials are (application,
// shot) pairs of the tile.  A chunk is a rectangle of ca = L / cs consecutive
// applications by cs consecutive shots (L, cs powers of two, cs <= T);
// chunk r = k * nS + cc (nS = T / cs) covers applications [k ca, k ca + ca)
// and shots [cc cs, cc cs + cs); position p of the chunk is application
// k ca + (p >> lg cs), shot cc cs + (p & (cs - 1)).  Positions whose
// application is past the instruction's end are virtual and dropped.  With
// cs = min(L, T) this is the plain app-major trial order (trial = r L + p).
// Philox block j of chunk r has counter (j, r, g, DOMAIN_NOISE | ordinal):
//   block 0        : w0,w1 -> 64-bit uniform for the Binomial(L, p) count,
//                    w2,w3 -> word pair 0;
//   block b >= 1   : word pairs 2b-1 (w0,w1) and 2b (w2,w3).
// Hit h of attempt a uses pair a*NZ_MAX_LIST + h: position = top lg L bits of
// the first word (exactly uniform), Pauli pick = mulhi(second word, npat).
// All positions are redrawn (next attempt) while any two coincide.  Counts
// above NZ_MAX_LIST use selection sampling with block 2^31 + i per trial, as
// does p == 1.  In the common case a chunk costs one Philox block.
__device__ __forceinline__ void noise_block(const TileKey& tk, uint32_t j, uint32_t r, uint32_t ordinal,
                                            uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& w3) {
    w0 = j; w1 = r; w2 = tk.g; w3 = DOMAIN_NOISE | ordinal;
    philox4x32_10(w0, w1, w2, w3, tk.k0, tk.k1);
}

// Decoded noise descriptor (the (c, d, e) words of a device op)
struct NoiseOp {
    uint32_t ordinal;
    uint32_t lgL, lgcs, npat, ch, zone;
    uint32_t tab_off, tab_len;
};
__device__ __forceinline__ NoiseOp decode_noise(uint32_t c, uint32_t d, uint32_t e) {
    NoiseOp n;
    n.ordinal = c;
    n.lgL = d & 31u;
    n.lgcs = (d >> 5) & 31u;
    n.npat = (d >> 10) & 15u;
    n.ch = (d >> 14) & 7u;
    n.zone = (d >> 17) & 3u;
    n.tab_off = e & 0xFFFFFFu;
    n.tab_len = e >> 24;
    return n;
}

__device__ __forceinline__ NoiseOp noise_op_of(const NoiseParam& np, uint32_t ordinal) {
    NoiseOp n;
    n.ordinal = ordinal;
    n.lgL = 31u - __clz(np.L);
    n.lgcs = 31u - __clz(np.cs);
    n.npat = np.npat;
    n.ch = np.ch;
    n.zone = np.zone;
    n.tab_off = np.tab;
    n.tab_len = np.len;
    return n;
}

// Binomial count of chunk r from block 0 (thresholds: tab[0..len))
__device__ __forceinline__ uint32_t chunk_count(const unsigned long long* tab, uint32_t len, uint32_t w0,
                                                uint32_t w1) {
    const unsigned long long u = ((unsigned long long)w1 << 32) | w0;
    uint32_t count = 0;
    while (count < len && u >= tab[count]) count++;
    return count;
}

// Every hit of chunk r with position < vlen: emit(position, pick).  General
// path (any count, duplicates, p == 1); `tab` = all threshold tables (the op's
// at nz.tab_off); `sl` = NZ_MAX_LIST words of scratch.
template <typename Emit>
__device__ __forceinline__ void noise_chunk(const TileKey& tk, const NoiseOp& nz, const unsigned long long* tab,
                                            uint32_t r, uint32_t vlen, uint32_t* sl, Emit emit) {
    const uint32_t L = 1u << nz.lgL;
    const uint32_t lg = nz.lgL;
    uint32_t w0, w1, w2, w3;
    if (nz.zone == NZONE_ALL) {
        for (uint32_t i = 0; i < vlen; i++) {
            noise_block(tk, 0x80000000u + i, r, nz.ordinal, w0, w1, w2, w3);
            emit(i, nz.npat > 1 ? __umulhi(w2, nz.npat) : 0u);
        }
        return;
    }
    if (nz.zone == NZONE_NONE) return;
    noise_block(tk, 0u, r, nz.ordinal, w0, w1, w2, w3);
    const uint32_t count = chunk_count(tab + nz.tab_off, nz.tab_len, w0, w1);
    if (count == 0) return;
    const uint32_t sh = 32u - lg;
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
                    if (need != blk) { noise_block(tk, need, r, nz.ordinal, w0, w1, w2, w3); blk = need; }
                    if (k & 1u) { a = w0; b = w1; } else { a = w2; b = w3; }
                }
                const uint32_t pos = lg ? (a >> sh) : 0u;
                for (uint32_t q = 0; q < h; q++) dup |= (sl[q] >> 4) == pos;
                sl[h] = (pos << 4) | (nz.npat > 1 ? __umulhi(b, nz.npat) : 0u);
            }
            if (!dup) break;
        }
        for (uint32_t h = 0; h < count; h++) {
            const uint32_t e = sl[h];
            if ((e >> 4) < vlen) emit(e >> 4, e & 15u);
        }
    } else {
        uint32_t needed = count;
        for (uint32_t i = 0; needed > 0; i++) {
            noise_block(tk, 0x80000000u + i, r, nz.ordinal, w0, w1, w2, w3);
            if (__umul64hi(((uint64_t)w1 << 32) | w0, (uint64_t)(L - i)) < needed) {
                if (i < vlen) emit(i, nz.npat > 1 ? __umulhi(w2, nz.npat) : 0u);
                needed--;
            }
        }
    }
}

// Fast path of one chunk: the hits when there are at most two (no collision),
// as (pos << 4 | pick) words; returns the count, or ~0u when the chunk needs
// the general path (more hits, colliding positions, p == 1).
__device__ __forceinline__ uint32_t chunk_fast(const TileKey& tk, const NoiseOp& nz, const unsigned long long* tab,
                                               uint32_t r, uint32_t& h0, uint32_t& h1) {
    if (nz.zone != NZONE_TAB) return nz.zone == NZONE_NONE ? 0u : ~0u;
    uint32_t w0, w1, w2, w3;
    noise_block(tk, 0u, r, nz.ordinal, w0, w1, w2, w3);
    const uint32_t count = chunk_count(tab + nz.tab_off, nz.tab_len, w0, w1);
    if (count == 0) return 0u;
    const uint32_t sh = 32u - nz.lgL;
    h0 = ((nz.lgL ? (w2 >> sh) : 0u) << 4) | (nz.npat > 1 ? __umulhi(w3, nz.npat) : 0u);
    if (count == 1) return 1u;
    if (count > 2) return ~0u;
    noise_block(tk, 1u, r, nz.ordinal, w0, w1, w2, w3);  // pair 1 = block 1 (w0, w1)
    h1 = ((nz.lgL ? (w0 >> sh) : 0u) << 4) | (nz.npat > 1 ? __umulhi(w1, nz.npat) : 0u);
    return (h0 >> 4) == (h1 >> 4) ? ~0u : 2u;
}

__device__ __forceinline__ uint32_t transpose32_lane(uint32_t v, int lane) {
    // lane l holds row l (bit b = column b); afterwards lane l holds column l.
    // Stage j swaps, between lanes l and l ^ j, the off-diagonal j-bit blocks.
    // j = 16, 8 move whole bytes: one PRMT with a per-lane selector.
    uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v, 16);
    v = __byte_perm(v, o, (lane & 16) ? 0x3276u : 0x5410u);
    o = __shfl_xor_sync(0xFFFFFFFFu, v, 8);
    v = __byte_perm(v, o, (lane & 8) ? 0x3715u : 0x6240u);
    // j = 4, 2, 1: rotate the partner's word into place (the bits that wrap
    // around fall outside the inserted mask), then one bit-select
#pragma unroll
    for (int j = 4; j > 0; j >>= 1) {
        const uint32_t mlo = j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
        const bool hi = (lane & j) != 0;
        const uint32_t keep = hi ? ~mlo : mlo;
        o = __shfl_xor_sync(0xFFFFFFFFu, v, j);
        o = __funnelshift_l(o, o, hi ? 32 - j : j);
        v = (v & keep) | (o & ~keep);
    }
    return v;
}

}  // namespace pfs
