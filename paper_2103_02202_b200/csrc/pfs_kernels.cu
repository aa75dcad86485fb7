// sm_100a kernels of the bulk Pauli-frame sampler.
//
// frame_kernel  — persistent program interpreter.  Each thread group of a CTA
//                 owns a tile of T = 32 W shots and keeps the whole frame table
//                 of that tile (x and z bit-planes, qubit-major, shots packed
//                 in uint32 words: SURVEY.md Appendix D) resident in shared
//                 memory for the entire circuit.  Reference semantics per op:
//                   gate rules      stabsim/frame_sim.py:64-72 (gates.py:70-92)
//                   M / R / MR      stabsim/frame_sim.py:74-90
//                   noise           stabsim/frame_sim.py:92-167, entropy.py:65-113
//                   detectors       stabsim/io_formats.py:208-227
//                 Noise is sampled inline (counter-based Philox):
//                 a noise instruction fused into its gate / collapse op is
//                 applied by the item that owns the rows, in registers.
// rows_to_b8 / tiles_to_b8 — 32x32 warp-shuffle bit transposes to shot-major
//                 b8 (stabsim/bitvec.py:193-209, io_formats.py:94-96).
#include <cuda_runtime.h>

#include <cstdint>

#include "pfs_internal.h"
#include "pfs_device.cuh"

// PFS_PROFILE=1 builds the profiling library (op clock traces, ablations);
// the production kernels carry none of it.
#ifndef PFS_PROFILE
#define PFS_PROFILE 0
#endif

namespace pfs {

// ---------------------------------------------------------------- vectors
template <int V> struct VW { uint32_t w[V]; };

template <int V> __device__ __forceinline__ VW<V> vld(const uint32_t* p);
template <> __device__ __forceinline__ VW<4> vld<4>(const uint32_t* p) {
    uint4 v = *reinterpret_cast<const uint4*>(p); return VW<4>{{v.x, v.y, v.z, v.w}};
}
template <> __device__ __forceinline__ VW<2> vld<2>(const uint32_t* p) {
    uint2 v = *reinterpret_cast<const uint2*>(p); return VW<2>{{v.x, v.y}};
}
template <> __device__ __forceinline__ VW<1> vld<1>(const uint32_t* p) { return VW<1>{{*p}}; }

template <int V> __device__ __forceinline__ void vst(uint32_t* p, const VW<V>& v);
template <> __device__ __forceinline__ void vst<4>(uint32_t* p, const VW<4>& v) {
    *reinterpret_cast<uint4*>(p) = make_uint4(v.w[0], v.w[1], v.w[2], v.w[3]);
}
template <> __device__ __forceinline__ void vst<2>(uint32_t* p, const VW<2>& v) {
    *reinterpret_cast<uint2*>(p) = make_uint2(v.w[0], v.w[1]);
}
template <> __device__ __forceinline__ void vst<1>(uint32_t* p, const VW<1>& v) { *p = v.w[0]; }

// streaming (evict-first) global stores
template <int V> __device__ __forceinline__ void vstcs(uint32_t* p, const VW<V>& v);
template <> __device__ __forceinline__ void vstcs<4>(uint32_t* p, const VW<4>& v) {
    __stcs(reinterpret_cast<uint4*>(p), make_uint4(v.w[0], v.w[1], v.w[2], v.w[3]));
}
template <> __device__ __forceinline__ void vstcs<2>(uint32_t* p, const VW<2>& v) {
    __stcs(reinterpret_cast<uint2*>(p), make_uint2(v.w[0], v.w[1]));
}
template <> __device__ __forceinline__ void vstcs<1>(uint32_t* p, const VW<1>& v) { __stcs(p, v.w[0]); }

template <int V> __device__ __forceinline__ VW<V> vxor(const VW<V>& a, const VW<V>& b) {
    VW<V> r;
#pragma unroll
    for (int j = 0; j < V; j++) r.w[j] = a.w[j] ^ b.w[j];
    return r;
}
template <int V> __device__ __forceinline__ VW<V> vzero() {
    VW<V> r;
#pragma unroll
    for (int j = 0; j < V; j++) r.w[j] = 0u;
    return r;
}
// v.w[word] ^= bit (word is a runtime index: unrolled selects, no local memory)
template <int V> __device__ __forceinline__ void vflip(VW<V>& v, uint32_t word, uint32_t bit) {
#pragma unroll
    for (int j = 0; j < V; j++) v.w[j] ^= (word == (uint32_t)j) ? bit : 0u;
}

// global-memory loads through the read-only path for immutable inputs
template <int V> __device__ __forceinline__ VW<V> vldg(const uint32_t* p);
template <> __device__ __forceinline__ VW<4> vldg<4>(const uint32_t* p) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p)); return VW<4>{{v.x, v.y, v.z, v.w}};
}
template <> __device__ __forceinline__ VW<2> vldg<2>(const uint32_t* p) {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p)); return VW<2>{{v.x, v.y}};
}
template <> __device__ __forceinline__ VW<1> vldg<1>(const uint32_t* p) { return VW<1>{{__ldg(p)}}; }

template <int C> struct Log2;
template <> struct Log2<1> { static constexpr int v = 0; };
template <> struct Log2<2> { static constexpr int v = 1; };
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };

// Words c V .. c V + V - 1 of coin row e (injected mode: the
// caller's rows)
template <int W, int V>
__device__ __forceinline__ VW<V> coin_vec(const KParams& kp, const TileKey& tk, uint32_t e, int c, int64_t tile) {
    VW<V> o;
    if (kp.coins != nullptr) {
        const uint32_t* src = kp.coins + (int64_t)e * kp.inject_words + tile * W + c * V;
#pragma unroll
        for (int j = 0; j < V; j++) o.w[j] = __ldg(src + j);
        return o;
    }
#if PFS_PROFILE
    if (kp.debug_skip & 4) return vzero<V>();
#endif
    // word w of coin row e = word (w & 3) of Philox(e, w >> 2, g, DOMAIN_COIN),
    // inline: a call inside the op loop would spill the loop's live values
    uint32_t b[4] = {e, (uint32_t)(c * V) >> 2, tk.g, DOMAIN_COIN};
    philox_rounds(b[0], b[1], b[2], b[3], tk.k0, tk.k1);
#pragma unroll
    for (int j = 0; j < V; j++) o.w[j] = b[(c * V + j) & 3];
    return o;
}

// Items of one op, U per thread per batch: all U operand loads (L1-resident
// target indices) are issued before any of the dependent shared-memory work.
template <int U, typename Load, typename Work>
__device__ __forceinline__ void batched_items(int tid, int nth, int items, Load load, Work work) {
    for (int i0 = tid; i0 < items; i0 += U * nth) {
        decltype(load(0)) v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + u * nth;
            v[u] = i < items ? load(i) : decltype(load(0)){};
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + u * nth;
            if (i < items) work(i, v[u]);
        }
    }
}

// One frame rule on rows held in registers (stabsim/gates.py:70-92; all XORs
// read old values)
template <int V>
__device__ __forceinline__ void apply_rule(uint32_t code, VW<V>& x0, VW<V>& z0, VW<V>& x1, VW<V>& z1) {
    switch (code) {
        case R_SWAPXZ: { const VW<V> t = x0; x0 = z0; z0 = t; break; }
        case R_ZXORX: z0 = vxor<V>(z0, x0); break;
        case R_XXORZ: x0 = vxor<V>(x0, z0); break;
        case R_CX: x1 = vxor<V>(x1, x0); z0 = vxor<V>(z0, z1); break;
        case R_CZ: { const VW<V> a = vxor<V>(z0, x1); z1 = vxor<V>(z1, x0); z0 = a; break; }
        case R_CY: {
            const VW<V> nz0 = vxor<V>(z0, vxor<V>(x1, z1));
            z1 = vxor<V>(z1, x0);
            x1 = vxor<V>(x1, x0);
            z0 = nz0;
            break;
        }
        case R_SWAP: { VW<V> t = x0; x0 = x1; x1 = t; t = z0; z0 = z1; z1 = t; break; }
        default: break;
    }
}

// Frame rows of application `app`: ar targets per app (gates, noise), or
// (row | COIN_DEAD, slot) pairs (collapses)
struct AppRows {
    uint32_t r0, r1;
};
__device__ __forceinline__ AppRows app_rows(const uint32_t* tg, uint32_t app, int ar, bool pairs) {
    if (pairs) return AppRows{tg[2 * app] & ~COIN_DEAD, 0u};
    if (ar == 2) {
        const uint2 q = reinterpret_cast<const uint2*>(tg)[app];
        return AppRows{q.x, q.y};
    }
    return AppRows{tg[app], 0u};
}

// XOR one sampled Pauli (channel ch, pattern pick) into shot s of the rows of
// one application: owner-thread read-modify-write (fused ops) or atomics
// (standalone noise, whose chunks may share a word)
template <int W, bool ATOMIC>
__device__ __forceinline__ void xor_pauli(uint32_t* X, uint32_t* Z, const AppRows& rr, int ar, uint32_t ch,
                                          uint32_t pick, uint32_t s) {
    uint32_t xm, zm;
    pattern_of(ch, pick, xm, zm);
    const uint32_t bit = 1u << (s & 31u), w = s >> 5;
    auto flip = [&](uint32_t* p) { if (ATOMIC) atomicXor(p, bit); else *p ^= bit; };
    if (xm & 1u) flip(X + (size_t)rr.r0 * W + w);
    if (zm & 1u) flip(Z + (size_t)rr.r0 * W + w);
    if (ar == 2) {
        if (xm & 2u) flip(X + (size_t)rr.r1 * W + w);
        if (zm & 2u) flip(Z + (size_t)rr.r1 * W + w);
    }
}

// General noise path of one chunk (any count, colliding positions, p == 1):
// out of line, one copy per kernel.  Chunk r covers applications [a0, a0 +
// na) and shots [s0, s0 + cs).
template <int W, bool ATOMIC>
__device__ __noinline__ void chunk_hits_slow(const TileKey tk, const NoiseOp nz, const unsigned long long* tab,
                                             uint32_t r, uint32_t a0, uint32_t na, uint32_t s0, const uint32_t* tg,
                                             int ar, bool pairs, uint32_t* X, uint32_t* Z, uint32_t* sl) {
    const uint32_t msk = (1u << nz.lgcs) - 1;
    noise_chunk(tk, nz, tab, r, na << nz.lgcs, sl, [&](uint32_t pos, uint32_t pick) {
        xor_pauli<W, ATOMIC>(X, Z, app_rows(tg, a0 + (pos >> nz.lgcs), ar, pairs), ar, nz.ch, pick, s0 + (pos & msk));
    });
}

// The noise of one chunk into the frame, one thread: one Philox block in the
// common case (at most two hits, distinct), else the general path
template <int W, bool ATOMIC>
__device__ __forceinline__ void chunk_hits(const TileKey& tk, const NoiseOp& nz, const unsigned long long* tab,
                                           uint32_t r, uint32_t a0, uint32_t na, uint32_t s0, const uint32_t* tg,
                                           int ar, bool pairs, uint32_t* X, uint32_t* Z, uint32_t* sl) {
    uint32_t h0 = 0, h1 = 0;
    const uint32_t nh = chunk_fast(tk, nz, tab, r, h0, h1);
    if (nh == ~0u) {
        chunk_hits_slow<W, ATOMIC>(tk, nz, tab, r, a0, na, s0, tg, ar, pairs, X, Z, sl);
        return;
    }
    const uint32_t vl = na << nz.lgcs, msk = (1u << nz.lgcs) - 1;
    if (nh > 0 && (h0 >> 4) < vl)
        xor_pauli<W, ATOMIC>(X, Z, app_rows(tg, a0 + ((h0 >> 4) >> nz.lgcs), ar, pairs), ar, nz.ch, h0 & 15u,
                             s0 + ((h0 >> 4) & msk));
    if (nh > 1 && (h1 >> 4) < vl)
        xor_pauli<W, ATOMIC>(X, Z, app_rows(tg, a0 + ((h1 >> 4) >> nz.lgcs), ar, pairs), ar, nz.ch, h1 & 15u,
                             s0 + ((h1 >> 4) & msk));
}

// Warp-cooperative noise: lane l draws one chunk r (valid lanes) — block 0
// gives the Binomial count and the first position pair — the warp compacts the
// hits (prefix sum), each lane resolves one hit per round (extra Philox blocks
// for hits h >= 1) into the warp scratch, then each lane XORs one
// hit into the frame (shared-memory atomics: hits of a chunk may share a word).
// Chunks whose positions collide, counts above NZ_MAX_LIST, p == 1, or a warp
// total above WSCR take the general path, lane by lane.  The chunk covers
// applications [a0, a0 + na) and shots [s0, s0 + cs).  Every lane of the warp
// must call this (shuffles).
// Hit entry of a pre-sampled noise list (noise_kernel -> frame kernel), ready
// to apply: low word = plane word offset of target 0 (row W + word, 20 bits) |
// bit index << 20 | x0 z0 x1 z1 flip flags << 25; high word = plane word offset
// of target 1 (bits 24-31 of the high word are free: noise_kernel's staging
// keeps the consumer warp there)
template <int W>
__device__ __forceinline__ unsigned long long make_hit(const AppRows& rr, uint32_t ch, uint32_t pick, uint32_t s) {
    uint32_t xm, zm;
    pattern_of(ch, pick, xm, zm);
    const uint32_t w = s >> 5;
    const uint32_t lo = (rr.r0 * W + w) | ((s & 31u) << 20) | ((xm & 1u) << 25) | ((zm & 1u) << 26) |
                        ((xm >> 1) << 27) | ((zm >> 1) << 28);
    const uint32_t hi = rr.r1 * W + w;
    return (unsigned long long)lo | ((unsigned long long)hi << 32);
}
// xa = shared address of the group's x plane, zb = bytes from the x to the z
// plane; fire-and-forget shared-memory XOR reductions (hits may share a word)
__device__ __forceinline__ void apply_hit_entry(uint32_t xa, uint32_t zb, unsigned long long e) {
    const uint32_t lo = (uint32_t)e, hi = (uint32_t)(e >> 32);
    const uint32_t bit = 1u << ((lo >> 20) & 31u);
    const uint32_t p0 = xa + ((lo & 0xFFFFFu) << 2), p1 = xa + ((hi & 0xFFFFFu) << 2);
    if (lo & (1u << 25)) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(p0), "r"(bit) : "memory");
    if (lo & (1u << 26)) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(p0 + zb), "r"(bit) : "memory");
    if (lo & (1u << 27)) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(p1), "r"(bit) : "memory");
    if (lo & (1u << 28)) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(p1 + zb), "r"(bit) : "memory");
}

template <int W>
__device__ __forceinline__ void warp_chunks(const TileKey& tk, const NoiseOp& nz, const unsigned long long* tab,
                                            unsigned long long t0, unsigned long long t1, bool valid, uint32_t r,
                                            uint32_t a0, uint32_t na, uint32_t s0, const uint32_t* tg, int ar,
                                            bool pairs, uint32_t* X, uint32_t* Z, uint32_t* sl, uint32_t* wscr,
                                            int lane) {
    if (nz.zone == NZONE_NONE) return;
    const uint32_t sh = 32u - nz.lgL, msk = (1u << nz.lgcs) - 1;
    uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0, count = 0;
    if (valid && nz.zone == NZONE_TAB) {
        w0 = 0u; w1 = r; w2 = tk.g; w3 = DOMAIN_NOISE | nz.ordinal;  // block 0, inline
        philox_rounds(w0, w1, w2, w3, tk.k0, tk.k1);
        // count = min{m : u < t[m]}: the first two thresholds come from
        // registers (uniform per op), the rare tail from the table
        const unsigned long long u = ((unsigned long long)w1 << 32) | w0;
        count = (nz.tab_len > 0 && u >= t0) ? ((nz.tab_len > 1 && u >= t1) ? 2u : 1u) : 0u;
        if (count == 2u)
            while (count < nz.tab_len && u >= tab[nz.tab_off + count]) count++;
    }
    bool slow = valid && (nz.zone == NZONE_ALL || count > (uint32_t)NZ_MAX_LIST);
    uint32_t c = slow ? 0u : count;
    uint32_t pre = c;  // inclusive prefix of the warp's hit counts
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pre, d);
        if (lane >= d) pre += v;
    }
    uint32_t H = __shfl_sync(0xFFFFFFFFu, pre, 31);
    if (H > (uint32_t)WSCR) {  // rare: too many hits for the scratch
        slow |= c > 0;
        c = 0;
        pre = 0;
        H = 0;
    }
    const uint32_t excl = pre - c;
    auto owner_of = [&](uint32_t j) {  // smallest lane q with pre[q] > j
        uint32_t lo = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
            const uint32_t pv = __shfl_sync(0xFFFFFFFFu, pre, (int)(lo + st - 1));
            if (pv <= j) lo += st;
        }
        return (int)(lo > 31u ? 31u : lo);
    };
    if (H <= 32u) {
        // one hit per lane: its position, pick and frame rows are resolved in a
        // single round (the operand loads overlap the collision check)
        const uint32_t j = (uint32_t)lane;
        const int ow = owner_of(j);
        const uint32_t oexcl = __shfl_sync(0xFFFFFFFFu, excl, ow);
        const uint32_t orr = __shfl_sync(0xFFFFFFFFu, r, ow);
        const uint32_t oa0 = __shfl_sync(0xFFFFFFFFu, a0, ow);
        const uint32_t os0 = __shfl_sync(0xFFFFFFFFu, s0, ow);
        const uint32_t ovl = __shfl_sync(0xFFFFFFFFu, na, ow) << nz.lgcs;
        uint32_t x = __shfl_sync(0xFFFFFFFFu, w2, ow);
        uint32_t y = __shfl_sync(0xFFFFFFFFu, w3, ow);
        uint32_t pos = 0, pick = 0;
        AppRows rr{0u, 0u};
        const bool mine = j < H;
        if (mine) {
            const uint32_t h = j - oexcl;
            if (h > 0) {
                uint32_t b0, b1, b2, b3;
                noise_block(tk, (h + 1) >> 1, orr, nz.ordinal, b0, b1, b2, b3);
                x = (h & 1u) ? b0 : b2;
                y = (h & 1u) ? b1 : b3;
            }
            pos = nz.lgL ? (x >> sh) : 0u;
            pick = nz.npat > 1 ? __umulhi(y, nz.npat) : 0u;
            wscr[j] = pos;
            if (pos < ovl) rr = app_rows(tg, oa0 + (pos >> nz.lgcs), ar, pairs);
        }
        // positions of one chunk must be distinct: two hits compare by
        // shuffle, more through the scratch
        const uint32_t p0 = __shfl_sync(0xFFFFFFFFu, pos, (int)(excl & 31u));
        const uint32_t p1 = __shfl_sync(0xFFFFFFFFu, pos, (int)((excl + 1) & 31u));
        if (c == 2) slow |= p0 == p1;
        if (__any_sync(0xFFFFFFFFu, c > 2)) {
            __syncwarp();
            for (uint32_t h = 1; h < c; h++)
                for (uint32_t q = 0; q < h; q++) slow |= wscr[excl + h] == wscr[excl + q];
        }
        const uint32_t slowm = __ballot_sync(0xFFFFFFFFu, slow);
        if (mine && pos < ovl && !((slowm >> ow) & 1u))
            xor_pauli<W, true>(X, Z, rr, ar, nz.ch, pick, os0 + (pos & msk));
    } else {
        for (uint32_t j0 = 0; j0 < H; j0 += 32) {
            const uint32_t j = j0 + (uint32_t)lane;
            const int ow = owner_of(j);
            const uint32_t oexcl = __shfl_sync(0xFFFFFFFFu, excl, ow);
            const uint32_t orr = __shfl_sync(0xFFFFFFFFu, r, ow);
            uint32_t x = __shfl_sync(0xFFFFFFFFu, w2, ow);
            uint32_t y = __shfl_sync(0xFFFFFFFFu, w3, ow);
            if (j < H) {
                const uint32_t h = j - oexcl;
                if (h > 0) {
                    uint32_t b0, b1, b2, b3;
                    noise_block(tk, (h + 1) >> 1, orr, nz.ordinal, b0, b1, b2, b3);
                    x = (h & 1u) ? b0 : b2;
                    y = (h & 1u) ? b1 : b3;
                }
                wscr[j] = ((nz.lgL ? (x >> sh) : 0u) << 4) | (nz.npat > 1 ? __umulhi(y, nz.npat) : 0u);
            }
        }
        __syncwarp();
        for (uint32_t h = 1; h < c; h++)  // positions of one chunk must be distinct
            for (uint32_t q = 0; q < h; q++) slow |= (wscr[excl + h] >> 4) == (wscr[excl + q] >> 4);
        const uint32_t slowm = __ballot_sync(0xFFFFFFFFu, slow);
        for (uint32_t j0 = 0; j0 < H; j0 += 32) {
            const uint32_t j = j0 + (uint32_t)lane;
            const int ow = owner_of(j);
            const uint32_t oa0 = __shfl_sync(0xFFFFFFFFu, a0, ow);
            const uint32_t os0 = __shfl_sync(0xFFFFFFFFu, s0, ow);
            const uint32_t ovl = __shfl_sync(0xFFFFFFFFu, na, ow) << nz.lgcs;
            if (j < H && !((slowm >> ow) & 1u)) {
                const uint32_t e = wscr[j], pos = e >> 4;
                if (pos < ovl)
                    xor_pauli<W, true>(X, Z, app_rows(tg, oa0 + (pos >> nz.lgcs), ar, pairs), ar, nz.ch, e & 15u,
                                       os0 + (pos & msk));
            }
        }
    }
    if (slow) chunk_hits_slow<W, true>(tk, nz, tab, r, a0, na, s0, tg, ar, pairs, X, Z, sl);
    __syncwarp();  // the scratch is reused by the next call
}

// Fused noise of the applications [A0, A1) a warp owns in this op (A0 a
// multiple of ca): every chunk (k, vector c, sub-chunk u) of those
// applications, 32 per warp-cooperative pass.  Injected mode: each
// application's mask rows.  Every lane must call this.
template <int W>
__device__ __forceinline__ void warp_range_noise(const KParams& kp, const TileKey& tk, const NoiseOp& nz,
                                                 const unsigned long long* tab, uint32_t count, uint32_t A0,
                                                 uint32_t A1, const uint32_t* tg, int ar, bool pairs, uint32_t* X,
                                                 uint32_t* Z, uint32_t* sl, uint32_t* wscr, int lane, uint32_t rowb,
                                                 int64_t tile) {
    constexpr int V = W >= 4 ? 4 : W;
    constexpr int C = W / V;
    constexpr int LC = Log2<C>::v;
    constexpr uint32_t S = 32u * V;
    __syncwarp();  // the warp's row updates are visible to the lanes applying hits
    if (kp.masks != nullptr) {
        for (uint32_t j = (uint32_t)lane; j < ((A1 - A0) << LC); j += 32) {
            const uint32_t app = A0 + (j >> LC);
            const int c = (int)(j & (C - 1));
            const AppRows rr = app_rows(tg, app, ar, pairs);
            for (int sl2 = 0; sl2 < ar; sl2++) {
                const uint32_t* m = kp.masks + (int64_t)(rowb + 2u * (app * ar + sl2)) * kp.inject_words + tile * W + c * V;
                const size_t p = (size_t)(sl2 ? rr.r1 : rr.r0) * W + c * V;
                vst<V>(X + p, vxor<V>(vld<V>(X + p), vldg<V>(m)));
                vst<V>(Z + p, vxor<V>(vld<V>(Z + p), vldg<V>(m + kp.inject_words)));
            }
        }
        __syncwarp();
        return;
    }
#if PFS_PROFILE
    if (kp.debug_skip & 2) return;  // profiling ablation: no noise draws (wrong results)
#endif
    if (nz.zone == NZONE_NONE) return;
    const uint32_t lgca = nz.lgL - nz.lgcs;
    const uint32_t cs = 1u << nz.lgcs;
    const uint32_t nS = (32u * W) >> nz.lgcs;
    const uint32_t m = cs >= S ? 1u : S / cs;      // chunks per vector
    const uint32_t per_k = (uint32_t)C * m;         // chunks per application block
    const uint32_t k0 = A0 >> lgca;
    const uint32_t nch = ((A1 - A0 + (1u << lgca) - 1) >> lgca) * per_k;
    const unsigned long long t0 = nz.tab_len > 0 ? tab[nz.tab_off] : ~0ull;
    const unsigned long long t1 = nz.tab_len > 1 ? tab[nz.tab_off + 1] : ~0ull;
    for (uint32_t q0 = 0; q0 < nch; q0 += 32) {
        const uint32_t q = q0 + (uint32_t)lane;
        const bool valid = q < nch;
        const uint32_t k = k0 + q / per_k, rem = q % per_k;
        const uint32_t c = rem / m, u = rem - c * m;
        const uint32_t a0 = k << lgca;
        warp_chunks<W>(tk, nz, tab, t0, t1, valid, k * nS + c * m + u, a0, valid ? min(1u << lgca, count - a0) : 0u,
                       c * S + u * cs, tg, ar, pairs, X, Z, sl, wscr, lane);
    }
}

// A standalone noise instruction: one chunk per lane, warp-cooperative draws,
// hits XORed with shared-memory atomics (consecutive noise ops commute: no
// barrier between them)
template <int W>
__device__ __forceinline__ void noise_op(const KParams& kp, const TileKey& tk, uint32_t* X, uint32_t* Z,
                                         const uint32_t* tg, uint32_t code, uint32_t count, const NoiseOp& nz,
                                         uint32_t rowb, const unsigned long long* tab, uint32_t* sl, uint32_t* wscr,
                                         int tid, int nth, int64_t tile) {
    constexpr int V = W >= 4 ? 4 : W;
    constexpr int C = W / V;
    constexpr int LC = Log2<C>::v;
    const int ar = code == CH_DEP2 ? 2 : 1;
    const int lane = tid & 31;
    if (kp.masks != nullptr) {
        // injected masks: per target, x row then z row
        const int items = (int)((count * ar) << LC);
        for (int i = tid; i < items; i += nth) {
            const int j = i >> LC, c = i & (C - 1);
            const size_t p = (size_t)__ldg(tg + j) * W + c * V;
            const uint32_t* mrow = kp.masks + (int64_t)(rowb + 2 * j) * kp.inject_words + tile * W + c * V;
            const VW<V> mx = vldg<V>(mrow), mz = vldg<V>(mrow + kp.inject_words);
#pragma unroll
            for (int q = 0; q < V; q++) {  // atomics: targets may repeat (F_DUP)
                if (mx.w[q]) atomicXor(X + p + q, mx.w[q]);
                if (mz.w[q]) atomicXor(Z + p + q, mz.w[q]);
            }
        }
        return;
    }
    if (nz.zone == NZONE_NONE) return;
#if PFS_PROFILE
    if (kp.debug_skip & 2) return;
#endif
    const uint32_t lgca = nz.lgL - nz.lgcs;
    const uint32_t nS = (32u * W) >> nz.lgcs;
    const uint32_t nch = ((count + (1u << lgca) - 1) >> lgca) * nS;
    const unsigned long long t0 = nz.tab_len > 0 ? tab[nz.tab_off] : ~0ull;
    const unsigned long long t1 = nz.tab_len > 1 ? tab[nz.tab_off + 1] : ~0ull;
    for (uint32_t rb = (uint32_t)(tid - lane); rb < nch; rb += nth) {
        const uint32_t r = rb + (uint32_t)lane;
        const bool valid = r < nch;
        const uint32_t k = r / nS, cc = r - k * nS;
        const uint32_t a0 = k << lgca;
        warp_chunks<W>(tk, nz, tab, t0, t1, valid, r, a0, valid ? min(1u << lgca, count - a0) : 0u, cc << nz.lgcs,
                       tg, ar, false, X, Z, sl, wscr, lane);
    }
}

// ------------------------------------------------------------ stream executor
#ifndef PFS_GATE_BATCH
#define PFS_GATE_BATCH 2
#endif
constexpr int GATE_BATCH = PFS_GATE_BATCH;  // applications whose rows a lane loads before it stores any
constexpr int GATE_AHEAD = (int)GATE_AHEAD_PASSES;
#ifndef PFS_DET_BATCH
#define PFS_DET_BATCH 6
#endif
constexpr int DET_BATCH = PFS_DET_BATCH;    // detector columns whose term loads a thread keeps in flight   // operand words of the next gate op held in registers

// Shared-memory vectors by 32-bit shared address (gate hot path: explicit
// address arithmetic, loads of a batch issued before its stores)
template <int V> __device__ __forceinline__ VW<V> slds(uint32_t a);
template <> __device__ __forceinline__ VW<4> slds<4>(uint32_t a) {
    VW<4> v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ VW<2> slds<2>(uint32_t a) {
    VW<2> v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.w[0]), "=r"(v.w[1]) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ VW<1> slds<1>(uint32_t a) {
    VW<1> v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v.w[0]) : "r"(a));
    return v;
}
template <int V> __device__ __forceinline__ void ssts(uint32_t a, const VW<V>& v);
template <> __device__ __forceinline__ void ssts<4>(uint32_t a, const VW<4>& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]) : "memory");
}
template <> __device__ __forceinline__ void ssts<2>(uint32_t a, const VW<2>& v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.w[0]), "r"(v.w[1]) : "memory");
}
template <> __device__ __forceinline__ void ssts<1>(uint32_t a, const VW<1>& v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v.w[0]) : "memory");
}

// One batch of gate applications for this lane: operand word = row of target 0
// | row of target 1 << 16 (padding words name the group's dummy row, so no
// lane is predicated off); bx / bz = shared addresses of this lane's vector of
// row 0 in the x / z plane.  All rows of the batch are loaded before any store
// (the applications of an op are independent).
template <int W, uint32_t RULE, int U>
__device__ __forceinline__ void gate_batch(uint32_t bx, uint32_t bz, const uint32_t (&w)[U]) {
    constexpr int V = W >= 4 ? 4 : W;
    constexpr int ar = RULE >= R_CX ? 2 : 1;
    constexpr uint32_t RB = W * 4;  // row bytes
    uint32_t oa[U], ob[U];
    VW<V> x0[U], z0[U], x1[U], z1[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        oa[u] = (w[u] & 0xFFFFu) * RB;
        x0[u] = slds<V>(bx + oa[u]);
        z0[u] = slds<V>(bz + oa[u]);
        if (ar == 2) {
            ob[u] = (w[u] >> 16) * RB;
            x1[u] = slds<V>(bx + ob[u]);
            z1[u] = slds<V>(bz + ob[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        apply_rule<V>(RULE, x0[u], z0[u], x1[u], z1[u]);
        if (ar == 1) {
            if (RULE != R_ZXORX) ssts<V>(bx + oa[u], x0[u]);
            if (RULE != R_XXORZ) ssts<V>(bz + oa[u], z0[u]);
        } else {
            if (RULE != R_CZ) ssts<V>(bx + ob[u], x1[u]);
            if (RULE == R_SWAP) ssts<V>(bx + oa[u], x0[u]);
            ssts<V>(bz + oa[u], z0[u]);
            if (RULE != R_CX) ssts<V>(bz + ob[u], z1[u]);
        }
    }
}

// One gate op in stream form (SOp, lower_stream): the warp's block of packed
// operand words, one word per application, PI = 32 / C applications per warp
// pass; the C lanes that share an application take one V-word vector of its
// rows each.  The words of the first GATE_AHEAD passes arrive in registers
// (pw, loaded while the previous op ran); later passes load one batch ahead.
template <int W, uint32_t RULE>
__device__ __forceinline__ void gate_stream(uint32_t bx, uint32_t bz, const uint32_t* blk, uint32_t K,
                                            const uint32_t (&pw)[GATE_AHEAD], uint32_t nop) {
    constexpr int V = W >= 4 ? 4 : W;
    constexpr int PI = 32 / (W / V);
    constexpr int U = GATE_BATCH;
    static_assert(GATE_AHEAD % U == 0, "whole batches ahead");
#pragma unroll
    for (int k = 0; k < GATE_AHEAD; k += U) {
        if ((uint32_t)k < K) {
            uint32_t w[U];
#pragma unroll
            for (int u = 0; u < U; u++) w[u] = pw[k + u];
            gate_batch<W, RULE, U>(bx, bz, w);
        }
    }
    if (K > (uint32_t)GATE_AHEAD) {
        uint32_t c[U];
#pragma unroll
        for (int u = 0; u < U; u++) c[u] = (GATE_AHEAD + u < K) ? __ldg(blk + (GATE_AHEAD + u) * PI) : nop;
        for (uint32_t k = GATE_AHEAD; k < K; k += U) {
            uint32_t nx[U];
#pragma unroll
            for (int u = 0; u < U; u++) nx[u] = (k + U + u < K) ? __ldg(blk + (k + U + u) * PI) : nop;
            gate_batch<W, RULE, U>(bx, bz, c);
#pragma unroll
            for (int u = 0; u < U; u++) c[u] = nx[u];
        }
    }
}

// The warp's share [A0, A1) of an op's applications (SOp.K / SOp.r0 per warp)
__device__ __forceinline__ void warp_share_of(uint32_t count, uint32_t Kc, int warp, uint32_t& A0, uint32_t& A1) {
    A0 = min(count, (uint32_t)warp * Kc);
    A1 = min(count, A0 + Kc);
}

// Shared-memory map of frame_kernel (word offsets into the dynamic array): the
// per-warp scratch of the general noise paths, the stream ops (when they fit),
// then per group its x plane, z plane and record ring, then the counters.
struct FrameMap {
    uint32_t dsc_word, fr0;
};
__device__ __forceinline__ FrameMap frame_map(const KParams& kp) {
    FrameMap m;
    m.dsc_word = (blockDim.x >> 5) * WSCR;
    m.fr0 = m.dsc_word + (kp.desc_in_smem ? 12u * (uint32_t)kp.n_ops : 0u);
    return m;
}

// General path of an op's fused noise for this warp's applications (rare, out
// of line, few arguments: it rebuilds its context): injected mask rows, or the
// draws made here when noise_kernel did not pre-sample the op (p == 0 / 1,
// heavy noise) or its hits did not fit.  Reads the op's DOp; xg = the group's
// x plane.  Every lane of the warp must call this.
template <int W>
__device__ __noinline__ void fused_noise_general(const KParams& kp, int oi, uint32_t Kc, uint32_t xg, int64_t tile) {
    extern __shared__ __align__(16) uint32_t smem[];
    const DOp o = kp.ops[oi];
    const uint32_t kind = o.kcf & 0xFFu, code = (o.kcf >> 8) & 0xFFu;
    const bool pairs = kind != K_GATE;
    const int ar = (kind == K_GATE && code >= R_CX) ? 2 : 1;
    const NoiseOp nz = decode_noise(o.c, o.d, o.e);
    const uint32_t rowb = kp.masks != nullptr ? __ldg(kp.noise_rowb + nz.ordinal) : 0u;
    const int gsz = blockDim.x / kp.groups;
    const int tid = threadIdx.x % gsz;
    uint32_t A0, A1;
    warp_share_of(o.count, Kc, tid >> 5, A0, A1);
    if (A0 >= A1) return;
    const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
    uint32_t* const X = smem + xg;
    uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    warp_range_noise<W>(kp, tk, nz, kp.noise_tab, o.count, A0, A1, kp.targets + o.off, ar, pairs, X,
                        X + (size_t)(kp.num_qubits + DUMMY_ROWS) * W, sl, smem + (threadIdx.x >> 5) * WSCR, tid & 31, rowb, tile);
}

// A standalone noise op (reads its DOp), out of line
template <int W>
__device__ __noinline__ void noise_general(const KParams& kp, int oi, uint32_t xg, int64_t tile) {
    extern __shared__ __align__(16) uint32_t smem[];
    const DOp o = kp.ops[oi];
    const NoiseOp nz = decode_noise(o.c, o.d, o.e);
    const uint32_t rowb = kp.masks != nullptr ? __ldg(kp.noise_rowb + nz.ordinal) : 0u;
    const int gsz = blockDim.x / kp.groups;
    const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
    uint32_t* const X = smem + xg;
    uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    noise_op<W>(kp, tk, X, X + (size_t)(kp.num_qubits + DUMMY_ROWS) * W, kp.targets + o.off, (o.kcf >> 8) & 0xFFu, o.count, nz, rowb,
                kp.noise_tab, sl, smem + (threadIdx.x >> 5) * WSCR, (int)(threadIdx.x % gsz), gsz, tile);
}

// Pre-sampled hit lists (noise_kernel): the span and first hit entry of the
// next pre-sampled op travel in registers, loaded while the current op runs
struct HitPipe {
    uint2 nsp;                // the next pre-sampled op's span of this warp
    unsigned long long e0n;   // its entry for this lane (0: none)
};
__device__ __forceinline__ unsigned long long first_entry(const unsigned long long* hits, const uint2 sp, int lane) {
    const uint32_t j = sp.x + (uint32_t)lane;
    return (sp.x != NO_SLOT && j < sp.y) ? __ldg(hits + j) : 0ull;
}

// M / R / MR / SPILL items of this warp's targets [A0, A1): (target, vector)
// items over the warp's lanes, four operand pairs in flight.  KIND is a template
// argument: no per-item dispatch.
template <int W, uint32_t KIND>
__device__ __forceinline__ void collapse_kind(const KParams& kp, const TileKey& tk, uint32_t* X, uint32_t* Z,
                                              uint32_t* ring, const uint2* tp, uint32_t A0, uint32_t A1,
                                              uint32_t rec0, uint32_t coin0, int lane, int64_t tile) {
    constexpr int V = W >= 4 ? 4 : W;
    constexpr int C = W / V;
    constexpr int LC = Log2<C>::v;
    batched_items<4>(lane, 32, (int)((A1 - A0) << LC), [&](int i) { return __ldg(tp + A0 + (i >> LC)); },
                     [&](int i, uint2 rs) {
        const uint32_t app = A0 + (uint32_t)(i >> LC);
        const int c = i & (C - 1);
        const bool live = !(rs.x & COIN_DEAD);
        const uint32_t p = (rs.x & ~COIN_DEAD) * W + c * V;
        if (KIND == K_SPILL) {
            vst<V>(ring + rs.y * W + c * V, vld<V>(X + p));
            return;
        }
        if (KIND == K_R) {
            // spill the record homed in x, then reset
            if (rs.y != NO_SLOT) vst<V>(ring + rs.y * W + c * V, vld<V>(X + p));
            vst<V>(X + p, vzero<V>());
            vst<V>(Z + p, live ? coin_vec<W, V>(kp, tk, coin0 + app, c, tile) : vzero<V>());
            return;
        }
        // M / MR: the record is the x row
        if (rs.y != NO_SLOT || kp.rec_out != nullptr || KIND == K_MR) {
            const VW<V> x = vld<V>(X + p);
            if (rs.y != NO_SLOT) vst<V>(ring + rs.y * W + c * V, x);
            if (kp.rec_out != nullptr)
                vst<V>(kp.rec_out + (int64_t)(rec0 + app) * kp.out_row_stride + tile * kp.out_tile_stride + c * V, x);
        }
        if (KIND == K_M) {
            if (live) vst<V>(Z + p, vxor<V>(vld<V>(Z + p), coin_vec<W, V>(kp, tk, coin0 + app, c, tile)));
        } else {  // MR: the measure's coin row (coin0 + 2 app) is overwritten by the reset's
            vst<V>(X + p, vzero<V>());
            vst<V>(Z + p, live ? coin_vec<W, V>(kp, tk, coin0 + 2 * app + 1, c, tile) : vzero<V>());
        }
    });
}
template <int W>
__device__ __forceinline__ void collapse_stream(const KParams& kp, const TileKey& tk, uint32_t* X, uint32_t* Z,
                                                uint32_t* ring, const uint2* tp, uint32_t kind, uint32_t A0,
                                                uint32_t A1, uint32_t rec0, uint32_t coin0, int lane, int64_t tile) {
    switch (kind) {
        case K_R: collapse_kind<W, K_R>(kp, tk, X, Z, ring, tp, A0, A1, rec0, coin0, lane, tile); break;
        case K_M: collapse_kind<W, K_M>(kp, tk, X, Z, ring, tp, A0, A1, rec0, coin0, lane, tile); break;
        case K_MR: collapse_kind<W, K_MR>(kp, tk, X, Z, ring, tp, A0, A1, rec0, coin0, lane, tile); break;
        default: collapse_kind<W, K_SPILL>(kp, tk, X, Z, ring, tp, A0, A1, rec0, coin0, lane, tile); break;
    }
}

// ------------------------------------------------------------ noise kernel
// Pre-samples the fused noise of a launch's tiles (DESIGN.md §4 draws, exactly
// the ones the frame kernel would make inline).  Work item = (tile, fused op,
// consumer warps [wb, we) of the frame kernel): a warp walks the chunks of
// those warps' applications, one chunk per lane per pass (Binomial count from
// block 0, positions from the pairs, distinctness by redraw, the general path
// for long chunks), stages the resolved hit entries (tagged with the consumer
// warp) in shared memory, allocates room in the tile's block with one global
// atomic, and scatters them into one contiguous span per consumer warp.  An
// item whose hits do not fit leaves its warps to draw inline.
template <int W>
__global__ void __launch_bounds__(NK_WARPS * 32, 4) noise_kernel(const __grid_constant__ KParams kp) {
    constexpr int V = W >= 4 ? 4 : W;
    constexpr int C = W / V;
    constexpr uint32_t S = 32u * V;
    __shared__ unsigned long long ent_all[NK_WARPS][NK_SCR];
    __shared__ uint32_t sl_all[NK_WARPS * 32][NZ_MAX_LIST];
    __shared__ uint32_t wc_all[NK_WARPS][2][16];
    __shared__ uint32_t wn_all[NK_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* const ent = ent_all[warp];
    uint32_t* const sl = sl_all[threadIdx.x];
    uint32_t* const wcnt = wc_all[warp][0];
    uint32_t* const wfill = wc_all[warp][1];
    uint32_t* const wn = &wn_all[warp];
    const int64_t items = kp.n_tiles * (int64_t)kp.n_items;
    for (int64_t it = (int64_t)blockIdx.x * NK_WARPS + warp; it < items; it += (int64_t)gridDim.x * NK_WARPS) {
        const int64_t tile = it / kp.n_items;
        const uint2 item = __ldg(kp.hit_items + (it - tile * kp.n_items));
        const uint32_t o = item.x, wb = item.y & 0xFFFFu, we = item.y >> 16;
        const uint4 fi = __ldg(kp.fused + o);
        const NoiseParam np = kp.noise[o];
        const NoiseOp nz = noise_op_of(np, o);
        const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
        const uint32_t K = fi.x;
        const uint32_t A0 = min(np.apps, wb * K), A1 = min(np.apps, we * K);
        const bool pairs = (fi.w & FUSED_PAIRS) != 0;
        const uint32_t* tg = kp.targets + (fi.w & ~FUSED_PAIRS);
        const int ar = np.ch == CH_DEP2 ? 2 : 1;
        if (lane < 16) { wcnt[lane] = 0u; wfill[lane] = 0u; }
        if (lane == 0) *wn = 0u;
        __syncwarp();
        bool over = false;
        if (A0 < A1) {
            const unsigned long long* tab = kp.noise_tab + nz.tab_off;
            const unsigned long long t0 = nz.tab_len > 0 ? tab[0] : ~0ull;
            const unsigned long long t1 = nz.tab_len > 1 ? tab[1] : ~0ull;
            const uint32_t lgca = nz.lgL - nz.lgcs, cs = 1u << nz.lgcs, msk = cs - 1u;
            const uint32_t nS = (32u * W) >> nz.lgcs;
            // chunks per vector m and per application block per_k: powers of two
            const uint32_t lgm = cs >= S ? 0u : (uint32_t)__ffs(S / cs) - 1u;
            const uint32_t lgpk = lgm + (uint32_t)Log2<C>::v;
            const uint32_t k0 = A0 >> lgca;
            const uint32_t nch = ((A1 - A0 + (1u << lgca) - 1) >> lgca) << lgpk;
            const uint32_t sh = 32u - nz.lgL;
            // consumer warp of chunk row kq = kq / (rows per warp), by reciprocal (exact below 2^16)
            const uint32_t rpw = K >> lgca;
            const uint32_t magic = rpw > 1u ? (uint32_t)(0x100000000ull / rpw) + 1u : 0u;
            // a hit into the staging buffer, tagged with its consumer warp
            auto put = [&](uint32_t a0, uint32_t s0, uint32_t wl, uint32_t pos, uint32_t pick) {
                const uint32_t slot = atomicAdd(wn, 1u);
                if (slot < (uint32_t)NK_SCR) {
                    ent[slot] = make_hit<W>(app_rows(tg, a0 + (pos >> nz.lgcs), ar, pairs), nz.ch, pick, s0 + (pos & msk)) |
                                ((unsigned long long)wl << 56);
                    atomicAdd(&wcnt[wl], 1u);
                }
            };
            for (uint32_t q0 = 0; q0 < nch; q0 += 32) {
                // ---- phase 1, one chunk per lane: Binomial count from Philox block 0
                const uint32_t q = q0 + (uint32_t)lane;
                const bool valid = q < nch;
                const uint32_t kq = q >> lgpk, rem = q & ((1u << lgpk) - 1u);
                const uint32_t c = rem >> lgm, u = rem & ((1u << lgm) - 1u);
                const uint32_t k = k0 + kq;
                const uint32_t r = k * nS + (c << lgm) + u;
                const uint32_t a0 = k << lgca;
                const uint32_t vl = valid ? (min(1u << lgca, np.apps - a0) << nz.lgcs) : 0u;
                const uint32_t s0 = c * S + u * cs;
                const uint32_t wl = rpw > 1u ? __umulhi(kq, magic) : kq;  // consumer warp (item-local)
                uint32_t w2 = 0u, w3 = 0u, cnt = 0u;
                if (valid) {
                    uint32_t w0 = 0u, w1 = r;
                    w2 = tk.g; w3 = DOMAIN_NOISE | nz.ordinal;  // block 0
                    philox_rounds(w0, w1, w2, w3, tk.k0, tk.k1);
                    const unsigned long long uu = ((unsigned long long)w1 << 32) | w0;
                    cnt = (nz.tab_len > 0 && uu >= t0) ? ((nz.tab_len > 1 && uu >= t1) ? 2u : 1u) : 0u;
                    if (cnt == 2u)
                        while (cnt < nz.tab_len && uu >= tab[cnt]) cnt++;
                }
                bool general = cnt > (uint32_t)NZ_MAX_LIST;
                const uint32_t cf = general ? 0u : cnt;  // hits drawn by the hit-parallel phase
                uint32_t pre = cf;                        // inclusive prefix over the lanes
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                    if (lane >= d) pre += v;
                }
                const uint32_t excl = pre - cf;
                // ---- phase 2, one hit per lane: runs of whole chunks with at most 32 hits;
                // hit h of a chunk takes word pair h (block (h + 1) >> 1; pair 0 = block 0's w2, w3)
                uint32_t regen = 0u;  // chunks whose positions collide: the reference path redraws them
                for (uint32_t c0 = 0; c0 < 32u;) {
                    const uint32_t base = __shfl_sync(0xFFFFFFFFu, excl, (int)c0);
                    const uint32_t inm = __ballot_sync(0xFFFFFFFFu, (uint32_t)lane >= c0 && pre - base <= 32u);
                    const uint32_t c1 = c0 + (uint32_t)__popc(inm);
                    const uint32_t Hs = __shfl_sync(0xFFFFFFFFu, pre, (int)c1 - 1) - base;
                    if (Hs > 0u) {
                        const uint32_t j = (uint32_t)lane;
                        const bool mine = j < Hs;
                        uint32_t lo = c0;  // owner chunk: the first lane in [c0, c1) with pre - base > j
#pragma unroll
                        for (int st = 16; st > 0; st >>= 1) {
                            const uint32_t idx = lo + (uint32_t)st - 1u;
                            const uint32_t pv = __shfl_sync(0xFFFFFFFFu, pre, (int)min(idx, 31u)) - base;
                            if (idx < c1 && pv <= j) lo = idx + 1u;
                        }
                        const int o = (int)min(lo, c1 - 1u);
                        const uint32_t h = j - (__shfl_sync(0xFFFFFFFFu, excl, o) - base);
                        const uint32_t o_cnt = __shfl_sync(0xFFFFFFFFu, cf, o);
                        const uint32_t o_r = __shfl_sync(0xFFFFFFFFu, r, o);
                        const uint32_t o_a0 = __shfl_sync(0xFFFFFFFFu, a0, o);
                        const uint32_t o_vl = __shfl_sync(0xFFFFFFFFu, vl, o);
                        const uint32_t o_s0 = __shfl_sync(0xFFFFFFFFu, s0, o);
                        const uint32_t o_wl = __shfl_sync(0xFFFFFFFFu, wl, o);
                        uint32_t x = __shfl_sync(0xFFFFFFFFu, w2, o);
                        uint32_t y = __shfl_sync(0xFFFFFFFFu, w3, o);
                        if (__any_sync(0xFFFFFFFFu, mine && h > 0u)) {
                            uint32_t b0 = (h + 1u) >> 1, b1 = o_r, b2 = tk.g, b3 = DOMAIN_NOISE | nz.ordinal;
                            philox_rounds(b0, b1, b2, b3, tk.k0, tk.k1);
                            if (h > 0u) { x = (h & 1u) ? b0 : b2; y = (h & 1u) ? b1 : b3; }
                        }
                        const uint32_t pos = nz.lgL ? (x >> sh) : 0u;
                        const uint32_t pick = nz.npat > 1 ? __umulhi(y, nz.npat) : 0u;
                        // the positions of one chunk must be distinct: compare with the earlier siblings
                        const uint32_t maxh = __reduce_max_sync(0xFFFFFFFFu, mine ? h : 0u);
                        bool dup = false;
                        for (uint32_t d = 1; d <= maxh; d++) {
                            const uint32_t p = __shfl_up_sync(0xFFFFFFFFu, pos, d);
                            if (mine && h >= d) dup |= p == pos;
                        }
                        const uint32_t dupm = __ballot_sync(0xFFFFFFFFu, mine && dup);
                        const uint32_t sib = (o_cnt >= 32u ? 0xFFFFFFFFu : ((1u << o_cnt) - 1u)) << (j - h);
                        const bool cdup = mine && (dupm & sib) != 0u;
                        if (mine && !cdup && pos < o_vl) put(o_a0, o_s0, o_wl, pos, pick);
                        regen |= __reduce_or_sync(0xFFFFFFFFu, (cdup && h == 0u) ? (1u << o) : 0u);
                    }
                    c0 = c1;
                }
                // ---- phase 3 (rare): long or colliding chunks through the reference path
                general |= ((regen >> lane) & 1u) != 0u;
                if (general)
                    noise_chunk(tk, nz, kp.noise_tab, r, vl, sl,
                                [&](uint32_t pos, uint32_t pick) { put(a0, s0, wl, pos, pick); });
            }
            __syncwarp();
            over = *wn > (uint32_t)NK_SCR;
        }
        const uint32_t n = over ? 0u : *wn;
        uint2* spans = kp.spans_global + (tile * kp.num_noise + o) * kp.list_warps;
        uint32_t base = 0u;
        if (lane == 0 && !over && n > 0u) base = atomicAdd(kp.fill_global + 2 * tile, n);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        over |= (int64_t)base + n > kp.hit_block;
        // an item whose hits did not fit sends its tile through the general
        // frame loop (its consumer warps draw inline)
        if (lane == 0 && over) kp.fill_global[2 * tile + 1] = 1u;
        // consumer warp spans: exclusive prefix of the per-warp counts
        const uint32_t nwl = we - wb;
        uint32_t v = (uint32_t)lane < nwl ? wcnt[lane] : 0u, pre = v;
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, pre, d);
            if (lane >= d) pre += t;
        }
        if ((uint32_t)lane < nwl) {
            const uint32_t beg = base + pre - v;
            spans[wb + lane] = over ? make_uint2(NO_SLOT, 0u) : make_uint2(beg, beg + v);
            wfill[lane] = beg;
        }
        __syncwarp();
        if (!over) {
            unsigned long long* hits = kp.hits_global + tile * kp.hit_block;
            for (uint32_t i = (uint32_t)lane; i < n; i += 32) {
                const unsigned long long e = ent[i];
                const uint32_t slot = atomicAdd(&wfill[(uint32_t)(e >> 56) & 15u], 1u);
                hits[slot] = e & ((1ull << 56) - 1);
            }
        }
        __syncwarp();  // staging reused by the next item
    }
}

cudaError_t launch_noise_kernel(int W, const KParams& kp, int grid, cudaStream_t st) {
    if (kp.n_tiles <= 0 || kp.n_items <= 0) return cudaSuccess;
    switch (W) {
        case 1: noise_kernel<1><<<grid, NK_WARPS * 32, 0, st>>>(kp); break;
        case 2: noise_kernel<2><<<grid, NK_WARPS * 32, 0, st>>>(kp); break;
        case 4: noise_kernel<4><<<grid, NK_WARPS * 32, 0, st>>>(kp); break;
        case 8: noise_kernel<8><<<grid, NK_WARPS * 32, 0, st>>>(kp); break;
        case 16: noise_kernel<16><<<grid, NK_WARPS * 32, 0, st>>>(kp); break;
        case 32: noise_kernel<32><<<grid, NK_WARPS * 32, 0, st>>>(kp); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------ frame kernel
// One tile of one thread group: the stream ops (SOp) over the group's frame in
// shared memory.  Per op a thread reads three descriptor vectors, prefetches
// the next op's operand block, passes the group barrier where the compiler
// found a conflict, and walks its warp's operand words.  Fused noise comes from
// noise_kernel's per-warp hit spans (span and first entry prefetched one
// pre-sampled op ahead).  GENERAL = false is the hot instantiation: every noise
// instruction is fused and pre-sampled and no list overflowed, so the loop
// makes no calls (a call inside it makes ptxas spill the loop's live values);
// GENERAL = true adds the out-of-line paths (injected masks, inline draws,
// standalone noise ops) and runs as one call per tile.
template <int W, bool RING_SMEM, bool GENERAL>
__device__ __forceinline__ void frame_tile_body(const KParams& kp, const int64_t tile) {
    constexpr int V = W >= 4 ? 4 : W;  // words per vector access
    constexpr int C = W / V;           // vectors per row
    constexpr int LC = Log2<C>::v;
    constexpr int PI = 32 / C;         // applications per warp pass
    extern __shared__ __align__(16) uint32_t smem[];
    const int n = kp.num_qubits;
    const int G = kp.groups;
    const int gsz = blockDim.x / G;
    const int grp = threadIdx.x / gsz;
    const int tid = threadIdx.x - grp * gsz;  // thread index within the group
    const int nth = gsz;
    const int lane = tid & 31, warp = tid >> 5;
    // each plane has n rows and DUMMY_ROWS dummy rows (rows n ..): the targets of padding operand words
    const uint32_t zoff = (uint32_t)(n + DUMMY_ROWS) * W;
    const uint32_t gw = 2u * zoff + (RING_SMEM ? (uint32_t)kp.num_slots * W : 0u);  // words per group
    const FrameMap fm = frame_map(kp);
    const uint32_t xg = fm.fr0 + (uint32_t)grp * gw;  // the group's x plane
    uint32_t* const X = smem + xg;
    uint32_t* const Z = X + zoff;
    uint32_t* const ring = RING_SMEM ? (Z + zoff)
                                     : (kp.ring_global + ((size_t)blockIdx.x * G + grp) * kp.num_slots * W);
    uint32_t* const cnt = smem + fm.fr0 + (uint32_t)G * gw;
    const uint4* const dsc_s = reinterpret_cast<const uint4*>(smem + fm.dsc_word);
    const uint4* const dsc_g = reinterpret_cast<const uint4*>(kp.sops);
    const bool dsm = kp.desc_in_smem != 0;
    const bool use_lists = !GENERAL || (kp.hits_global != nullptr && kp.masks == nullptr);
    const uint32_t bar_id = 1u + (uint32_t)grp;
    auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(gsz) : "memory"); };
    // shared addresses of this lane's vector of row 0 in the x / z plane
    const uint32_t bx = (uint32_t)__cvta_generic_to_shared(X + (lane & (C - 1)) * V);
    const uint32_t bz = bx + zoff * 4u;
    const uint32_t nop = ((uint32_t)n + ((uint32_t)(lane >> LC) & (DUMMY_ROWS - 1))) * 0x10001u;  // a dummy row
    // one generic load serves both placements (two predicated loads per vector
    // cost 5 % of the d=25 kernel time; d=100, descriptors in global memory, loses 2 %)
    const uint4* const dsc_any = dsm ? dsc_s : dsc_g;
    auto ldesc = [&](int i) -> uint4 { return dsc_any[i]; };

    const unsigned long long* const hits = kp.hits_global + tile * kp.hit_block;
    const uint2* const spans = kp.spans_global + (tile * kp.num_noise) * kp.list_warps + warp;
    HitPipe hp{make_uint2(NO_SLOT, 0u), 0ull};
    if (use_lists && kp.first_span != NO_SLOT) hp.nsp = __ldg(spans + kp.first_span);
    {
        // ---- FrameBatch.__init__: x = 0, z = coin rows 0..n-1 (frame_sim.py:36-39) ----
        const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
        for (int i = tid; i < (n << LC); i += nth) {
            const int q = i >> LC, c = i & (C - 1);
            const uint32_t row = __ldg(kp.row_of + q);
            const bool live = !((__ldg(kp.init_dead + (q >> 5)) >> (q & 31)) & 1u);
            vst<V>(X + (size_t)row * W + c * V, vzero<V>());
            vst<V>(Z + (size_t)row * W + c * V, live ? coin_vec<W, V>(kp, tk, (uint32_t)q, c, tile) : vzero<V>());
        }
        for (int i = tid; i < (kp.num_obs << LC); i += nth) {
            const int k = i >> LC, c = i & (C - 1);
            vst<V>(ring + (size_t)k * W + c * V, vzero<V>());
        }
    }
    if (use_lists) hp.e0n = first_entry(hits, hp.nsp, lane);
    group_sync();

    // the first descriptor vector runs one op ahead; a gate op's first
    // GATE_AHEAD operand words are loaded while the op before it runs
    uint4 nd0 = kp.n_ops > 0 ? ldesc(0) : make_uint4(0, 0, 0, 0);
    uint32_t nw[GATE_AHEAD];
    auto load_ahead = [&]() {
        if ((nd0.x & 0xFFu) == K_GATE) {
            // (a warp's block holds at least GATE_AHEAD passes of words: no predicates)
            const uint32_t* const nblk = kp.arena + nd0.z + (uint32_t)warp * max(nd0.w, (uint32_t)GATE_AHEAD) * PI + (lane >> LC);
#pragma unroll
            for (int j = 0; j < GATE_AHEAD; j++) nw[j] = __ldg(nblk + j * PI);
        }
    };
#pragma unroll
    for (int j = 0; j < GATE_AHEAD; j++) nw[j] = nop;
    load_ahead();
    for (int oi = 0; oi < kp.n_ops; oi++) {
#if PFS_PROFILE
        const bool stamp = kp.op_clock != nullptr && blockIdx.x == 0 && grp == 0 && tid == 0 && tile == 0;
        if (stamp) kp.op_clock[(size_t)kp.n_ops * 9 + oi] = clock64();   // op top (before the header)
#endif
        const uint4 d0 = nd0;
        const uint4 d1 = ldesc(3 * oi + 1), d2 = ldesc(3 * oi + 2);
        uint32_t pw[GATE_AHEAD];
#pragma unroll
        for (int j = 0; j < GATE_AHEAD; j++) pw[j] = nw[j];
        if (oi + 1 < kp.n_ops) {
            nd0 = ldesc(3 * oi + 3);
            if (!dsm && lane == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(dsc_g + 3 * oi + 6));
            load_ahead();
        }
        const uint32_t kind = d0.x & 0xFFu, code = (d0.x >> 8) & 0xFFu, flags = d0.x >> 16;
        const uint32_t count = d0.y, off = d0.z, K = d0.w;
        const bool fz = (flags & F_NOISE) != 0;
        // this op's pre-sampled hits: its span (prefetched); start the next
        // pre-sampled op's span load
        const bool pre = GENERAL ? (use_lists && (flags & F_PRESAMPLED)) : fz;
        uint2 sp = make_uint2(NO_SLOT, 0u);
        if (pre) {
            sp = hp.nsp;
            hp.nsp = __ldg(spans + d1.w);
        }
#if PFS_PROFILE
        if (stamp) kp.op_clock[(size_t)kp.n_ops * 11 + oi] = clock64();  // header done, at the barrier
#endif
        if (flags & F_BARRIER) group_sync();
#if PFS_PROFILE
        if (kp.op_clock != nullptr && blockIdx.x == 0 && grp == 0 && tid == 0 &&
            tile == 0)  // profiling: op-boundary timestamps of the first tile
            kp.op_clock[oi] = clock64();
        if (kp.debug_skip) {
            const uint32_t bit = kind == K_NOISE ? 1u : kind == K_DET ? 8u : kind == K_GATE ? 16u
                               : (kind == K_M || kind == K_R || kind == K_MR) ? 32u : 0u;
            if (kp.debug_skip & bit) continue;
        }
#endif
        // the fused noise of this warp's applications (Kc per warp), then
        // the first entry of the next pre-sampled op (its span has arrived)
        auto fused_noise = [&](uint32_t Kc) {
#if PFS_PROFILE
            if (kp.debug_skip & 2) return;
#endif
            if (!GENERAL || (pre && sp.x != NO_SLOT)) {
                __syncwarp();  // the warp's row updates are visible to the lanes applying hits
                uint32_t j = sp.x + (uint32_t)lane;
                const uint32_t xa = (uint32_t)__cvta_generic_to_shared(X);
                if (j < sp.y) apply_hit_entry(xa, zoff * 4u, hp.e0n);
                for (j += 32u; j < sp.y; j += 32u) apply_hit_entry(xa, zoff * 4u, __ldg(hits + j));
            } else if (GENERAL) {
                fused_noise_general<W>(kp, oi, Kc, xg, tile);
            }
            if (pre) hp.e0n = first_entry(hits, hp.nsp, lane);
        };

        switch (kind) {
        case K_GATE: {
            const uint32_t* const blk = kp.arena + off + (uint32_t)warp * max(K, (uint32_t)GATE_AHEAD) * PI + (lane >> LC);
            switch (code) {
                case R_SWAPXZ: gate_stream<W, R_SWAPXZ>(bx, bz, blk, K, pw, nop); break;
                case R_ZXORX: gate_stream<W, R_ZXORX>(bx, bz, blk, K, pw, nop); break;
                case R_XXORZ: gate_stream<W, R_XXORZ>(bx, bz, blk, K, pw, nop); break;
                case R_CX: gate_stream<W, R_CX>(bx, bz, blk, K, pw, nop); break;
                case R_CZ: gate_stream<W, R_CZ>(bx, bz, blk, K, pw, nop); break;
                case R_CY: gate_stream<W, R_CY>(bx, bz, blk, K, pw, nop); break;
                case R_SWAP: gate_stream<W, R_SWAP>(bx, bz, blk, K, pw, nop); break;
                default: break;
            }
#if PFS_PROFILE
            if (stamp) kp.op_clock[(size_t)kp.n_ops * 10 + oi] = clock64();  // gate rows done
#endif
            if (fz) fused_noise(d2.z);
            break;
        }
        case K_R: case K_M: case K_MR: case K_SPILL: {
            uint32_t A0, A1;
            warp_share_of(count, K, warp, A0, A1);
            // fused noise precedes a measurement (X_ERROR before M), follows a reset
            if (fz && kind != K_R) fused_noise(K);
            if (A0 < A1 && !(flags & F_NOROWS)) {
                const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
                collapse_stream<W>(kp, tk, X, Z, ring, reinterpret_cast<const uint2*>(kp.arena + off), kind, A0, A1,
                                   d1.x, d1.y, lane, tile);
            }
            if (fz && kind == K_R) fused_noise(K);
            break;
        }
        case K_NOISE:
#if PFS_PROFILE
            if (kp.debug_skip & 2) break;
#endif
            if (GENERAL) noise_general<W>(kp, oi, xg, tile);
            break;
        case K_DET: {
            const uint32_t oa = d1.x;
            const int items = (int)(count << LC);
            // a term is a ring slot, or XROW | row: the record still in that
            // x row.  Uniform ops (code = terms per column) read their terms
            // from the arena block, the others through the CSR arrays.
            auto src = [&](uint32_t t) -> const uint32_t* {
                return (t & XROW) ? X + (size_t)(t & ~XROW) * W : ring + (size_t)t * W;
            };
            if (RING_SMEM && code >= 1u && code <= 2u && kp.counts == nullptr && kp.ev_out != nullptr) {
                // one or two terms per column, events to the scratch table: all
                // term loads of a batch, then all row loads, then the stores
                constexpr uint32_t RB = W * 4;
                constexpr int U = 4;
                const uint32_t xa = (uint32_t)__cvta_generic_to_shared(X);
                const uint32_t ra = (uint32_t)__cvta_generic_to_shared(ring);
                uint32_t* const evt = kp.ev_out + tile * kp.out_tile_stride;
                const int64_t rs = kp.out_row_stride;
                for (int i0 = tid; i0 < items; i0 += U * nth) {
                    uint32_t t0[U], t1[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int i = i0 + u * nth;
                        t0[u] = t1[u] = NO_SLOT;
                        if (i < items) {
                            const uint32_t* const e = kp.arena + off + (uint32_t)(i >> LC) * code;
                            t0[u] = __ldg(e);
                            if (code == 2u) t1[u] = __ldg(e + 1);
                        }
                    }
                    VW<V> a[U], b[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const uint32_t cb = (uint32_t)((i0 + u * nth) & (C - 1)) * (V * 4);
                        a[u] = b[u] = vzero<V>();
                        if (t0[u] != NO_SLOT)
                            a[u] = slds<V>(((t0[u] & XROW) ? xa + (t0[u] & ~XROW) * RB : ra + t0[u] * RB) + cb);
                        if (t1[u] != NO_SLOT)
                            b[u] = slds<V>(((t1[u] & XROW) ? xa + (t1[u] & ~XROW) * RB : ra + t1[u] * RB) + cb);
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int i = i0 + u * nth;
                        if (i < items)  // streaming store: the scratch must not evict the hit lists from L2
                            vstcs<V>(evt + (int64_t)(oa + (uint32_t)(i >> LC)) * rs + (i & (C - 1)) * V, vxor<V>(a[u], b[u]));
                    }
                }
                break;
            }
            const uint32_t* const tb = code ? kp.arena : kp.det_terms;
            batched_items<DET_BATCH>(tid, nth, items,
                [&](int i) {
                    const uint32_t ci = (uint32_t)(i >> LC);
                    const uint32_t col = oa + ci;
                    uint32_t e0, e1;
                    if (code) { e0 = off + ci * code; e1 = e0 + code; }
                    else { e0 = __ldg(kp.det_ptr + col); e1 = __ldg(kp.det_ptr + col + 1); }
                    const uint32_t s0 = e0 < e1 ? __ldg(tb + e0) : NO_SLOT;
                    const uint32_t s1 = e0 + 1 < e1 ? __ldg(tb + e0 + 1) : NO_SLOT;
                    return make_uint4(e0, e1, s0, s1);
                },
                [&](int i, uint4 d) {
                    const uint32_t col = oa + (uint32_t)(i >> LC);
                    const int c = i & (C - 1);
                    VW<V> acc = vzero<V>();
                    if (d.z != NO_SLOT) acc = vld<V>(src(d.z) + c * V);
                    if (d.w != NO_SLOT) acc = vxor<V>(acc, vld<V>(src(d.w) + c * V));
                    for (uint32_t e = d.x + 2; e < d.y; e++) acc = vxor<V>(acc, vld<V>(src(__ldg(tb + e)) + c * V));
                    if (kp.ev_out != nullptr)
                        vst<V>(kp.ev_out + (int64_t)col * kp.out_row_stride + tile * kp.out_tile_stride + c * V, acc);
                    if (kp.counts != nullptr) {
                        uint32_t tot = 0;
#pragma unroll
                        for (int jw = 0; jw < V; jw++) {
                            const int64_t s0 = tile * (int64_t)(32 * W) + 32 * (c * V + jw);
                            const int64_t rem = kp.num_shots - s0;
                            const uint32_t m = rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
                            tot += __popc(acc.w[jw] & m);
                        }
                        if (tot) {
                            if (kp.counts_in_smem) atomicAdd(cnt + col, tot);
                            else atomicAdd(kp.counts + col, (unsigned long long)tot);
                        }
                    }
                });
            break;
        }
        case K_OBS: {
            const uint32_t oa = d1.x;
            const uint32_t* const tg = kp.arena + off;
            for (int c = tid; c < C; c += nth) {
                VW<V> acc = vld<V>(ring + (size_t)oa * W + c * V);
                for (uint32_t j = 0; j < count; j++) {
                    const uint32_t t = __ldg(tg + j);
                    const uint32_t* s = (t & XROW) ? X + (size_t)(t & ~XROW) * W : ring + (size_t)t * W;
                    acc = vxor<V>(acc, vld<V>(s + c * V));
                }
                vst<V>(ring + (size_t)oa * W + c * V, acc);
            }
            break;
        }
        default: break;
        }
#if PFS_PROFILE
        if (kp.op_clock != nullptr && blockIdx.x == 0 && grp == 0 && tile == 0 &&
            (tid & 31) == 0 && (tid >> 5) < 8)  // profiling: per-warp end of op work
            kp.op_clock[(size_t)kp.n_ops * (1 + (tid >> 5)) + oi] = clock64();
#endif
    }
    group_sync();  // the group's frame is reused by its next tile
}

template <int W, bool RING_SMEM>
__device__ __noinline__ void frame_tile_general(const KParams& kp, const int64_t tile) {
    frame_tile_body<W, RING_SMEM, true>(kp, tile);
}

// Persistent kernel: kp.groups independent thread groups per CTA, each with
// its own tile, frame (x plane, z plane), record ring and named barrier — one
// group's op latency overlaps the other group's work.
template <int W, bool RING_SMEM>
__global__ void __launch_bounds__(FRAME_MAX_THREADS, 1) frame_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int G = kp.groups;
    const int grp = threadIdx.x / (blockDim.x / G);
    const FrameMap fm = frame_map(kp);
    const uint32_t gw = 2u * (uint32_t)(kp.num_qubits + DUMMY_ROWS) * W + (RING_SMEM ? (uint32_t)kp.num_slots * W : 0u);
    uint32_t* const cnt = smem + fm.fr0 + (uint32_t)G * gw;
    if (kp.counts_in_smem)
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x) cnt[i] = 0u;
    if (kp.desc_in_smem) {
        uint4* const d = reinterpret_cast<uint4*>(smem + fm.dsc_word);
        const uint4* const dsc_g = reinterpret_cast<const uint4*>(kp.sops);
        for (int i = threadIdx.x; i < 3 * kp.n_ops; i += blockDim.x) d[i] = __ldg(dsc_g + i);
    }
    __syncthreads();
    for (int64_t tile = (int64_t)blockIdx.x * G + grp; tile < kp.n_tiles; tile += (int64_t)gridDim.x * G) {
        // the hot loop serves programs whose noise is all fused and pre-sampled,
        // for tiles whose hit lists all fitted (noise_kernel's overflow mark)
        const bool fast = kp.all_presampled && kp.hits_global != nullptr && kp.masks == nullptr &&
                          __ldg(kp.fill_global + 2 * tile + 1) == 0u;
        if (fast) frame_tile_body<W, RING_SMEM, false>(kp, tile);
        else frame_tile_general<W, RING_SMEM>(kp, tile);
    }
    if (kp.counts_in_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x)
            if (cnt[i]) atomicAdd(kp.counts + i, (unsigned long long)cnt[i]);
    }
}


// x and z planes of num_qubits rows plus the dummy rows padding operand words name
size_t frame_smem_bytes(int num_qubits, int W) { return (size_t)2 * (num_qubits + DUMMY_ROWS) * W * 4; }

template <int W, bool RS>
static cudaError_t launch_t(const LaunchCfg& cfg, const KParams& kp, cudaStream_t st) {
    frame_kernel<W, RS><<<cfg.grid, cfg.threads, cfg.smem_bytes, st>>>(kp);
    return cudaGetLastError();
}
template <int W, bool RS>
static cudaError_t smem_t(const LaunchCfg& cfg) {
    return cudaFuncSetAttribute(frame_kernel<W, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)cfg.smem_bytes);
}

#define PFS_DISPATCH(FN, ...)                                                        \
    switch (cfg.W) {                                                                 \
        case 1: return cfg.ring_smem ? FN<1, true>(__VA_ARGS__) : FN<1, false>(__VA_ARGS__);   \
        case 2: return cfg.ring_smem ? FN<2, true>(__VA_ARGS__) : FN<2, false>(__VA_ARGS__);   \
        case 4: return cfg.ring_smem ? FN<4, true>(__VA_ARGS__) : FN<4, false>(__VA_ARGS__);   \
        case 8: return cfg.ring_smem ? FN<8, true>(__VA_ARGS__) : FN<8, false>(__VA_ARGS__);   \
        case 16: return cfg.ring_smem ? FN<16, true>(__VA_ARGS__) : FN<16, false>(__VA_ARGS__); \
        case 32: return cfg.ring_smem ? FN<32, true>(__VA_ARGS__) : FN<32, false>(__VA_ARGS__); \
        default: return cudaErrorInvalidValue;                                       \
    }

cudaError_t launch_frame_kernel(const LaunchCfg& cfg, const KParams& kp, cudaStream_t stream) {
    PFS_DISPATCH(launch_t, cfg, kp, stream)
}
cudaError_t set_frame_kernel_smem(const LaunchCfg& cfg) { PFS_DISPATCH(smem_t, cfg) }

// ------------------------------------------------------------ transpose
// Tile: 256 rows x 512 shots.  Block of 256 threads (8 warps).
constexpr int TR_ROWS = 256;
constexpr int TR_WORDS = 16;  // 512 shots


__global__ void __launch_bounds__(256) rows_to_b8_kernel(const uint32_t* __restrict__ rows,
                                                         int64_t num_rows, int64_t row_words,
                                                         int64_t num_shots,
                                                         const uint8_t* __restrict__ xor_bits,
                                                         uint8_t* __restrict__ out, int64_t pitch) {
    __shared__ uint32_t tin[TR_ROWS][TR_WORDS + 1];
    __shared__ uint32_t tout[TR_WORDS * 32][TR_ROWS / 32 + 1];
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.y * TR_ROWS;
    const int64_t w0 = (int64_t)blockIdx.x * TR_WORDS;
    {
        const int64_t r = r0 + t;
        uint32_t v[TR_WORDS];
        if (r < num_rows) {
            const uint32_t* src = rows + r * row_words + w0;
            if (w0 + TR_WORDS <= row_words && (row_words & 3) == 0) {
#pragma unroll
                for (int k = 0; k < TR_WORDS / 4; k++) {
                    const uint4 q = __ldg(reinterpret_cast<const uint4*>(src) + k);
                    v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
                }
            } else {
#pragma unroll
                for (int k = 0; k < TR_WORDS; k++) v[k] = (w0 + k < row_words) ? __ldg(src + k) : 0u;
            }
            if (xor_bits != nullptr && (__ldg(xor_bits + r) & 1u)) {
#pragma unroll
                for (int k = 0; k < TR_WORDS; k++) v[k] = ~v[k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < TR_WORDS; k++) v[k] = 0u;
        }
#pragma unroll
        for (int k = 0; k < TR_WORDS; k++) tin[t][k] = v[k];
    }
    __syncthreads();
    const int warp = t >> 5, lane = t & 31;
    for (int pair = warp; pair < (TR_ROWS / 32) * TR_WORDS; pair += 8) {
        const int rb = pair / TR_WORDS, w = pair % TR_WORDS;
        uint32_t v = tin[rb * 32 + lane][w];
        v = transpose32_lane(v, lane);
        tout[w * 32 + lane][rb] = v;
    }
    __syncthreads();
    const int64_t nbytes = (num_rows + 7) >> 3;
    const int64_t b0 = r0 >> 3;
    const int64_t span = (nbytes - b0) < 32 ? (nbytes - b0) : 32;
    const bool full = (pitch & 15) == 0 && ((uintptr_t)out & 15) == 0 && b0 + 32 <= pitch;
    if (full) {
        for (int sl = t; sl < TR_WORDS * 32; sl += 256) {
            const int64_t s = w0 * 32 + sl;
            if (s >= num_shots) break;
            uint4* dst = reinterpret_cast<uint4*>(out + s * pitch + b0);
            dst[0] = make_uint4(tout[sl][0], tout[sl][1], tout[sl][2], tout[sl][3]);
            dst[1] = make_uint4(tout[sl][4], tout[sl][5], tout[sl][6], tout[sl][7]);
        }
    } else {
        // unaligned pitch (exact b8 rows): one warp per shot row, one byte per
        // lane, so each store instruction writes one contiguous 32-byte run
        for (int sl = warp; sl < TR_WORDS * 32; sl += 8) {
            const int64_t s = w0 * 32 + sl;
            if (s >= num_shots) break;
            if (lane < span)
                out[s * pitch + b0 + lane] = (uint8_t)(tout[sl][lane >> 2] >> ((lane & 3) * 8));
        }
    }
}

// Tile-major input: block (tile t, rows r0..r0+255) is one contiguous run of
// 256 W words, so loads are fully coalesced; each shot's 32 output bytes are
// one aligned sector when the pitch allows.
// TW = tile words, W = words handled per CTA (TW > 16 splits a tile in parts)
template <int TW, int W, bool WM>
__global__ void __launch_bounds__(256) tiles_to_b8_kernel(const uint32_t* __restrict__ tiles,
                                                          int64_t num_rows, int64_t num_shots,
                                                          const uint8_t* __restrict__ xor_bits,
                                                          uint8_t* __restrict__ out, int64_t pitch) {
    constexpr int Wp = W + 1;
    constexpr int PARTS = TW / W;
    // tin and tout share one buffer (the transposed words wait in registers
    // across a barrier): ~9 KB at W = 8, so a CTA fits beside a frame CTA
    constexpr int TIN = 256 * Wp, TOUT = 32 * W * 9;
    __shared__ uint32_t tbuf[TIN > TOUT ? TIN : TOUT];
    uint32_t* const tin = tbuf;
    uint32_t* const tout = tbuf;
    const int t = threadIdx.x;
    // row block fastest: the CTAs writing one shot's consecutive 32-byte runs
    // run together, so their sectors merge into whole lines in L2
    const int64_t nrb = (num_rows + 255) >> 8;
    const int64_t rest = (int64_t)blockIdx.x / nrb;
    const int64_t tile = rest / PARTS;
    const int part = (int)(rest % PARTS);
    const int64_t r0 = ((int64_t)blockIdx.x % nrb) * 256;
    const int rows = (int)((num_rows - r0) < 256 ? (num_rows - r0) : 256);
    const uint32_t* src = WM ? tiles + tile * num_rows * TW + (int64_t)part * W * num_rows + r0
                             : tiles + tile * num_rows * TW + r0 * TW + part * W;
    // thread t owns row t of the block: its W words are contiguous (16-byte
    // vector loads when W >= 4), all issued before use; word-major input: one
    // coalesced 1 KB run per word
    const int r = t;
    uint32_t v[W];
    if (r < rows) {
        const uint32_t* rp = src + (size_t)r * TW;
        if constexpr (WM) {
#pragma unroll
            for (int k = 0; k < W; k++) v[k] = __ldg(src + (int64_t)k * num_rows + r);
        } else if constexpr (W >= 4) {
#pragma unroll
            for (int k = 0; k < W / 4; k++) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(rp) + k);
                v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < W; k++) v[k] = __ldg(rp + k);
        }
        if (xor_bits != nullptr && (__ldg(xor_bits + r0 + r) & 1u)) {
#pragma unroll
            for (int k = 0; k < W; k++) v[k] = ~v[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < W; k++) v[k] = 0u;
    }
#pragma unroll
    for (int k = 0; k < W; k++) tin[r * Wp + k] = v[k];
    __syncthreads();
    const int warp = t >> 5, lane = t & 31;
    uint32_t xt[W];  // pairs warp, warp + 8, ... (8 W pairs over 8 warps)
#pragma unroll
    for (int k = 0; k < W; k++) {
        const int pair = warp + 8 * k, rb = pair / W, w = pair % W;
        xt[k] = transpose32_lane(tin[(rb * 32 + lane) * Wp + w], lane);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < W; k++) {
        const int pair = warp + 8 * k, rb = pair / W, w = pair % W;
        tout[(w * 32 + lane) * 9 + rb] = xt[k];
    }
    __syncthreads();
    const int64_t nbytes = (num_rows + 7) >> 3;
    const int64_t b0 = r0 >> 3;
    const int64_t span = (nbytes - b0) < 32 ? (nbytes - b0) : 32;
    const int64_t s0 = tile * 32 * TW + part * 32 * W;
    const bool full = (pitch & 15) == 0 && ((uintptr_t)out & 15) == 0 && b0 + 32 <= pitch;
    if (full) {
        // two lanes per shot, 16 bytes each: a store instruction writes 16
        // whole 32-byte runs instead of 32 half ones
        for (int i = t; i < 64 * W; i += 256) {
            const int sl = i >> 1, half = i & 1;
            const int64_t s = s0 + sl;
            if (s >= num_shots) break;
            const uint32_t* o = tout + sl * 9 + 4 * half;
            reinterpret_cast<uint4*>(out + s * pitch + b0)[half] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    } else {
        for (int sl = warp; sl < 32 * W; sl += 8) {
            const int64_t s = s0 + sl;
            if (s >= num_shots) break;
            if (lane < span) out[s * pitch + b0 + lane] = (uint8_t)(tout[sl * 9 + (lane >> 2)] >> ((lane & 3) * 8));
        }
    }
}

template <bool WM>
static cudaError_t tiles_to_b8_t(const uint32_t* tiles, int64_t num_rows, int W, int64_t n_tiles,
                                 int64_t num_shots, const uint8_t* xor_bits, uint8_t* out,
                                 int64_t pitch, cudaStream_t stream) {
    if (num_rows <= 0 || num_shots <= 0 || n_tiles <= 0) return cudaSuccess;
    const int64_t parts = W > 16 ? W / 16 : 1;
    const int64_t nblk = n_tiles * parts * ((num_rows + 255) / 256);
    if (nblk > 0x7FFFFFFFll) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)nblk);
    switch (W) {
        case 1: tiles_to_b8_kernel<1, 1, WM><<<grid, 256, 0, stream>>>(tiles, num_rows, num_shots, xor_bits, out, pitch); break;
        case 2: tiles_to_b8_kernel<2, 2, WM><<<grid, 256, 0, stream>>>(tiles, num_rows, num_shots, xor_bits, out, pitch); break;
        case 4: tiles_to_b8_kernel<4, 4, WM><<<grid, 256, 0, stream>>>(tiles, num_rows, num_shots, xor_bits, out, pitch); break;
        case 8: tiles_to_b8_kernel<8, 8, WM><<<grid, 256, 0, stream>>>(tiles, num_rows, num_shots, xor_bits, out, pitch); break;
        case 16: tiles_to_b8_kernel<16, 16, WM><<<grid, 256, 0, stream>>>(tiles, num_rows, num_shots, xor_bits, out, pitch); break;
        case 32: tiles_to_b8_kernel<32, 16, WM><<<grid, 256, 0, stream>>>(tiles, num_rows, num_shots, xor_bits, out, pitch); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
cudaError_t launch_tiles_to_b8(const uint32_t* tiles, int64_t num_rows, int W, int64_t n_tiles,
                               int64_t num_shots, const uint8_t* xor_bits, uint8_t* out,
                               int64_t pitch, cudaStream_t stream, bool word_major) {
    return word_major ? tiles_to_b8_t<true>(tiles, num_rows, W, n_tiles, num_shots, xor_bits, out, pitch, stream)
                      : tiles_to_b8_t<false>(tiles, num_rows, W, n_tiles, num_shots, xor_bits, out, pitch, stream);
}

// ------------------------------------------------------------ detector_events
// Shot-major b8 (any pitch) -> row-major rows [R][row_words]: the inverse of
// rows_to_b8.  Tile: 256 rows (32 bytes per shot) x 256 shots.
__global__ void __launch_bounds__(256) b8_to_rows_kernel(const uint8_t* __restrict__ in,
                                                         int64_t in_pitch, int64_t num_rows,
                                                         int64_t num_shots, uint32_t* __restrict__ rows,
                                                         int64_t row_words) {
    __shared__ uint32_t sin[256][9];   // [shot][byte-word]
    __shared__ uint32_t sout[256][9];  // [row][shot-word]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int64_t s0 = (int64_t)blockIdx.x * 256;
    const int64_t r0 = (int64_t)blockIdx.y * 256;
    const int64_t nbytes = (num_rows + 7) >> 3;
    const int64_t b0 = r0 >> 3;
    for (int sl = warp; sl < 256; sl += 8) {  // one warp per shot: 32 consecutive bytes
        const int64_t s = s0 + sl;
        uint32_t b = 0u;
        if (s < num_shots && b0 + lane < nbytes) b = __ldg(in + s * in_pitch + b0 + lane);
        // pack 4 bytes per word with shuffles
        const uint32_t b1 = __shfl_down_sync(0xFFFFFFFFu, b, 1);
        const uint32_t b2 = __shfl_down_sync(0xFFFFFFFFu, b, 2);
        const uint32_t b3 = __shfl_down_sync(0xFFFFFFFFu, b, 3);
        if ((lane & 3) == 0) sin[sl][lane >> 2] = b | (b1 << 8) | (b2 << 16) | (b3 << 24);
    }
    __syncthreads();
    for (int pair = warp; pair < 64; pair += 8) {  // (row block rb, shot word w)
        const int rb = pair >> 3, w = pair & 7;
        uint32_t v = sin[w * 32 + lane][rb];   // lane = shot, bits = rows rb*32..
        v = transpose32_lane(v, lane);         // lane = row, bits = shots w*32..
        sout[rb * 32 + lane][w] = v;
    }
    __syncthreads();
    const int64_t r = r0 + t;
    if (r < num_rows) {
        const int64_t w0 = s0 >> 5;
        for (int w = 0; w < 8; w++)
            if (w0 + w < row_words) rows[r * row_words + w0 + w] = sout[t][w];
    }
}

// events[d][w] = XOR over e in [ptr[d], ptr[d+1]) of rows[idx[e]][w]
__global__ void rows_xor_kernel(const uint32_t* __restrict__ rows, int64_t row_words,
                                const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                                int64_t num_dets, uint32_t* __restrict__ ev) {
    const int64_t d = blockIdx.y;
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= num_dets || w >= row_words) return;
    uint32_t acc = 0u;
    for (int64_t e = __ldg(ptr + d); e < __ldg(ptr + d + 1); e++) acc ^= __ldg(rows + __ldg(idx + e) * row_words + w);
    ev[d * row_words + w] = acc;
}

cudaError_t launch_detector_events(const uint8_t* flips, int64_t in_pitch, int64_t num_shots,
                                   int64_t num_results, const int64_t* ptr, const int64_t* idx,
                                   int64_t num_dets, uint32_t* rows, uint32_t* ev, uint8_t* out,
                                   int64_t out_pitch, cudaStream_t st) {
    const int64_t words = (num_shots + 31) / 32;
    if (num_results > 0) {
        dim3 g1((unsigned)((num_shots + 255) / 256), (unsigned)((num_results + 255) / 256));
        b8_to_rows_kernel<<<g1, 256, 0, st>>>(flips, in_pitch, num_results, num_shots, rows, words);
    }
    dim3 g2((unsigned)((words + 255) / 256), (unsigned)num_dets);
    rows_xor_kernel<<<g2, 256, 0, st>>>(rows, words, ptr, idx, num_dets, ev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_rows_to_b8(ev, num_dets, words, num_shots, nullptr, out, out_pitch, st);
}

// ------------------------------------------------------------ SMEM roofline probe
// Every thread streams LDS.128 x4 + STS.128 x2 per iteration over a 64 KB
// buffer with conflict-free addressing (the CX access mix); bytes moved =
// (loads + stores) x 16 B.
__global__ void __launch_bounds__(1024) smem_probe_kernel(int iters, uint32_t* sink) {
    extern __shared__ __align__(16) uint4 sbuf[];
    const int n = 4096;  // 64 KB of uint4
    const int t = threadIdx.x;
    for (int i = t; i < n; i += blockDim.x) sbuf[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    uint4 acc = make_uint4(0, 0, 0, 0);
    int base = t;
    for (int it = 0; it < iters; it++) {
        const int a0 = (base) & (n - 1), a1 = (base + 1024) & (n - 1);
        const int a2 = (base + 2048) & (n - 1), a3 = (base + 3072) & (n - 1);
        uint4 x0 = sbuf[a0], x1 = sbuf[a1], z0 = sbuf[a2], z1 = sbuf[a3];
        x1.x ^= x0.x; x1.y ^= x0.y; x1.z ^= x0.z; x1.w ^= x0.w;
        z0.x ^= z1.x; z0.y ^= z1.y; z0.z ^= z1.z; z0.w ^= z1.w;
        sbuf[a1] = x1;
        sbuf[a2] = z0;
        acc.x ^= x1.x; acc.y ^= z0.y;
        base += blockDim.x;
    }
    if ((acc.x ^ acc.y) == 0x12345678u) sink[0] = acc.x;
}

cudaError_t smem_probe(int device, double* gbs) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return e;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    uint32_t* sink = nullptr;
    if ((e = cudaMalloc(&sink, 4)) != cudaSuccess) return e;
    const int threads = 1024, iters = 4096;
    const int grid = sms * 2;
    const size_t sm = 64 * 1024;
    cudaFuncSetAttribute(smem_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    smem_probe_kernel<<<grid, threads, sm>>>(iters, sink);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(a);
        smem_probe_kernel<<<grid, threads, sm>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const double bytes = (double)grid * threads * iters * 6.0 * 16.0;
    *gbs = bytes / (best * 1e-3) / 1e9;
    return e;
}

cudaError_t launch_rows_to_b8(const uint32_t* rows, int64_t num_rows, int64_t row_words,
                              int64_t num_shots, const uint8_t* xor_bits, uint8_t* out,
                              int64_t pitch, cudaStream_t stream) {
    if (num_rows <= 0 || num_shots <= 0) return cudaSuccess;
    const int64_t used_words = (num_shots + 31) / 32;
    dim3 grid((unsigned)((used_words + TR_WORDS - 1) / TR_WORDS),
              (unsigned)((num_rows + TR_ROWS - 1) / TR_ROWS));
    if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
    rows_to_b8_kernel<<<grid, 256, 0, stream>>>(rows, num_rows, row_words, num_shots, xor_bits,
                                                out, pitch);
    return cudaGetLastError();
}

}  // namespace pfs
