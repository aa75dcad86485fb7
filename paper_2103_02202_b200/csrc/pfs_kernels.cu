// sm_100a kernels of the bulk Pauli-frame sampler.
//
// frame_kernel  — persistent program interpreter.  Each CTA owns a tile of
//                 T = 32 W shots and keeps the whole frame table of that tile
//                 (x and z bit-planes, qubit-major, shots packed in uint32
//                 words: SURVEY.md Appendix D) resident in shared memory for the
//                 entire circuit.  Reference semantics per op:
//                   gate rules      stabsim/frame_sim.py:64-72 (gates.py:326-348)
//                   M / R / MR      stabsim/frame_sim.py:74-90
//                   noise           stabsim/frame_sim.py:92-167, entropy.py:65-88
//                   detectors       stabsim/io_formats.py:208-227
// rows_to_b8    — 32x32 warp-shuffle bit transpose of row-major bit tables to
//                 shot-major b8 (stabsim/bitvec.py:193-209, io_formats.py:94-96).
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

// global-memory loads through the read-only path for immutable inputs
template <int V> __device__ __forceinline__ VW<V> vldg(const uint32_t* p);
template <> __device__ __forceinline__ VW<4> vldg<4>(const uint32_t* p) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p)); return VW<4>{{v.x, v.y, v.z, v.w}};
}
template <> __device__ __forceinline__ VW<2> vldg<2>(const uint32_t* p) {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p)); return VW<2>{{v.x, v.y}};
}
template <> __device__ __forceinline__ VW<1> vldg<1>(const uint32_t* p) { return VW<1>{{__ldg(p)}}; }

// words c*V .. c*V+V-1 of the four rows of coin group k (V Philox blocks)
template <int W, int V>
__device__ __forceinline__ void coin_group_vec(const KParams& kp, uint32_t k, int c, uint32_t g, int64_t tile,
                                               uint32_t lo, uint32_t hi, VW<V> o[4]) {
#pragma unroll
    for (int j = 0; j < V; j++) {
        uint32_t b[4];
        coin_group<W>(kp, k, (uint32_t)(c * V + j), g, tile, lo, hi, b);
#pragma unroll
        for (int r = 0; r < 4; r++) o[r].w[j] = b[r];
    }
}

template <int C> struct Log2;
template <> struct Log2<1> { static constexpr int v = 0; };
template <> struct Log2<2> { static constexpr int v = 1; };
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };

// XOR one sampled Pauli (pattern pick) into the frame of app `app`, shot s.
template <int W>
__device__ __forceinline__ void apply_hit(uint32_t* X, uint32_t* Z, const uint32_t* tg, uint32_t ch,
                                          int ar, uint32_t trial, uint32_t pick) {
    constexpr uint32_t T = 32 * W;
    const uint32_t app = trial / T, s = trial % T;
    uint32_t xm, zm;
    pattern_of(ch, pick, xm, zm);
    const uint32_t bit = 1u << (s & 31);
    const uint32_t w = s >> 5;
    for (int sl = 0; sl < ar; sl++) {
        const size_t row = (size_t)__ldg(tg + app * ar + sl) * W + w;
        if ((xm >> sl) & 1u) atomicXor(X + row, bit);
        if ((zm >> sl) & 1u) atomicXor(Z + row, bit);
    }
}

// Pre-generated hit entry (u64): q0 (20 bits) | q1 (20) | word (5) | bit (5) |
// x mask (2) | z mask (2).  Resolved to frame rows by the producer warps, so
// applying a hit is just one or two shared-memory atomics.
__device__ __forceinline__ uint64_t make_hit(uint32_t q0, uint32_t q1, uint32_t w, uint32_t bit,
                                             uint32_t xm, uint32_t zm) {
    return (uint64_t)q0 | ((uint64_t)q1 << 20) | ((uint64_t)w << 40) | ((uint64_t)bit << 45) |
           ((uint64_t)xm << 50) | ((uint64_t)zm << 52);
}

template <int W>
__device__ __forceinline__ void apply_entry(uint32_t* X, uint32_t* Z, uint64_t e, bool plain = false) {
    const uint32_t q0 = (uint32_t)e & 0xFFFFFu, q1 = (uint32_t)(e >> 20) & 0xFFFFFu;
    const uint32_t w = (uint32_t)(e >> 40) & 31u, bit = 1u << ((uint32_t)(e >> 45) & 31u);
    const uint32_t xm = (uint32_t)(e >> 50) & 3u, zm = (uint32_t)(e >> 52) & 3u;
    if (plain) {  // profiling ablation only (racy)
        if (xm & 1u) X[(size_t)q0 * W + w] ^= bit;
        if (zm & 1u) Z[(size_t)q0 * W + w] ^= bit;
        if (xm & 2u) X[(size_t)q1 * W + w] ^= bit;
        if (zm & 2u) Z[(size_t)q1 * W + w] ^= bit;
        return;
    }
    if (xm & 1u) atomicXor(X + (size_t)q0 * W + w, bit);
    if (zm & 1u) atomicXor(Z + (size_t)q0 * W + w, bit);
    if (xm & 2u) atomicXor(X + (size_t)q1 * W + w, bit);
    if (zm & 2u) atomicXor(Z + (size_t)q1 * W + w, bit);
}

// Sample the pre-generated noise ops of global tile g into hit lists.
// Data-parallel per warp: a work item is 32 consecutive chunks of one op (lane
// l owns chunk 32*item + l).  (1) every lane draws its chunk's Philox block 0
// (count + first hit), converged; (2) the item's hits are compacted across the
// warp and each lane produces one hit per round: its pair, position, pick,
// target rows and hit-list entry (one atomic per item reserves the slots);
// (3) duplicate positions inside a chunk are detected afterwards and, rarely,
// redrawn serially.  The draws equal noise_chunk's; virtual
// trials past the op's end become no-op entries.
template <int W>
__device__ __forceinline__ uint64_t hit_entry(const uint32_t* tg, int ar, uint32_t ch, uint32_t trial,
                                              uint32_t pick, bool real) {
    constexpr uint32_t T = 32 * W;
    if (!real) return 0ull;  // xm = zm = 0: applies nothing
    const uint32_t app = trial / T, s = trial % T;
    uint32_t xm, zm;
    pattern_of(ch, pick, xm, zm);
    const uint32_t q0 = __ldg(tg + app * ar);
    const uint32_t q1 = ar == 2 ? __ldg(tg + app * ar + 1) : 0u;
    return make_hit(q0, q1, s >> 5, s & 31, xm, zm);
}

template <int W>
__device__ __forceinline__ void noise_prepass(const KParams& kp, uint32_t g, uint32_t* ncnt,
                                              uint64_t* hits, int item_begin, int item_end,
                                              uint32_t* wscr) {
    const int lane = threadIdx.x & 31;
    int k = -1;
    uint32_t ord = 0, item_base = 0, next_base = 0, ch = 0;
    NoiseParam np{};
    unsigned long long t0 = 0, t1 = 0;
    const uint32_t* tg = nullptr;
    int ar = 1;
    if (item_begin < item_end) {  // first op: binary search on item bases
        int lo = 0, hi = kp.num_pregen - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int)__ldg(&kp.noise[__ldg(kp.pregen_ops + mid)].chunk_base) <= item_begin) lo = mid;
            else hi = mid - 1;
        }
        k = lo - 1;
    }
    for (int item = item_begin; item < item_end; item++) {
        while (next_base == 0 || (uint32_t)item >= next_base) {  // op cursor (monotone)
            k++;
            ord = __ldg(kp.pregen_ops + k);
            np = kp.noise[ord];
            item_base = np.chunk_base;
            next_base = item_base + ((np.nchunks + 31u) >> 5);
            ch = __ldg(&kp.noise_ch[ord]);
            ar = ch == CH_DEP2 ? 2 : 1;
            tg = kp.targets + __ldg(&kp.noise_off[ord]);
            const unsigned long long* tab = reinterpret_cast<const unsigned long long*>(kp.noise_tab) + np.tab_full;
            t0 = np.len_full > 0 ? __ldg(tab) : ~0ull;
            t1 = np.len_full > 1 ? __ldg(tab + 1) : ~0ull;
        }
        const uint32_t L = np.L;
        const uint32_t lg = 31u - __clz(L);
        const uint32_t sh = 32u - lg;
        const uint32_t r0 = ((uint32_t)item - item_base) * 32u;
        const uint32_t r = r0 + (uint32_t)lane;
        const bool valid = r < np.nchunks;
        uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0, count = 0;
        if (valid) {
            noise_block(0u, r, g, ord, kp.seed, w0, w1, w2, w3);
            const unsigned long long u = ((unsigned long long)w1 << 32) | w0;
            if (u >= t0) {
                count = 1;
                if (u >= t1) {
                    count = 2;
                    const unsigned long long* tab =
                        reinterpret_cast<const unsigned long long*>(kp.noise_tab) + np.tab_full;
                    while (count < np.len_full && u >= __ldg(tab + count)) count++;
                }
            }
        }
        const bool big = count > (uint32_t)NZ_MAX_LIST;
        const uint32_t c = big ? 0u : count;
        uint32_t pre = c;  // inclusive prefix
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pre, d);
            if (lane >= d) pre += v;
        }
        const uint32_t H = __shfl_sync(0xFFFFFFFFu, pre, 31);
        const uint32_t excl = pre - c;
        uint32_t sbase = 0;
        if (lane == 0 && H) sbase = atomicAdd(ncnt + ord, H);
        sbase = __shfl_sync(0xFFFFFFFFu, sbase, 0);
        for (uint32_t j0 = 0; j0 < H; j0 += 32) {
            const uint32_t j = j0 + (uint32_t)lane;
            // owner chunk: smallest lane q with pre[q] > j
            uint32_t lo = 0;
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
                const uint32_t rr = r0 + owner;
                if (h > 0) {
                    uint32_t b0, b1, b2, b3;
                    noise_block((h + 1) >> 1, rr, g, ord, kp.seed, b0, b1, b2, b3);
                    x = (h & 1u) ? b0 : b2;
                    y = (h & 1u) ? b1 : b3;
                }
                const uint32_t pos = lg ? (x >> sh) : 0u;
                const uint32_t pick = np.npat > 1 ? __umulhi(y, np.npat) : 0u;
                const uint32_t vlen = (rr + 1 == np.nchunks) ? np.last_len : L;
                wscr[j] = pos;
                const uint32_t slot = sbase + j;
                if (slot < np.cap)
                    hits[np.cap_base + slot] = hit_entry<W>(tg, ar, ch, rr * L + pos, pick, pos < vlen);
            }
        }
        __syncwarp();
        // duplicate positions within a chunk (probability ~count^2 / 2L)
        bool dup = false;
        for (uint32_t h = 1; h < c; h++)
            for (uint32_t q = 0; q < h; q++) dup |= wscr[excl + h] == wscr[excl + q];
        __syncwarp();
        if (dup) {  // redraw every position of this chunk (attempts >= 1), same slots
            const uint32_t vlen = (r + 1 == np.nchunks) ? np.last_len : L;
            uint32_t sl[NZ_MAX_LIST];  // rare path: per-lane local memory
            for (uint32_t attempt = 1; dup; attempt++) {
                dup = false;
                uint32_t blk = 0xFFFFFFFFu, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
                for (uint32_t h = 0; h < c; h++) {
                    const uint32_t kk = attempt * NZ_MAX_LIST + h;
                    const uint32_t need = (kk + 1) >> 1;
                    if (need != blk) { noise_block(need, r, g, ord, kp.seed, b0, b1, b2, b3); blk = need; }
                    const uint32_t x = (kk & 1u) ? b0 : b2, y = (kk & 1u) ? b1 : b3;
                    const uint32_t pos = lg ? (x >> sh) : 0u;
                    for (uint32_t q = 0; q < h; q++) dup |= (sl[q] >> 4) == pos;
                    sl[h] = (pos << 4) | (np.npat > 1 ? __umulhi(y, np.npat) : 0u);
                }
            }
            for (uint32_t h = 0; h < c; h++) {
                const uint32_t slot = sbase + excl + h;
                const uint32_t pos = sl[h] >> 4;
                if (slot < np.cap)
                    hits[np.cap_base + slot] = hit_entry<W>(tg, ar, ch, r * L + pos, sl[h] & 15u, pos < vlen);
            }
        }
        if (big) {  // selection sampling, ~1e-6 of chunks
            const uint32_t vlen = (r + 1 == np.nchunks) ? np.last_len : L;
            uint32_t needed = count;
            for (uint32_t i = 0; needed > 0; i++) {
                noise_block(0x80000000u + i, r, g, ord, kp.seed, w0, w1, w2, w3);
                if (__umul64hi(((uint64_t)w1 << 32) | w0, (uint64_t)(L - i)) < needed) {
                    if (i < vlen) {
                        const uint32_t slot = atomicAdd(ncnt + ord, 1u);
                        if (slot < np.cap)
                            hits[np.cap_base + slot] = hit_entry<W>(tg, ar, ch, r * L + i,
                                                                    np.npat > 1 ? __umulhi(w2, np.npat) : 0u, true);
                    }
                    needed--;
                }
            }
        }
        __syncwarp();
    }
}

// Noise sampling kernel: runs before the frame kernel over every tile of the
// launch at full occupancy (no shared-memory frame), writing each tile's hit
// lists and per-op hit counts to global memory (L2-resident for a chunk).
// grid = (ceil(items / (8 * NZ_ITEMS_PER_WARP)), tiles), 256 threads.
constexpr int NZ_ITEMS_PER_WARP = 4;
#ifndef NZ_MIN_BLOCKS
#define NZ_MIN_BLOCKS 5
#endif
template <int W>
__global__ void __launch_bounds__(256, NZ_MIN_BLOCKS) noise_kernel(const __grid_constant__ KParams kp) {
    __shared__ uint32_t wscr_all[8][32 * NZ_MAX_LIST];  // 16 KB: fits beside a frame CTA
    const int warp = threadIdx.x >> 5;
    const int64_t tile = blockIdx.y;
    const uint32_t g = (uint32_t)(kp.tile_offset + (uint64_t)tile);
    const int wi = blockIdx.x * 8 + warp;
    const int b = wi * NZ_ITEMS_PER_WARP;
    const int e = min(kp.pregen_chunks, b + NZ_ITEMS_PER_WARP);
    noise_prepass<W>(kp, g, kp.ncnt_global + tile * kp.num_noise,
                     kp.hits_global + tile * kp.hit_capacity, b, e, wscr_all[warp]);
}

// Items of one op, U per thread per batch: all U operand loads (L2-resident
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

// ------------------------------------------------------------ frame kernel
// Persistent kernel: each CTA runs the op stream over its tiles with the frame
// in shared memory; noise comes pre-sampled per tile from noise_kernel (hit
// lists in global memory), applied with shared-memory atomics.
template <int W, bool RING_SMEM>
__global__ void __launch_bounds__(FRAME_MAX_THREADS, 1) frame_kernel(const __grid_constant__ KParams kp) {
    constexpr int V = W >= 4 ? 4 : W;  // words per vector access
    constexpr int C = W / V;           // vector chunks per row
    constexpr int LC = Log2<C>::v;
    extern __shared__ __align__(16) uint32_t smem[];
    const int n = kp.num_qubits;
    // kp.groups independent thread groups per CTA, each with its own tile,
    // frame, record ring and named barrier: one group's op latency overlaps
    // the other group's work
    const int G = kp.groups;
    const int gsz = blockDim.x / G;
    const int grp = threadIdx.x / gsz;
    const int tid = threadIdx.x - grp * gsz;  // thread index within the group
    const int nth = gsz;
    const size_t fw = (size_t)2 * n * W;      // frame words per group
    uint32_t* const X = smem + grp * fw;
    uint32_t* const Z = X + (size_t)n * W;
    uint32_t* const ring = RING_SMEM ? (smem + G * fw + (size_t)grp * kp.num_slots * W)
                                     : (kp.ring_global + ((size_t)blockIdx.x * G + grp) * kp.num_slots * W);
    uint32_t* const cnt = smem + G * fw + (RING_SMEM ? (size_t)G * kp.num_slots * W : 0);
    uint32_t* const ncnt0 = cnt + (kp.counts_in_smem ? kp.num_cols : 0);
    uint32_t* const ncnt = ncnt0 + grp * kp.num_noise;  // this tile's hits per op
    // 16-byte aligned tail: the op descriptors (when they fit)
    // (offset arithmetic on the shared array keeps the loads in the shared
    // address space: LDS, not generic LD)
    const size_t dsc_word = ((size_t)(ncnt0 + G * kp.num_noise - smem) + 3) & ~(size_t)3;
    uint4* const dsc_s = reinterpret_cast<uint4*>(smem + dsc_word);
    const uint4* const dsc_g = reinterpret_cast<const uint4*>(kp.ops);
    const bool dsm = kp.desc_in_smem != 0;
    auto ldesc = [&](int i) -> uint4 { return dsm ? dsc_s[i] : __ldg(dsc_g + i); };
    // per-lane scratch of the inline noise sampler (large-p ops / list overflow), global
    uint32_t* const sl = kp.noise_scratch +
                         ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    const int ss = 1;
    const bool pregen = kp.masks == nullptr && kp.num_pregen > 0 && !(kp.debug_skip & 2);
    const uint32_t bar_id = 1u + (uint32_t)grp;
    auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(gsz) : "memory"); };

    if (kp.counts_in_smem)
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x) cnt[i] = 0u;
    if (dsm)
        for (int i = threadIdx.x; i < 2 * kp.n_ops; i += blockDim.x) dsc_s[i] = __ldg(dsc_g + i);
    __syncthreads();

    for (int64_t tile = (int64_t)blockIdx.x * G + grp; tile < kp.n_tiles; tile += (int64_t)gridDim.x * G) {
        const uint32_t g = (uint32_t)(kp.tile_offset + (uint64_t)tile);
        const uint64_t* const hits = kp.hits_global + tile * kp.hit_capacity;
        {
            // ---- FrameBatch.__init__: x = 0, z = coins (frame_sim.py:36-39) ----
            for (int i = tid; i < (n << LC); i += nth) {
                const int q = i >> LC, c = i & (C - 1);
                vst<V>(X + (size_t)q * W + c * V, vzero<V>());
            }
            {  // z = coin rows 0..n-1: items = (coin group, V-word chunk)
                const int items = (int)coin_k1((uint32_t)n) << LC;
                for (int i = tid; i < items; i += nth) {
                    const uint32_t k = (uint32_t)(i >> LC);
                    const int c = i & (C - 1);
                    if (!coin_group_live(k, 0u, (uint32_t)n)) continue;
                    const uint32_t live = init_live_rows(kp, k, (uint32_t)n);
                    VW<V> o[4];
                    if (live) coin_group_vec<W, V>(kp, k, c, g, tile, 0u, (uint32_t)n, o);
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        const uint32_t e = coin_row0(k) + 32u * r;
                        if (e < (uint32_t)n)  // coin row e is qubit e's initial z (frame_sim.py:38-39)
                            vst<V>(Z + (size_t)__ldg(kp.row_of + e) * W + c * V, ((live >> r) & 1u) ? o[r] : vzero<V>());
                    }
                }
            }
            for (int i = tid; i < (kp.num_obs << LC); i += nth) {
                const int k = i >> LC, c = i & (C - 1);
                vst<V>(ring + (size_t)k * W + c * V, vzero<V>());
            }
            if (pregen)
                for (int i = tid; i < kp.num_noise; i += nth) {
                    const uint32_t c = kp.ncnt_global[tile * kp.num_noise + i];
                    const NoiseParam* np = kp.noise + i;
                    const uint32_t cap = __ldg(&np->cap);
                    ncnt[i] = c <= cap ? c : NO_SLOT;  // overflow -> inline resampling
                    // pull this op's hit list into L2 ahead of use (TMA bulk prefetch)
                    const uint32_t nb = min(c, cap) * 8u;
                    if ((__ldg(&np->flags) & NZ_PREGEN) && nb) {
                        // bulk copies need 16-byte aligned addresses and sizes
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(hits + __ldg(&np->cap_base));
                        const uintptr_t lo = a0 & ~(uintptr_t)15;
                        const uint32_t sz = (uint32_t)(((a0 + nb) - lo + 15) & ~(uintptr_t)15);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                                     ::"l"(lo), "r"(sz) : "memory");
                    }
                }
            group_sync();  // counts visible
            // the next pre-sampled noise op's first hit (one per thread) rides in
            // a register from the previous noise op on, so applying it does not
            // put an L2 round trip on the op chain
            uint64_t pf_hit = 0;
            auto prefetch_hit = [&](uint32_t ord, uint32_t base) {
                pf_hit = 0;
                if (!pregen || ord == NO_SLOT) return;
                const uint32_t nh = ncnt[ord];
                if (nh != NO_SLOT && (uint32_t)tid < nh) pf_hit = __ldcg(hits + base + tid);
            };
            prefetch_hit(kp.first_pregen, kp.first_cap_base);

            // descriptors run one op ahead in registers
            uint4 h0 = kp.n_ops > 0 ? ldesc(0) : make_uint4(0, 0, 0, 0);
            uint4 h1n = kp.n_ops > 0 ? ldesc(1) : make_uint4(0, 0, 0, 0);
            for (int oi = 0; oi < kp.n_ops; oi++) {
                const uint32_t kind = h0.x & 0xFFu, code = (h0.x >> 8) & 0xFFu, flags = h0.x >> 16;
                const uint32_t count = h0.y, off = h0.z, oa = h0.w;
                const uint4 h1 = h1n;
                if (oi + 1 < kp.n_ops) { h0 = ldesc(2 * oi + 2); h1n = ldesc(2 * oi + 3); }
                const uint32_t ob = h1.x, oc = h1.y;
                if (flags & F_BARRIER) group_sync();
#if PFS_PROFILE
                if (kp.op_clock != nullptr && blockIdx.x == 0 && grp == 0 && tid == 0 &&
                    tile == 0)  // profiling: op-boundary timestamps of the first tile
                    kp.op_clock[oi] = clock64();
#endif
                const uint32_t* const tgg = kp.targets + off;  // operands (L1/L2-resident)
                const uint32_t* const tg = tgg;
#if PFS_PROFILE
                if (kp.debug_skip) {
                    const uint32_t bit = kind == K_NOISE ? 1u : kind == K_DET ? 8u : kind == K_GATE ? 16u
                                       : (kind == K_M || kind == K_R || kind == K_MR) ? 32u : 0u;
                    if (kp.debug_skip & bit) continue;
                }
#endif
                switch (kind) {
                case K_GATE: {
                    const int items = (int)(count << LC);
                    auto q1 = [&](int i) { return tg[i >> LC]; };
                    auto q2 = [&](int i) { return reinterpret_cast<const uint2*>(tg)[i >> LC]; };
                    switch (code) {
                    case R_SWAPXZ:
                        batched_items<4>(tid, nth, items, q1, [&](int i, uint32_t q) {
                            const size_t p = (size_t)q * W + (i & (C - 1)) * V;
                            const VW<V> a = vld<V>(X + p), b = vld<V>(Z + p);
                            vst<V>(X + p, b); vst<V>(Z + p, a);
                        });
                        break;
                    case R_ZXORX:
                        batched_items<4>(tid, nth, items, q1, [&](int i, uint32_t q) {
                            const size_t p = (size_t)q * W + (i & (C - 1)) * V;
                            vst<V>(Z + p, vxor<V>(vld<V>(Z + p), vld<V>(X + p)));
                        });
                        break;
                    case R_XXORZ:
                        batched_items<4>(tid, nth, items, q1, [&](int i, uint32_t q) {
                            const size_t p = (size_t)q * W + (i & (C - 1)) * V;
                            vst<V>(X + p, vxor<V>(vld<V>(X + p), vld<V>(Z + p)));
                        });
                        break;
                    default:  // two-qubit rules
                        batched_items<4>(tid, nth, items, q2, [&](int i, uint2 qq) {
                            const int cv = (i & (C - 1)) * V;
                            const size_t p0 = (size_t)qq.x * W + cv, p1 = (size_t)qq.y * W + cv;
                            const VW<V> x0 = vld<V>(X + p0), x1 = vld<V>(X + p1);
                            const VW<V> z0 = vld<V>(Z + p0), z1 = vld<V>(Z + p1);
                            switch (code) {
                            case R_CX:
                                vst<V>(X + p1, vxor<V>(x1, x0)); vst<V>(Z + p0, vxor<V>(z0, z1)); break;
                            case R_CZ:
                                vst<V>(Z + p0, vxor<V>(z0, x1)); vst<V>(Z + p1, vxor<V>(z1, x0)); break;
                            case R_CY:
                                vst<V>(X + p1, vxor<V>(x1, x0));
                                vst<V>(Z + p0, vxor<V>(z0, vxor<V>(x1, z1)));
                                vst<V>(Z + p1, vxor<V>(z1, x0)); break;
                            default:  // SWAP
                                vst<V>(X + p0, x1); vst<V>(X + p1, x0);
                                vst<V>(Z + p0, z1); vst<V>(Z + p1, z0); break;
                            }
                        });
                    }
                    break;
                }
                case K_M: case K_MR: case K_R: {
                    // items = (coin group, V-word chunk): V Philox blocks, up to four rows
                    const uint32_t lo = ob, hi = ob + (kind == K_MR ? 2u : 1u) * count;
                    const uint32_t k0 = coin_k0(lo);
                    const int items = (int)(coin_k1(hi) - k0) << LC;
                    for (int i = tid; i < items; i += nth) {
                        const uint32_t k = k0 + (uint32_t)(i >> LC);
                        const int c = i & (C - 1);
                        if (!coin_group_live(k, lo, hi)) continue;
                        uint2 qsv[4];  // operands load while the coin blocks compute
                        const uint32_t live = collapse_rows(tg, kind, k, lo, hi, qsv);
                        VW<V> o[4];
                        if (live) coin_group_vec<W, V>(kp, k, c, g, tile, lo, hi, o);
#pragma unroll
                        for (int r = 0; r < 4; r++) {
                            const uint32_t e = coin_row0(k) + 32u * r;
                            if (e < lo || e >= hi) continue;
                            const uint32_t rel = e - lo;
                            const bool lv = (live >> r) & 1u;  // dead coin rows: z is never read
                            const size_t p = (size_t)qsv[r].x * W + c * V;
                            if (kind == K_R) {
                                vst<V>(X + p, vzero<V>());
                                vst<V>(Z + p, lv ? o[r] : vzero<V>());
                                continue;
                            }
                            if (kind == K_MR && !(rel & 1u)) continue;  // the measure's coin row is overwritten
                            const uint32_t j = kind == K_MR ? rel >> 1 : rel;
                            const VW<V> xv = vld<V>(X + p);
                            if (kp.do_dets && qsv[r].y != NO_SLOT) vst<V>(ring + (size_t)qsv[r].y * W + c * V, xv);
                            if (kp.rec_out != nullptr)
                                vst<V>(kp.rec_out + (int64_t)(oa + j) * kp.out_row_stride + tile * kp.out_tile_stride + c * V, xv);
                            if (kind == K_M) {
                                if (lv) vst<V>(Z + p, vxor<V>(vld<V>(Z + p), o[r]));
                            } else {
                                vst<V>(X + p, vzero<V>());
                                vst<V>(Z + p, lv ? o[r] : vzero<V>());
                            }
                        }
                    }
                    break;
                }
                case K_NOISE: {
                    const int ar = code == CH_DEP2 ? 2 : 1;
                    if (kp.masks != nullptr) {
                        // injected masks: per target, x row then z row
                        const int items = (int)((count * ar) << LC);
                        for (int i = tid; i < items; i += nth) {
                            const int j = i >> LC, c = i & (C - 1);
                            const size_t p = (size_t)__ldg(tgg + j) * W + c * V;
                            const uint32_t* mrow = kp.masks + (int64_t)(oa + 2 * j) * kp.inject_words + tile * W + c * V;
                            const VW<V> mx = vldg<V>(mrow), mz = vldg<V>(mrow + kp.inject_words);
                            if (flags & F_DUP) {
#pragma unroll
                                for (int k = 0; k < V; k++) {
                                    if (mx.w[k]) atomicXor(X + p + k, mx.w[k]);
                                    if (mz.w[k]) atomicXor(Z + p + k, mz.w[k]);
                                }
                            } else {
                                vst<V>(X + p, vxor<V>(vld<V>(X + p), mx));
                                vst<V>(Z + p, vxor<V>(vld<V>(Z + p), mz));
                            }
                        }
                        break;
                    }
                    if ((flags & F_PREGEN) && pregen) {
                        const uint32_t nh = ncnt[ob];  // NO_SLOT: the hit list overflowed
                        const uint64_t cur = pf_hit;
                        prefetch_hit(h1.z, h1.w);  // the next pre-sampled noise op
                        if (nh != NO_SLOT) {
                            const uint64_t* hl = hits + oc;
                            if ((uint32_t)tid < nh) apply_entry<W>(X, Z, cur);
                            for (uint32_t i = tid + nth; i < nh; i += nth) apply_entry<W>(X, Z, hl[i]);
                        } else {
                            const NoiseParam* npp = kp.noise + ob;
                            for (uint32_t r = tid; r < __ldg(&npp->nchunks); r += nth)
                                noise_chunk(kp, *npp, ob, r, g, sl, ss, [&](uint32_t trial, uint32_t pick) {
                                    apply_hit<W>(X, Z, tgg, code, ar, trial, pick);
                                });
                        }
                        break;
                    }
                    if (kp.debug_skip & 2) break;
                    const NoiseParam np = kp.noise[ob];
                    if (np.flags & NZ_NONE) break;
                    // inline sampling (large-p ops)
                    for (uint32_t r = tid; r < np.nchunks; r += nth)
                        noise_chunk(kp, np, ob, r, g, sl, ss, [&](uint32_t trial, uint32_t pick) {
                            apply_hit<W>(X, Z, tgg, code, ar, trial, pick);
                        });
                    break;
                }
                case K_DET: {
                    if (!kp.do_dets) break;
                    const int items = (int)(count << LC);
                    // prefetch each column's term range and first two record slots;
                    // uniform ops (code = terms per column) address terms directly
                    batched_items<2>(tid, nth, items,
                        [&](int i) {
                            const uint32_t ci = (uint32_t)(i >> LC);
                            const uint32_t col = oa + ci;
                            uint32_t e0, e1;
                            if (code) { e0 = off + ci * code; e1 = e0 + code; }
                            else { e0 = __ldg(kp.det_ptr + col); e1 = __ldg(kp.det_ptr + col + 1); }
                            const uint32_t* tb = kp.det_terms;
                            const uint32_t s0 = e0 < e1 ? tb[e0] : NO_SLOT;
                            const uint32_t s1 = e0 + 1 < e1 ? tb[e0 + 1] : NO_SLOT;
                            return make_uint4(e0, e1, s0, s1);
                        },
                        [&](int i, uint4 d) {
                            const uint32_t col = oa + (uint32_t)(i >> LC);
                            const int c = i & (C - 1);
                            VW<V> acc = vzero<V>();
                            if (d.z != NO_SLOT) acc = vld<V>(ring + (size_t)d.z * W + c * V);
                            if (d.w != NO_SLOT) acc = vxor<V>(acc, vld<V>(ring + (size_t)d.w * W + c * V));
                            const uint32_t* tb = kp.det_terms;
                            for (uint32_t e = d.x + 2; e < d.y; e++) {
                                const uint32_t s = tb[e];
                                acc = vxor<V>(acc, vld<V>(ring + (size_t)s * W + c * V));
                            }
                            if (kp.ev_out != nullptr)
                                vst<V>(kp.ev_out + (int64_t)col * kp.out_row_stride +
                                           tile * kp.out_tile_stride + c * V, acc);
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
                    if (!kp.do_dets) break;
                    for (int c = tid; c < C; c += nth) {
                        VW<V> acc = vld<V>(ring + (size_t)oa * W + c * V);
                        for (uint32_t j = 0; j < count; j++) {
                            const uint32_t s = tg[j];
                            acc = vxor<V>(acc, vld<V>(ring + (size_t)s * W + c * V));
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
        }
        group_sync();  // the group's frame is reused by its next tile
    }
    if (kp.counts_in_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x)
            if (cnt[i]) atomicAdd(kp.counts + i, (unsigned long long)cnt[i]);
    }
}

// ------------------------------------------------------- warp-private kernel
// Each warp owns one 32-shot word column (word w of tile t) for the whole
// circuit: its frame is x/z interleaved per qubit (uint2 XZ[q], 8 bytes) plus
// its record ring, all in shared memory.  Lanes take the applications of an op
// (at most one per qubit, so lanes never collide) and warps never wait for
// each other: no CTA barriers, only __syncwarp between ops.  The CTA's warps
// run the same op stream on different words, so operand loads (targets,
// detector terms, hit lists) hit L1 for all but the leading warp.
template <int W>
__device__ __forceinline__ void warp_apply_entry(uint32_t* xz, uint64_t e, uint32_t w) {
    if (((uint32_t)(e >> 40) & 31u) != w) return;
    const uint32_t q0 = (uint32_t)e & 0xFFFFFu, q1 = (uint32_t)(e >> 20) & 0xFFFFFu;
    const uint32_t bit = 1u << ((uint32_t)(e >> 45) & 31u);
    const uint32_t xm = (uint32_t)(e >> 50) & 3u, zm = (uint32_t)(e >> 52) & 3u;
    if (xm & 1u) atomicXor(xz + 2 * q0, bit);
    if (zm & 1u) atomicXor(xz + 2 * q0 + 1, bit);
    if (xm & 2u) atomicXor(xz + 2 * q1, bit);
    if (zm & 2u) atomicXor(xz + 2 * q1 + 1, bit);
}

template <int W>
__global__ void __launch_bounds__(WARP_KERNEL_MAX_THREADS, 1) frame_warp_kernel(const __grid_constant__ KParams kp) {
    constexpr uint32_t T = 32 * W;
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int n = kp.num_qubits;
    const size_t dwords = kp.desc_in_smem ? (size_t)kp.n_ops * 8 : 0;
    const size_t per_warp = ((size_t)2 * n + kp.num_slots + kp.num_noise + 1) & ~(size_t)1;
    uint32_t* const xz = smem + dwords + (size_t)warp * per_warp;  // x = xz[2q], z = xz[2q+1]
    uint2* const XZ = reinterpret_cast<uint2*>(xz);
    uint32_t* const ring = xz + 2 * n;
    uint32_t* const ncnt = ring + kp.num_slots;
    const uint4* const dsc = kp.desc_in_smem ? reinterpret_cast<const uint4*>(smem)
                                             : reinterpret_cast<const uint4*>(kp.ops);
    uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    const bool pregen = kp.masks == nullptr && kp.num_pregen > 0 && !(kp.debug_skip & 2);
    if (kp.desc_in_smem) {
        uint4* d = reinterpret_cast<uint4*>(smem);
        for (int i = threadIdx.x; i < 2 * kp.n_ops; i += blockDim.x)
            d[i] = __ldg(reinterpret_cast<const uint4*>(kp.ops) + i);
        __syncthreads();
    }
    const int64_t units = kp.n_tiles * W;
    for (int64_t u = (int64_t)blockIdx.x * NW + warp; u < units; u += (int64_t)gridDim.x * NW) {
        const int64_t tile = u / W;
        const uint32_t w = (uint32_t)(u % W);
        if (tile * T + 32 * (int64_t)w >= kp.num_shots) continue;  // no live shot in this word
        const uint32_t g = (uint32_t)(kp.tile_offset + (uint64_t)tile);
        const uint64_t* const hits = kp.hits_global + tile * kp.hit_capacity;
        const int64_t obase = tile * kp.out_tile_stride + (int64_t)w * kp.out_word_stride;
        // ---- FrameBatch.__init__: x = 0, z = coin rows 0..n-1 (frame_sim.py:36-39) ----
        for (uint32_t k = (uint32_t)lane; k < coin_k1((uint32_t)n); k += 32) {
            const uint32_t live = init_live_rows(kp, k, (uint32_t)n);
            uint32_t o[4] = {0u, 0u, 0u, 0u};
            if (live) coin_group<W>(kp, k, w, g, tile, 0u, (uint32_t)n, o);
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const uint32_t e = coin_row0(k) + 32u * r;
                if (e < (uint32_t)n) XZ[__ldg(kp.row_of + e)] = make_uint2(0u, ((live >> r) & 1u) ? o[r] : 0u);
            }
        }
        for (int i = lane; i < kp.num_obs; i += 32) ring[i] = 0u;
        if (pregen)
            for (int i = lane; i < kp.num_noise; i += 32) {
                const uint32_t c = kp.ncnt_global[tile * kp.num_noise + i];
                ncnt[i] = c <= __ldg(&kp.noise[i].cap) ? c : NO_SLOT;  // overflow -> inline resampling
            }
        __syncwarp();
        // the next pre-generated noise op's first 32*NZ_PF hits ride in
        // registers from the previous noise op on, so a noise op never waits
        // for its hit list
        constexpr int NZ_PF = 4;
        uint64_t pf[NZ_PF];
        auto prefetch_hits = [&](uint32_t ord, uint32_t base) {
            uint32_t nh = ord != NO_SLOT && pregen ? ncnt[ord] : 0u;
            if (nh == NO_SLOT) nh = 0u;
#pragma unroll
            for (int t = 0; t < NZ_PF; t++) {
                const uint32_t i = (uint32_t)lane + 32u * t;
                pf[t] = i < nh ? __ldg(hits + base + i) : 0ull;
            }
        };
        prefetch_hits(kp.first_pregen, kp.first_cap_base);
        for (int oi = 0; oi < kp.n_ops; oi++) {
            const uint4 h0 = dsc[2 * oi], h1 = dsc[2 * oi + 1];
            const uint32_t kind = h0.x & 0xFFu, code = (h0.x >> 8) & 0xFFu, flags = h0.x >> 16;
            const uint32_t count = h0.y, off = h0.z, oa = h0.w, ob = h1.x, oc = h1.y;
            const uint32_t* const tg = kp.targets + off;
#if PFS_PROFILE
            if (kp.debug_skip) {
                const uint32_t bit = kind == K_NOISE ? 1u : kind == K_DET ? 8u : kind == K_GATE ? 16u
                                   : (kind == K_M || kind == K_R || kind == K_MR) ? 32u : 0u;
                if (kp.debug_skip & bit) continue;
            }
            if (kp.op_clock != nullptr && blockIdx.x == 0 && warp == 0 && lane == 0 && u == 0)
                kp.op_clock[oi] = clock64();
#endif
            switch (kind) {
            case K_GATE: {
                // U applications per lane in flight: all operand and frame loads
                // before any store (an op's applications touch distinct qubits)
                constexpr int U = 4;
                if (code <= R_XXORZ) {
                    for (uint32_t i0 = lane; i0 < count; i0 += 32 * U) {
                        uint32_t q[U];
                        uint2 v[U];
#pragma unroll
                        for (int t = 0; t < U; t++) {
                            const uint32_t i = i0 + 32u * t;
                            q[t] = i < count ? __ldg(tg + i) : 0u;
                        }
#pragma unroll
                        for (int t = 0; t < U; t++)
                            if (i0 + 32u * t < count) v[t] = XZ[q[t]];
#pragma unroll
                        for (int t = 0; t < U; t++) {
                            if (i0 + 32u * t >= count) continue;
                            uint2 a = v[t];
                            if (code == R_SWAPXZ) a = make_uint2(a.y, a.x);
                            else if (code == R_ZXORX) a.y ^= a.x;
                            else a.x ^= a.y;
                            XZ[q[t]] = a;
                        }
                    }
                } else {
                    const uint2* tg2 = reinterpret_cast<const uint2*>(tg);
                    for (uint32_t i0 = lane; i0 < count; i0 += 32 * U) {
                        uint2 qq[U], va[U], vb[U];
#pragma unroll
                        for (int t = 0; t < U; t++) {
                            const uint32_t i = i0 + 32u * t;
                            qq[t] = i < count ? __ldg(tg2 + i) : make_uint2(0u, 0u);
                        }
#pragma unroll
                        for (int t = 0; t < U; t++)
                            if (i0 + 32u * t < count) { va[t] = XZ[qq[t].x]; vb[t] = XZ[qq[t].y]; }
#pragma unroll
                        for (int t = 0; t < U; t++) {
                            if (i0 + 32u * t >= count) continue;
                            uint2 a = va[t], b = vb[t];
                            switch (code) {
                            case R_CX: b.x ^= a.x; a.y ^= b.y; break;
                            case R_CZ: { const uint32_t az = a.y ^ b.x, bz = b.y ^ a.x; a.y = az; b.y = bz; break; }
                            case R_CY: { const uint32_t az = a.y ^ b.x ^ b.y, bz = b.y ^ a.x;
                                         b.x ^= a.x; a.y = az; b.y = bz; break; }
                            default: { const uint2 t2 = a; a = b; b = t2; break; }  // SWAP
                            }
                            XZ[qq[t].x] = a;
                            XZ[qq[t].y] = b;
                        }
                    }
                }
                break;
            }
            case K_M: case K_MR: case K_R: {
                const uint32_t lo = ob, hi = ob + (kind == K_MR ? 2u : 1u) * count;
                for (uint32_t k = coin_k0(lo) + lane; k < coin_k1(hi); k += 32) {
                    if (!coin_group_live(k, lo, hi)) continue;
                    // the four rows' operands load while the coin block computes
                    uint2 qsv[4];
                    const uint32_t live = collapse_rows(tg, kind, k, lo, hi, qsv);
                    uint32_t o[4] = {0u, 0u, 0u, 0u};
                    if (live) coin_group<W>(kp, k, w, g, tile, lo, hi, o);
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        const uint32_t e = coin_row0(k) + 32u * r;
                        if (e < lo || e >= hi) continue;
                        const uint32_t rel = e - lo;
                        const uint32_t cv = ((live >> r) & 1u) ? o[r] : 0u;  // dead rows: z never read
                        if (kind == K_R) { XZ[qsv[r].x] = make_uint2(0u, cv); continue; }
                        if (kind == K_MR && !(rel & 1u)) continue;  // the measure's coin row is overwritten
                        const uint32_t j = kind == K_MR ? rel >> 1 : rel;
                        const uint2 qs = qsv[r];
                        const uint32_t xv = xz[2 * qs.x];
                        if (kp.do_dets && qs.y != NO_SLOT) ring[qs.y] = xv;
                        if (kp.rec_out != nullptr) kp.rec_out[obase + (int64_t)(oa + j) * kp.out_row_stride] = xv;
                        if (kind == K_M) xz[2 * qs.x + 1] ^= cv;
                        else XZ[qs.x] = make_uint2(0u, cv);
                    }
                }
                break;
            }
            case K_NOISE: {
                const int ar = code == CH_DEP2 ? 2 : 1;
                if (kp.masks != nullptr) {
                    // injected masks: per target, x row then z row
                    for (uint32_t j = lane; j < count * ar; j += 32) {
                        const uint32_t q = __ldg(tg + j);
                        const uint32_t* mrow = kp.masks + (int64_t)(oa + 2 * j) * kp.inject_words + tile * W + w;
                        const uint32_t mx = __ldg(mrow), mz = __ldg(mrow + kp.inject_words);
                        if (flags & F_DUP) {
                            if (mx) atomicXor(xz + 2 * q, mx);
                            if (mz) atomicXor(xz + 2 * q + 1, mz);
                        } else {
                            uint2 v = XZ[q];
                            v.x ^= mx; v.y ^= mz;
                            XZ[q] = v;
                        }
                    }
                    break;
                }
                if ((flags & F_PREGEN) && pregen) {
                    const uint32_t nh = ncnt[ob];
                    uint64_t cur[NZ_PF];
#pragma unroll
                    for (int t = 0; t < NZ_PF; t++) cur[t] = pf[t];
                    prefetch_hits(h1.z, h1.w);  // the next noise op's hits
                    if (nh != NO_SLOT) {
#pragma unroll
                        for (int t = 0; t < NZ_PF; t++) warp_apply_entry<W>(xz, cur[t], w);
                        const uint64_t* hl = hits + oc;
                        constexpr int U = 4;
                        for (uint32_t i0 = lane + 32 * NZ_PF; i0 < nh; i0 += 32 * U) {
                            uint64_t ent[U];
#pragma unroll
                            for (int t = 0; t < U; t++) {
                                const uint32_t i = i0 + 32u * t;
                                ent[t] = i < nh ? __ldg(hl + i) : 0ull;
                            }
#pragma unroll
                            for (int t = 0; t < U; t++) warp_apply_entry<W>(xz, ent[t], w);
                        }
                        break;
                    }
                } else if (kp.debug_skip & 2) {
                    break;
                }
                // inline sampling (large-p ops, hit-list overflow): this warp draws
                // every chunk of the tile and keeps the hits in its word
                const NoiseParam np = kp.noise[ob];
                if (np.flags & NZ_NONE) break;
                for (uint32_t r = lane; r < np.nchunks; r += 32)
                    noise_chunk(kp, np, ob, r, g, sl, 1, [&](uint32_t trial, uint32_t pick) {
                        const uint32_t app = trial / T, s = trial % T;
                        if ((s >> 5) != w) return;
                        uint32_t xm, zm;
                        pattern_of(code, pick, xm, zm);
                        const uint32_t bit = 1u << (s & 31);
                        for (int a = 0; a < ar; a++) {
                            const uint32_t q = __ldg(tg + app * ar + a);
                            if ((xm >> a) & 1u) atomicXor(xz + 2 * q, bit);
                            if ((zm >> a) & 1u) atomicXor(xz + 2 * q + 1, bit);
                        }
                    });
                break;
            }
            case K_DET: {
                if (!kp.do_dets) break;
                auto det_word = [&](uint32_t col, uint32_t acc) {
                    if (kp.ev_out != nullptr) kp.ev_out[obase + (int64_t)col * kp.out_row_stride] = acc;
                    if (kp.counts != nullptr) {
                        const int64_t rem = kp.num_shots - (tile * (int64_t)T + 32 * (int64_t)w);
                        const uint32_t m = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
                        const uint32_t tot = __popc(acc & m);
                        if (tot) atomicAdd(kp.counts + col, (unsigned long long)tot);
                    }
                };
                if (code == 2) {  // the common two-term detector: 4 columns per lane in flight
                    constexpr int U = 4;
                    for (uint32_t i0 = lane; i0 < count; i0 += 32 * U) {
                        uint32_t s0[U], s1[U];
#pragma unroll
                        for (int t = 0; t < U; t++) {
                            const uint32_t i = i0 + 32u * t;
                            s0[t] = i < count ? __ldg(kp.det_terms + off + 2 * i) : NO_SLOT;
                            s1[t] = i < count ? __ldg(kp.det_terms + off + 2 * i + 1) : NO_SLOT;
                        }
#pragma unroll
                        for (int t = 0; t < U; t++) {
                            const uint32_t i = i0 + 32u * t;
                            if (i >= count) continue;
                            const uint32_t acc = (s0[t] != NO_SLOT ? ring[s0[t]] : 0u) ^
                                                 (s1[t] != NO_SLOT ? ring[s1[t]] : 0u);
                            det_word(oa + i, acc);
                        }
                    }
                    break;
                }
                for (uint32_t i = lane; i < count; i += 32) {
                    const uint32_t col = oa + i;
                    uint32_t e0, e1;
                    if (code) { e0 = off + i * code; e1 = e0 + code; }
                    else { e0 = __ldg(kp.det_ptr + col); e1 = __ldg(kp.det_ptr + col + 1); }
                    uint32_t acc = 0u;
                    for (uint32_t e = e0; e < e1; e++) {
                        const uint32_t sidx = __ldg(kp.det_terms + e);
                        if (sidx != NO_SLOT) acc ^= ring[sidx];
                    }
                    det_word(col, acc);
                }
                break;
            }
            case K_OBS: {
                if (!kp.do_dets) break;
                uint32_t acc = 0u;
                for (uint32_t j = lane; j < count; j += 32) {
                    const uint32_t sidx = __ldg(tg + j);
                    if (sidx != NO_SLOT) acc ^= ring[sidx];
                }
                acc = __reduce_xor_sync(0xFFFFFFFFu, acc);
                if (lane == 0) ring[oa] ^= acc;
                break;
            }
            default: break;
            }
            __syncwarp();
        }
    }
}

template <int W>
static cudaError_t launch_w(const LaunchCfg& cfg, const KParams& kp, cudaStream_t st) {
    frame_warp_kernel<W><<<cfg.grid, cfg.threads, cfg.smem_bytes, st>>>(kp);
    return cudaGetLastError();
}
template <int W>
static cudaError_t smem_w(const LaunchCfg& cfg) {
    return cudaFuncSetAttribute(frame_warp_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)cfg.smem_bytes);
}
#define PFS_DISPATCH_W(FN, ...)                          \
    switch (cfg.W) {                                     \
        case 1: return FN<1>(__VA_ARGS__);               \
        case 2: return FN<2>(__VA_ARGS__);               \
        case 4: return FN<4>(__VA_ARGS__);               \
        case 8: return FN<8>(__VA_ARGS__);               \
        case 16: return FN<16>(__VA_ARGS__);             \
        case 32: return FN<32>(__VA_ARGS__);             \
        default: return cudaErrorInvalidValue;           \
    }
cudaError_t launch_frame_warp_kernel(const LaunchCfg& cfg, const KParams& kp, cudaStream_t stream) {
    PFS_DISPATCH_W(launch_w, cfg, kp, stream)
}
cudaError_t set_frame_warp_kernel_smem(const LaunchCfg& cfg) { PFS_DISPATCH_W(smem_w, cfg) }
size_t warp_kernel_smem_per_warp(int num_qubits, int64_t num_slots, int64_t num_noise) {
    return (((size_t)2 * num_qubits + num_slots + num_noise + 1) & ~(size_t)1) * 4;
}

size_t frame_smem_bytes(int num_qubits, int W) { return (size_t)2 * num_qubits * W * 4; }

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

cudaError_t launch_noise_kernel(int W, const KParams& kp, int64_t n_tiles, cudaStream_t st) {
    if (n_tiles <= 0 || kp.pregen_chunks <= 0) return cudaSuccess;
    dim3 grid((unsigned)((kp.pregen_chunks + 8 * NZ_ITEMS_PER_WARP - 1) / (8 * NZ_ITEMS_PER_WARP)),
              (unsigned)n_tiles);
    if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
    switch (W) {
        case 1: noise_kernel<1><<<grid, 256, 0, st>>>(kp); break;
        case 2: noise_kernel<2><<<grid, 256, 0, st>>>(kp); break;
        case 4: noise_kernel<4><<<grid, 256, 0, st>>>(kp); break;
        case 8: noise_kernel<8><<<grid, 256, 0, st>>>(kp); break;
        case 16: noise_kernel<16><<<grid, 256, 0, st>>>(kp); break;
        case 32: noise_kernel<32><<<grid, 256, 0, st>>>(kp); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

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
        for (int sl = t; sl < 32 * W; sl += 256) {
            const int64_t s = s0 + sl;
            if (s >= num_shots) break;
            const uint32_t* o = tout + sl * 9;
            uint4* dst = reinterpret_cast<uint4*>(out + s * pitch + b0);
            dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
            dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
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
