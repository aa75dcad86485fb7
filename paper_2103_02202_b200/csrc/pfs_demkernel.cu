// dem_kernel — detection events from the detector error model (pfs_dem.cpp).
//
// A CTA owns a tile of 32 shots at a time (the RNG tile of DESIGN.md §4 with
// W = 1): its warps take the tile's noise chunks, 32 (instruction, chunk) work
// items per pass, draw each one's hits with the frame sampler's own
// counter-based schedule (the same draws as noise_chunk), and
// XOR every hit's component
// signatures into one shared-memory word per output column (bit s = shot s).
// The column words are then transposed in 32x32 blocks and stored as the
// shot-major b8 rows (stabsim/io_formats.py:94-96, 208-227), or popcounted
// (counts mode), or written column-major (rows mode).
#include <cuda_runtime.h>

#include <cstdint>

#include "pfs_device.cuh"
#include "pfs_internal.h"

namespace pfs {

constexpr int DEM_WARPS = 16;

// The tile's noise chunks of ALL instructions, 32 per warp pass: lane l takes
// work item (ordinal o, chunk r) and draws exactly what noise_chunk draws for
// it — block 0 gives the Binomial count and the first hit, the
// warp compacts the hits and each lane makes one position per round (owner's
// ordinal and chunk shuffled in), duplicates / oversize counts are redrawn
// serially.  Packing chunks of different instructions keeps all lanes busy
// when an instruction has fewer than 32 chunks per 32-shot tile.
template <typename Apply>
__device__ __forceinline__ void noise_items_warp(const KParams& kp, const uint2* items, uint32_t n_items,
                                                 uint32_t first, const TileKey& tk, uint32_t* wscr, uint32_t* sl,
                                                 int lane, Apply apply) {
    const uint32_t it = first + (uint32_t)lane;
    const bool valid = it < n_items;
    const uint2 oc = valid ? __ldg(items + it) : make_uint2(0u, 0u);
    const uint32_t o = oc.x, r = oc.y;
    NoiseParam np{};
    if (valid) np = kp.noise[o];
    const bool all = valid && np.zone == NZONE_ALL;
    const uint32_t L = valid ? np.L : 1u;
    const uint32_t lg = 31u - __clz(L);
    const uint32_t sh = 32u - lg;
    // valid positions of chunk r (T = 32 shots, cs = min(L, 32): trial = r L + pos)
    uint32_t vlen = 0;
    if (valid) {
        const uint32_t nS = 32u / np.cs, k = r / nS;
        vlen = min(np.ca, np.apps - k * np.ca) * np.cs;
    }
    uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0, count = 0;
    if (valid && !all) {
        noise_block(tk, 0u, r, o, w0, w1, w2, w3);
        count = chunk_count(kp.noise_tab + np.tab, np.len, w0, w1);
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
    const uint32_t excl = pre - c;
    for (uint32_t j0 = 0; j0 < H; j0 += 32) {
        const uint32_t j = j0 + (uint32_t)lane;
        uint32_t lo = 0;  // owner lane: smallest q with pre[q] > j
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
            const uint32_t pv = __shfl_sync(0xFFFFFFFFu, pre, (int)(lo + st - 1));
            if (pv <= j) lo += st;
        }
        const int owner = (int)(lo > 31u ? 31u : lo);
        const uint32_t oexcl = __shfl_sync(0xFFFFFFFFu, excl, owner);
        const uint32_t oo = __shfl_sync(0xFFFFFFFFu, o, owner);
        const uint32_t orr = __shfl_sync(0xFFFFFFFFu, r, owner);
        const uint32_t osh = __shfl_sync(0xFFFFFFFFu, sh, owner);
        const uint32_t olg = __shfl_sync(0xFFFFFFFFu, lg, owner);
        const uint32_t onp = __shfl_sync(0xFFFFFFFFu, np.npat, owner);
        uint32_t x = __shfl_sync(0xFFFFFFFFu, w2, owner);
        uint32_t y = __shfl_sync(0xFFFFFFFFu, w3, owner);
        if (j < H) {
            const uint32_t h = j - oexcl;
            if (h > 0) {
                uint32_t b0, b1, b2, b3;
                noise_block(tk, (h + 1) >> 1, orr, oo, b0, b1, b2, b3);
                x = (h & 1u) ? b0 : b2;
                y = (h & 1u) ? b1 : b3;
            }
            const uint32_t pos = olg ? (x >> osh) : 0u;
            wscr[j] = (pos << 4) | (onp > 1 ? __umulhi(y, onp) : 0u);
        }
    }
    __syncwarp();
    bool dup = false;
    for (uint32_t h = 1; h < c; h++)
        for (uint32_t q = 0; q < h; q++) dup |= (wscr[excl + h] >> 4) == (wscr[excl + q] >> 4);
    // apply, one hit per lane (converged: a chunk lane walking its own hits left
    // half the lanes idle): hit j of the pass belongs to the chunk lane found by
    // the same search; chunks on the reference path are skipped here
    const bool slow = dup || big || all;
    const uint32_t slowm = __ballot_sync(0xFFFFFFFFu, slow);
    for (uint32_t j0 = 0; j0 < H; j0 += 32) {
        const uint32_t j = j0 + (uint32_t)lane;
        uint32_t lo = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
            const uint32_t pv = __shfl_sync(0xFFFFFFFFu, pre, (int)(lo + st - 1));
            if (pv <= j) lo += st;
        }
        const int owner = (int)(lo > 31u ? 31u : lo);
        const uint32_t oo = __shfl_sync(0xFFFFFFFFu, o, owner);
        const uint32_t obase = __shfl_sync(0xFFFFFFFFu, r * L, owner);
        const uint32_t ovlen = __shfl_sync(0xFFFFFFFFu, vlen, owner);
        if (j < H && !((slowm >> owner) & 1u)) {
            const uint32_t e = wscr[j];
            if ((e >> 4) < ovlen) apply(oo, obase + (e >> 4), e & 15u);
        }
    }
    if (slow) {
        const NoiseOp nz = noise_op_of(np, o);
        noise_chunk(tk, nz, kp.noise_tab, r, vlen, sl,
                    [&](uint32_t pos, uint32_t pick) { apply(o, r * L + pos, pick); });
    }
    __syncwarp();
}

// Visit the columns of a packed component word (up to 3 inline; long
// signatures through the CSR columns)
template <typename F>
__device__ __forceinline__ void for_word(const DemParams& dp, unsigned long long w, F f) {
    const uint32_t n = (uint32_t)(w >> 62);
    if (n) {
        f((uint32_t)(w & 0xFFFFFu));
        if (n > 1) f((uint32_t)((w >> 20) & 0xFFFFFu));
        if (n > 2) f((uint32_t)((w >> 40) & 0xFFFFFu));
        return;
    }
    const uint32_t b = (uint32_t)w, e1 = b + ((uint32_t)(w >> 32) & 0x3FFFFFFFu);
    for (uint32_t e = b; e < e1; e++) f(__ldg(dp.cols + e));
}

// A hit's components (mask bit k: x / z on slot 0 / 1): all signature words are
// loaded before any column is touched, so their L2 round trips overlap
template <typename F>
__device__ __forceinline__ void for_hit_columns(const DemParams& dp, uint32_t cb, uint32_t mask, F f) {
    unsigned long long w[4];
#pragma unroll
    for (int k = 0; k < 4; k++) w[k] = ((mask >> k) & 1u) ? __ldg(dp.comp_words + cb + k) : 0ull;
#pragma unroll
    for (int k = 0; k < 4; k++)
        if ((mask >> k) & 1u) for_word(dp, w[k], f);
}

// GC: the column words live in the tile-major global scratch kp.ev_out
// ([tile][col], zeroed by the host, transposed by tiles_to_b8 afterwards)
template <bool GC>
__global__ void __launch_bounds__(32 * DEM_WARPS, 2) dem_kernel(const __grid_constant__ KParams kp,
                                                                const __grid_constant__ DemParams dp) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int ncols = kp.num_cols;
    const int ncw = GC ? 0 : 32 * ((((ncols + 31) >> 5) + 3) & ~3);  // also 32 shot rows (16-byte aligned)
    uint32_t* const cnt = sm + ncw;                             // [ncols] (counts mode)
    uint32_t* const wscr = cnt + (kp.counts_in_smem ? ncw : 0) + (size_t)warp * 32 * NZ_MAX_LIST;
    uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    if (kp.counts_in_smem)
        for (int i = threadIdx.x; i < ncols; i += blockDim.x) cnt[i] = 0u;
    // b8 output from shared memory: the tile is kept shot-major (32 rows of
    // rw words, bit c of row s = column c of shot s), so each row already is
    // the shot's b8 row and is stored without a transpose
    const bool shot_major = !GC && dp.b8_out != nullptr && kp.counts == nullptr;
    const int rw = (((ncols + 31) >> 5) + 3) & ~3;  // words per shot row (16-byte multiple)
    for (int64_t tile = blockIdx.x; tile < kp.n_tiles; tile += gridDim.x) {
        const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
        // column words of the tile: shared, or the global output rows at
        // ev_out + col * out_row_stride + tile * out_tile_stride (b8 scratch
        // [tile][col], or the caller's column-major rows)
        uint32_t* const ev = GC ? kp.ev_out + (size_t)tile * kp.out_tile_stride : sm;
        const int64_t cs = GC ? kp.out_row_stride : 1;
        if (!GC) {
            for (int i = threadIdx.x; i < (shot_major ? 32 * rw : ncols); i += blockDim.x) ev[i] = 0u;
            __syncthreads();
        }
        for (uint32_t first = 32u * warp; first < (uint32_t)dp.n_items; first += 32u * NW) {
            noise_items_warp(kp, dp.items, (uint32_t)dp.n_items, first, tk, wscr, sl, lane,
                             [&](uint32_t o, uint32_t trial, uint32_t pick) {
                const uint32_t app = trial >> 5, bit = 1u << (trial & 31u);
                uint32_t xm, zm;
                pattern_of(__ldg(kp.noise_ch + o), pick, xm, zm);
                const uint32_t mask = (xm & 1u) | ((zm & 1u) << 1) | ((xm & 2u) << 1) | ((zm & 2u) << 2);
                const uint32_t cb = __ldg(dp.comp_base + o) + app * 4;
                if (shot_major) {
                    uint32_t* const row = ev + (trial & 31u) * rw;
                    for_hit_columns(dp, cb, mask, [&](uint32_t col) { atomicXor(row + (col >> 5), 1u << (col & 31u)); });
                } else {
                    for_hit_columns(dp, cb, mask, [&](uint32_t col) { atomicXor(ev + (int64_t)col * cs, bit); });
                }
            });
        }
        if (GC) continue;  // transposed by tiles_to_b8
        __syncthreads();
        const int64_t rem = kp.num_shots - tile * 32;
        const uint32_t tail = rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
        if (kp.counts != nullptr) {
            for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
                const uint32_t n = __popc(ev[c] & tail);
                if (n) {
                    if (kp.counts_in_smem) cnt[c] += n;  // one thread per column
                    else atomicAdd(kp.counts + c, (unsigned long long)n);
                }
            }
        } else if (shot_major) {
            // row s -> b8 row of shot tile*32+s: 16-byte stores when aligned
            const int nb = (int)dp.b8_bytes;
            const bool a16 = ((dp.b8_pitch | reinterpret_cast<uintptr_t>(dp.b8_out)) & 15) == 0;
            const int nv = a16 ? nb >> 4 : 0;  // whole 16-byte vectors per row
            const int nrow = rem >= 32 ? 32 : (rem <= 0 ? 0 : (int)rem);
            for (int i = threadIdx.x; i < nrow * nv; i += blockDim.x) {
                const int sr = i / nv, v = i - sr * nv;
                const uint4 q = *reinterpret_cast<const uint4*>(ev + sr * rw + 4 * v);
                *reinterpret_cast<uint4*>(dp.b8_out + (tile * 32 + sr) * dp.b8_pitch + 16 * v) = q;
            }
            const int tb = nb - 16 * nv;  // remaining bytes per row
            for (int i = threadIdx.x; i < nrow * tb; i += blockDim.x) {
                const int sr = i / tb, bI = 16 * nv + (i - sr * tb);
                dp.b8_out[(tile * 32 + sr) * dp.b8_pitch + bI] =
                    (uint8_t)(ev[sr * rw + (bI >> 2)] >> (8 * (bI & 3)));
            }
        } else if (dp.b8_out != nullptr) {
            // whole 32-column blocks store one aligned word per shot; the last,
            // partial block (and unaligned outputs) go bytewise
            const int nblk = (ncols + 31) >> 5;
            const int64_t shot = tile * 32 + lane;
            const bool live = shot < kp.num_shots;
            const bool aligned = ((dp.b8_pitch | reinterpret_cast<uintptr_t>(dp.b8_out)) & 3) == 0;
            const int nfull = aligned ? (int)(dp.b8_bytes >> 2) : 0;  // blocks with 4 whole bytes
            uint32_t* const row32 = reinterpret_cast<uint32_t*>(dp.b8_out + (live ? shot : 0) * dp.b8_pitch);
            for (int B = warp; B < nfull && B < nblk; B += NW) {
                const int col = B * 32 + lane;  // bits past the last column stay 0
                const uint32_t t = transpose32_lane(col < ncols ? ev[col] : 0u, lane);
                if (live) row32[B] = t;
            }
            for (int B = nfull + ((warp - nfull % NW + NW) % NW); B < nblk; B += NW) {
                const int col = B * 32 + lane;
                const uint32_t t = transpose32_lane(col < ncols ? ev[col] : 0u, lane);
                if (live) {
                    uint8_t* p = dp.b8_out + shot * dp.b8_pitch + (int64_t)B * 4;
                    const int64_t nb = dp.b8_bytes - (int64_t)B * 4;
                    for (int j = 0; j < 4 && j < nb; j++) p[j] = (uint8_t)(t >> (8 * j));
                }
            }
        } else if (dp.rows_out != nullptr) {
            for (int c = threadIdx.x; c < ncols; c += blockDim.x) dp.rows_out[(int64_t)c * dp.rows_stride + tile] = ev[c];
        }
        __syncthreads();
    }
    if (kp.counts_in_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < ncols; i += blockDim.x)
            if (cnt[i]) atomicAdd(kp.counts + i, (unsigned long long)cnt[i]);
    }
}

// Small circuits (a few hundred output columns): every warp owns its own
// 32-shot tile and column words, so tiles need no CTA barrier at all.
__global__ void __launch_bounds__(32 * DEM_WARPS, 2) dem_warp_kernel(const __grid_constant__ KParams kp,
                                                                     const __grid_constant__ DemParams dp) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int ncols = kp.num_cols;
    const int ncw = (ncols + 3) & ~3;
    uint32_t* const cnt = sm;  // [ncols] CTA counts (counts mode)
    uint32_t* const ev = sm + (kp.counts_in_smem ? ncw : 0) + (size_t)warp * (ncw + 32 * NZ_MAX_LIST);
    uint32_t* const wscr = ev + ncw;
    uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    if (kp.counts_in_smem)
        for (int i = threadIdx.x; i < ncols; i += blockDim.x) cnt[i] = 0u;
    __syncthreads();
    for (int64_t tile = (int64_t)blockIdx.x * NW + warp; tile < kp.n_tiles; tile += (int64_t)gridDim.x * NW) {
        const TileKey tk = tile_key(kp.seed, kp.tile_offset + (uint64_t)tile);
        for (int i = lane; i < ncols; i += 32) ev[i] = 0u;
        __syncwarp();
        for (uint32_t first = 0; first < (uint32_t)dp.n_items; first += 32u) {
            noise_items_warp(kp, dp.items, (uint32_t)dp.n_items, first, tk, wscr, sl, lane,
                             [&](uint32_t o, uint32_t trial, uint32_t pick) {
                const uint32_t app = trial >> 5, bit = 1u << (trial & 31u);
                uint32_t xm, zm;
                pattern_of(__ldg(kp.noise_ch + o), pick, xm, zm);
                const uint32_t mask = (xm & 1u) | ((zm & 1u) << 1) | ((xm & 2u) << 1) | ((zm & 2u) << 2);
                const uint32_t cb = __ldg(dp.comp_base + o) + app * 4;
                for_hit_columns(dp, cb, mask, [&](uint32_t col) { atomicXor(ev + col, bit); });
            });
        }
        __syncwarp();
        const int64_t rem = kp.num_shots - tile * 32;
        const uint32_t tail = rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
        if (kp.counts != nullptr) {
            for (int c = lane; c < ncols; c += 32) {
                const uint32_t n = __popc(ev[c] & tail);
                if (n) {
                    if (kp.counts_in_smem) atomicAdd(cnt + c, n);
                    else atomicAdd(kp.counts + c, (unsigned long long)n);
                }
            }
        } else if (dp.b8_out != nullptr) {
            const int64_t shot = tile * 32 + lane;
            const bool live = shot < kp.num_shots;
            const bool aligned = ((dp.b8_pitch | reinterpret_cast<uintptr_t>(dp.b8_out)) & 3) == 0;
            for (int B = 0; B * 32 < ncols; B++) {
                const int col = B * 32 + lane;
                const uint32_t t = transpose32_lane(col < ncols ? ev[col] : 0u, lane);
                if (!live) continue;
                uint8_t* p = dp.b8_out + shot * dp.b8_pitch + (int64_t)B * 4;
                const int64_t nb = dp.b8_bytes - (int64_t)B * 4;
                if (aligned && nb >= 4) *reinterpret_cast<uint32_t*>(p) = t;
                else for (int j = 0; j < 4 && j < nb; j++) p[j] = (uint8_t)(t >> (8 * j));
            }
        } else if (dp.rows_out != nullptr) {
            for (int c = lane; c < ncols; c += 32) dp.rows_out[(int64_t)c * dp.rows_stride + tile] = ev[c];
        }
        __syncwarp();
    }
    if (kp.counts_in_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < ncols; i += blockDim.x)
            if (cnt[i]) atomicAdd(kp.counts + i, (unsigned long long)cnt[i]);
    }
}

size_t dem_warp_smem_bytes(int warps, int64_t num_cols, bool counts) {
    const size_t ncw = ((size_t)num_cols + 3) & ~(size_t)3;
    return ((counts ? ncw : 0) + (size_t)warps * (ncw + 32 * NZ_MAX_LIST)) * 4;
}

size_t dem_smem_bytes(int warps, int64_t num_cols, bool counts) {
    const size_t ncw = 32 * (((((size_t)num_cols + 31) >> 5) + 3) & ~(size_t)3);  // 32 shot rows, 16-byte multiples
    return (ncw * (counts ? 2 : 1) + (size_t)warps * 32 * NZ_MAX_LIST) * 4;
}

cudaError_t set_dem_kernel_smem(size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(dem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(dem_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(dem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_dem_kernel(const KParams& kp, const DemParams& dp, bool global_cols, int grid, size_t smem,
                              cudaStream_t st) {
    if (dp.per_warp) dem_warp_kernel<<<grid, 32 * dp.warps, smem, st>>>(kp, dp);
    else if (global_cols) dem_kernel<true><<<grid, 32 * dp.warps, smem, st>>>(kp, dp);
    else dem_kernel<false><<<grid, 32 * dp.warps, smem, st>>>(kp, dp);
    return cudaGetLastError();
}

}  // namespace pfs
