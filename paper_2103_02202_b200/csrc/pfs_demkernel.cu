// dem_kernel — detection events from the detector error model (pfs_dem.cpp).
//
// A CTA owns a tile of 32 shots at a time (the RNG tile of DESIGN.md §4 with
// W = 1): its warps take the tile's noise instructions, draw each one's hits
// with the frame sampler's own counter-based schedule (noise_op_warp, the same
// draws as noise_chunk / noise_kernel), and XOR every hit's component
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

__global__ void __launch_bounds__(32 * DEM_WARPS, 1) dem_kernel(const __grid_constant__ KParams kp,
                                                                const __grid_constant__ DemParams dp) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int ncols = kp.num_cols;
    const int ncw = (ncols + 3) & ~3;
    uint32_t* const ev = sm;                                    // [ncols] column words of the tile
    uint32_t* const cnt = ev + ncw;                             // [ncols] (counts mode)
    uint32_t* const wscr = cnt + (kp.counts_in_smem ? ncw : 0) + (size_t)warp * 32 * NZ_MAX_LIST;
    uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
    if (kp.counts_in_smem)
        for (int i = threadIdx.x; i < ncols; i += blockDim.x) cnt[i] = 0u;
    for (int64_t tile = blockIdx.x; tile < kp.n_tiles; tile += gridDim.x) {
        const uint32_t g = (uint32_t)(kp.tile_offset + (uint64_t)tile);
        for (int i = threadIdx.x; i < ncols; i += blockDim.x) ev[i] = 0u;
        __syncthreads();
        for (int o = warp; o < kp.num_noise; o += NW) {
            const NoiseParam np = kp.noise[o];
            if (np.flags & NZ_NONE) continue;
            const uint32_t ch = __ldg(kp.noise_ch + o);
            const uint32_t cb = __ldg(dp.comp_base + o);
            noise_op_warp(kp, np, (uint32_t)o, g, wscr, sl, lane, [&](uint32_t trial, uint32_t pick) {
                const uint32_t app = trial >> 5, bit = 1u << (trial & 31u);
                uint32_t xm, zm;
                pattern_of(ch, pick, xm, zm);
                const uint32_t mask = (xm & 1u) | ((zm & 1u) << 1) | ((xm & 2u) << 1) | ((zm & 2u) << 2);
                for (uint32_t k = 0; k < 4; k++) {
                    if (!((mask >> k) & 1u)) continue;
                    const uint32_t ci = cb + app * 4 + k;
                    const uint32_t e1 = __ldg(dp.comp_ptr + ci + 1);
                    for (uint32_t e = __ldg(dp.comp_ptr + ci); e < e1; e++) atomicXor(ev + __ldg(dp.cols + e), bit);
                }
            });
        }
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
        } else if (dp.b8_out != nullptr) {
            const int nblk = (ncols + 31) >> 5;
            const int64_t shot = tile * 32 + lane;
            for (int B = warp; B < nblk; B += NW) {
                const int col = B * 32 + lane;
                uint32_t t = transpose32_lane(col < ncols ? ev[col] : 0u, lane);
                if (shot < kp.num_shots) {
                    uint8_t* p = dp.b8_out + shot * dp.b8_pitch + (int64_t)B * 4;
                    const int64_t nb = dp.b8_bytes - (int64_t)B * 4;
                    if (((dp.b8_pitch | reinterpret_cast<uintptr_t>(dp.b8_out)) & 3) == 0 && nb >= 4)
                        *reinterpret_cast<uint32_t*>(p) = t;
                    else
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

size_t dem_smem_bytes(int warps, int64_t num_cols, bool counts) {
    const size_t ncw = ((size_t)num_cols + 3) & ~(size_t)3;
    return (ncw * (counts ? 2 : 1) + (size_t)warps * 32 * NZ_MAX_LIST) * 4;
}

cudaError_t set_dem_kernel_smem(size_t smem) {
    return cudaFuncSetAttribute(dem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_dem_kernel(const KParams& kp, const DemParams& dp, int grid, size_t smem, cudaStream_t st) {
    dem_kernel<<<grid, 32 * dp.warps, smem, st>>>(kp, dp);
    return cudaGetLastError();
}

}  // namespace pfs
