// frame_col_kernel — the word-column frame interpreter.
//
// Every consumer warp owns ONE 32-shot word column of the frame table for the
// whole circuit: its own x and z bit-planes (qubit-major, one uint32 per qubit:
// shot s = bit s) and its own record ring, all in shared
// memory.  Lanes take the independent applications of an op, so warps never
// wait for each other: the only synchronisation is __syncwarp between ops and
// the op-block ring below.  Reference semantics per op:
//   gate rules      stabsim/frame_sim.py:64-72 (plans gates.py:326-348)
//   M / R / MR      stabsim/frame_sim.py:74-90
//   noise           stabsim/frame_sim.py:92-167, entropy.py:65-113 (draws: DESIGN.md §4)
//   detectors       stabsim/circuit.py:247-256, io_formats.py:208-227
//   b8 output       stabsim/bitvec.py:193-209, io_formats.py:94-96
//
// Op stream.  The host lays the program out as self-describing blocks
// (build_col_stream).  One producer warp bulk-copies (cp.async.bulk, TMA) each
// block into a ring of COL_SLOTS shared-memory slots; a full/empty mbarrier pair
// per slot lets the consumer warps drift up to COL_SLOTS blocks apart, so the
// op stream crosses L2 once per CTA pass instead of once per warp.
//
// Output.  Detection events (or measurement records) are produced per warp as
// one word per column; 32 consecutive columns are transposed in registers
// (5 __shfl_xor_sync butterflies) and each lane stores 4 bytes of its shot's
// b8 row, so the shot-major output is written once, with no intermediate
// column-major table and no separate transpose kernel.
//
// Randomness follows DESIGN.md §4 with a tile of one word (T = 32): coin rows
// and noise chunks are keyed by the global word index, so any split of a shot
// range across launches or GPUs gives bit-identical results.
#include <cuda_runtime.h>

#include <cstdint>

#include "pfs_device.cuh"
#include "pfs_internal.h"

namespace pfs {

namespace {

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(mbar)) : "memory");
}

// Output column sink of one warp: a two-block ring of column words; a block of
// 32 columns is transposed and stored as soon as its last column arrives.
struct Sink {
    uint32_t* buf;      // 64 words (shared)
    uint32_t flushed;   // blocks already stored (warp-uniform)
};

__device__ __forceinline__ void sink_flush(const ColParams& cp, const Sink& sk, uint32_t B, int64_t u,
                                           int64_t num_shots, int lane) {
    __syncwarp();
    uint32_t v = sk.buf[(B & 1u) * 32u + (uint32_t)lane];
    if (B * 32u + (uint32_t)lane >= (uint32_t)cp.ncols_out) v = 0u;
    uint32_t t = transpose32_lane(v, lane);  // lane s: columns 32B.. of shot s
    if (cp.ref_words != nullptr) t ^= __ldg(cp.ref_words + B);
    const int64_t shot = u * 32 + lane;
    if (shot < num_shots) {
        uint8_t* p = cp.b8_out + shot * cp.b8_pitch + (int64_t)B * 4;
        const int64_t nb = cp.b8_bytes - (int64_t)B * 4;
        if (cp.b8_aligned && nb >= 4) {
            *reinterpret_cast<uint32_t*>(p) = t;
        } else {
            for (int j = 0; j < 4 && j < nb; j++) p[j] = (uint8_t)(t >> (8 * j));
        }
    }
    __syncwarp();
}

// Warp-collective: lane-valid columns (a window of at most 32 consecutive
// columns, in increasing order across calls) enter the sink.
__device__ __forceinline__ void sink_put(const ColParams& cp, Sink& sk, bool valid, uint32_t col, uint32_t v,
                                         int64_t u, int64_t num_shots, int lane) {
    if (valid) sk.buf[((col >> 5) & 1u) * 32u + (col & 31u)] = v;
    const uint32_t cend = __reduce_max_sync(0xFFFFFFFFu, valid ? col + 1u : 0u);
    while ((sk.flushed + 1u) * 32u <= cend) {
        sink_flush(cp, sk, sk.flushed, u, num_shots, lane);
        sk.flushed++;
    }
}

template <uint32_t CODE>
__device__ __forceinline__ void gate2(uint32_t* X, uint32_t* Z, const uint32_t* P, uint32_t count, int lane) {
    constexpr int U = 4;
    const uint2* P2 = reinterpret_cast<const uint2*>(P);
    for (uint32_t i0 = (uint32_t)lane; i0 < count; i0 += 32 * U) {
        uint2 qq[U];
        uint32_t x0[U], x1[U], z0[U], z1[U];
#pragma unroll
        for (int t = 0; t < U; t++) {
            const uint32_t i = i0 + 32u * t;
            qq[t] = i < count ? P2[i] : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int t = 0; t < U; t++) {
            if (i0 + 32u * t >= count) continue;
            x0[t] = X[qq[t].x]; x1[t] = X[qq[t].y];
            z0[t] = Z[qq[t].x]; z1[t] = Z[qq[t].y];
        }
#pragma unroll
        for (int t = 0; t < U; t++) {
            if (i0 + 32u * t >= count) continue;
            const uint32_t a = qq[t].x, b = qq[t].y;
            if (CODE == R_CX) {
                X[b] = x1[t] ^ x0[t]; Z[a] = z0[t] ^ z1[t];
            } else if (CODE == R_CZ) {
                Z[a] = z0[t] ^ x1[t]; Z[b] = z1[t] ^ x0[t];
            } else if (CODE == R_CY) {
                X[b] = x1[t] ^ x0[t]; Z[a] = z0[t] ^ x1[t] ^ z1[t]; Z[b] = z1[t] ^ x0[t];
            } else {  // SWAP
                X[a] = x1[t]; X[b] = x0[t]; Z[a] = z1[t]; Z[b] = z0[t];
            }
        }
    }
}

template <uint32_t CODE>
__device__ __forceinline__ void gate1(uint32_t* X, uint32_t* Z, const uint32_t* P, uint32_t count, int lane) {
    constexpr int U = 4;
    for (uint32_t i0 = (uint32_t)lane; i0 < count; i0 += 32 * U) {
        uint32_t q[U], xv[U], zv[U];
#pragma unroll
        for (int t = 0; t < U; t++) {
            const uint32_t i = i0 + 32u * t;
            q[t] = i < count ? P[i] : 0u;
        }
#pragma unroll
        for (int t = 0; t < U; t++) {
            if (i0 + 32u * t >= count) continue;
            xv[t] = X[q[t]]; zv[t] = Z[q[t]];
        }
#pragma unroll
        for (int t = 0; t < U; t++) {
            if (i0 + 32u * t >= count) continue;
            if (CODE == R_SWAPXZ) { X[q[t]] = zv[t]; Z[q[t]] = xv[t]; }
            else if (CODE == R_ZXORX) Z[q[t]] = zv[t] ^ xv[t];
            else X[q[t]] = xv[t] ^ zv[t];  // R_XXORZ
        }
    }
}

}  // namespace

__global__ void __launch_bounds__(32 * (COL_MAX_WARPS + 1), 1)
frame_col_kernel(const __grid_constant__ KParams kp, const __grid_constant__ ColParams cp) {
    extern __shared__ __align__(16) uint8_t smem8[];
    constexpr uint32_t K = COL_SLOTS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = cp.nw;
    const uint32_t SB = (uint32_t)cp.slot_bytes;
    uint8_t* const slots = smem8;
    uint64_t* const full = reinterpret_cast<uint64_t*>(smem8 + K * SB);
    uint64_t* const empty = full + K;
    uint32_t* const cnt = reinterpret_cast<uint32_t*>(empty + K);
    const int64_t cnt_words = kp.counts_in_smem ? (((int64_t)kp.num_cols + 3) & ~3ll) : 0;
    const int n = kp.num_qubits;

    if (kp.counts_in_smem)
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x) cnt[i] = 0u;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < K; s++) { mbar_init(full + s, 1); mbar_init(empty + s, (uint32_t)NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t per_pass = (int64_t)gridDim.x * NW;
    const int64_t first = (int64_t)blockIdx.x * NW;
    const int64_t passes = cp.n_units > first ? (cp.n_units - first + per_pass - 1) / per_pass : 0;
    const int32_t nblk = cp.n_blocks;

    if (warp == NW) {
        // ---------------- producer: stream the op blocks into the slot ring ----------------
        if (lane == 0 && nblk > 0) {
            uint32_t seq = 0;
            uint2 nxt = __ldg(cp.binfo);
            for (int64_t p = 0; p < passes; p++) {
                for (int32_t i = 0; i < nblk; i++, seq++) {
                    const uint2 bi = nxt;
                    nxt = __ldg(cp.binfo + (i + 1 < nblk ? i + 1 : 0));
                    const uint32_t s = seq % K;
                    if (seq >= K) mbar_wait(empty + s, ((seq / K) - 1u) & 1u);
                    bulk_load(slots + s * SB, cp.stream + (size_t)bi.x * 4, bi.y, full + s);
                }
            }
        }
    } else {
        // ---------------- consumers: one word column per warp ----------------
        uint32_t* const X = reinterpret_cast<uint32_t*>(smem8 + K * SB + 2 * K * 8) + cnt_words +
                            (size_t)warp * cp.warp_words;
        uint32_t* const Z = X + n;
        uint32_t* const ring = Z + n;
        Sink sk{ring + kp.num_slots, 0u};
        uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
        const bool b8 = cp.b8_out != nullptr;
        uint32_t seq = 0;
        for (int64_t p = 0; p < passes; p++) {
            const int64_t u = first + p * per_pass + warp;  // local word index
            const bool live = u < cp.n_units;
            const uint32_t g = (uint32_t)(kp.tile_offset + (uint64_t)u);  // global word = RNG tile
            const int64_t rem = kp.num_shots - u * 32;
            const uint32_t tail = rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
            sk.flushed = 0u;
            if (live) {
                // ---- FrameBatch.__init__: x = 0, z = coin rows 0..n-1 (frame_sim.py:36-39) ----
                for (int q = lane; q < n; q += 32) X[q] = 0u;
                const uint32_t k1 = coin_k1((uint32_t)n);
                for (uint32_t kb = 0; kb < k1; kb += 32) {
                    const uint32_t k = kb + (uint32_t)lane;
                    if (k >= k1 || !coin_group_live(k, 0u, (uint32_t)n)) continue;
                    uint32_t o[4];
                    coin_group<1>(kp, k, 0u, g, u, 0u, (uint32_t)n, o);
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        const uint32_t e = coin_row0(k) + 32u * r;
                        if (e < (uint32_t)n) Z[e] = o[r];
                    }
                }
                for (int i = lane; i < kp.num_obs; i += 32) ring[i] = 0u;
                __syncwarp();
            }
            for (int32_t bi = 0; bi < nblk; bi++, seq++) {
                const uint32_t s = seq % K;
                mbar_wait(full + s, (seq / K) & 1u);
                const uint32_t* const hb = reinterpret_cast<const uint32_t*>(slots + s * SB);
                if (live) {
                    const uint32_t kcf = hb[0], count = hb[1], oa = hb[2], ob = hb[3];
                    const uint32_t kind = kcf & 0xFFu, code = (kcf >> 8) & 0xFFu, flags = kcf >> 16;
                    const uint32_t hw = COL_HEAD_WORDS + (kind == K_NOISE ? COL_NP_WORDS : 0u);
                    const uint32_t* const P = (flags & F_GLOBALP) ? cp.stream + hb[5] : hb + hw;
                    switch (kind) {
                    case K_GATE:
                        switch (code) {
                            case R_SWAPXZ: gate1<R_SWAPXZ>(X, Z, P, count, lane); break;
                            case R_ZXORX: gate1<R_ZXORX>(X, Z, P, count, lane); break;
                            case R_XXORZ: gate1<R_XXORZ>(X, Z, P, count, lane); break;
                            case R_CX: gate2<R_CX>(X, Z, P, count, lane); break;
                            case R_CZ: gate2<R_CZ>(X, Z, P, count, lane); break;
                            case R_CY: gate2<R_CY>(X, Z, P, count, lane); break;
                            default: gate2<R_SWAP>(X, Z, P, count, lane); break;
                        }
                        break;
                    case K_M: case K_MR: case K_R: {
                        // lanes take coin groups: one Philox block = four coin rows
                        // 32 apart, so a warp pass covers 128 consecutive rows
                        const uint32_t lo = ob, hi = ob + (kind == K_MR ? 2u : 1u) * count;
                        const uint32_t k1 = coin_k1(hi);
                        const bool emit = cp.records != 0;
                        for (uint32_t kb = coin_k0(lo); kb < k1; kb += 32) {
                            const uint32_t k = kb + (uint32_t)lane;
                            const bool kl = k < k1 && coin_group_live(k, lo, hi);
                            uint2 qsv[4];
#pragma unroll
                            for (int r = 0; r < 4; r++) {
                                const uint32_t e = coin_row0(k) + 32u * r;
                                qsv[r] = make_uint2(0u, NO_SLOT);
                                if (!kl || e < lo || e >= hi) continue;
                                const uint32_t rel = e - lo;
                                if (kind == K_R) qsv[r].x = P[rel];
                                else if (kind == K_M || (rel & 1u))
                                    qsv[r] = reinterpret_cast<const uint2*>(P)[kind == K_MR ? rel >> 1 : rel];
                            }
                            uint32_t o[4] = {0u, 0u, 0u, 0u};
                            if (kl) coin_group<1>(kp, k, 0u, g, u, lo, hi, o);
#pragma unroll
                            for (int r = 0; r < 4; r++) {
                                const uint32_t e = coin_row0(k) + 32u * r;
                                const bool in = kl && e >= lo && e < hi;
                                const uint32_t rel = e - lo;
                                const bool rec = in && kind != K_R && (kind == K_M || (rel & 1u));
                                const uint32_t j = kind == K_MR ? rel >> 1 : rel;
                                uint32_t xv = 0u;
                                if (in) {
                                    const uint32_t q = qsv[r].x;
                                    if (kind == K_R) {
                                        X[q] = 0u; Z[q] = o[r];
                                    } else if (rec) {
                                        xv = X[q];
                                        if (kp.do_dets && qsv[r].y != NO_SLOT) ring[qsv[r].y] = xv;
                                        if (kind == K_M) Z[q] ^= o[r];
                                        else { X[q] = 0u; Z[q] = o[r]; }
                                    }
                                }
                                if (emit) {
                                    if (b8) sink_put(cp, sk, rec, oa + j, xv, u, kp.num_shots, lane);
                                    else if (rec) cp.rows_out[(int64_t)(oa + j) * cp.rows_stride + u] = xv;
                                }
                            }
                        }
                        break;
                    }
                    case K_NOISE: {
                        const int ar = code == CH_DEP2 ? 2 : 1;
                        if (kp.masks != nullptr) {
                            // injected masks: per target, x row then z row
                            for (uint32_t j = (uint32_t)lane; j < count * ar; j += 32) {
                                const uint32_t q = P[j];
                                const uint32_t* mrow = kp.masks + (int64_t)(oa + 2 * j) * kp.inject_words + u;
                                const uint32_t mx = __ldg(mrow), mz = __ldg(mrow + kp.inject_words);
                                if (flags & F_DUP) {
                                    if (mx) atomicXor(X + q, mx);
                                    if (mz) atomicXor(Z + q, mz);
                                } else {
                                    X[q] ^= mx;
                                    Z[q] ^= mz;
                                }
                            }
                            break;
                        }
                        const NoiseParam np = *reinterpret_cast<const NoiseParam*>(hb + COL_HEAD_WORDS);
                        if (np.flags & NZ_NONE) break;
                        for (uint32_t r = (uint32_t)lane; r < np.nchunks; r += 32)
                            noise_chunk(kp, np, ob, r, g, sl, 1, [&](uint32_t trial, uint32_t pick) {
                                const uint32_t app = trial >> 5;
                                const uint32_t bit = 1u << (trial & 31u);
                                uint32_t xm, zm;
                                pattern_of(code, pick, xm, zm);
                                const uint32_t q0 = P[app * ar];
                                if (xm & 1u) atomicXor(X + q0, bit);
                                if (zm & 1u) atomicXor(Z + q0, bit);
                                if (ar == 2) {
                                    const uint32_t q1 = P[app * 2 + 1];
                                    if (xm & 2u) atomicXor(X + q1, bit);
                                    if (zm & 2u) atomicXor(Z + q1, bit);
                                }
                            });
                        break;
                    }
                    case K_DET: {
                        if (!kp.do_dets) break;
                        for (uint32_t c0 = 0; c0 < count; c0 += 32) {
                            const uint32_t i = c0 + (uint32_t)lane;
                            const bool valid = i < count;
                            uint32_t acc = 0u;
                            if (valid) {
                                if (code == 2) {
                                    const uint2 sv = reinterpret_cast<const uint2*>(P)[i];
                                    if (sv.x != NO_SLOT) acc = ring[sv.x];
                                    if (sv.y != NO_SLOT) acc ^= ring[sv.y];
                                } else if (code) {
                                    for (uint32_t e = 0; e < code; e++) {
                                        const uint32_t sidx = P[i * code + e];
                                        if (sidx != NO_SLOT) acc ^= ring[sidx];
                                    }
                                } else {
                                    const uint32_t e0 = P[i], e1 = P[i + 1];
                                    for (uint32_t e = e0; e < e1; e++) {
                                        const uint32_t sidx = P[count + 1 + e];
                                        if (sidx != NO_SLOT) acc ^= ring[sidx];
                                    }
                                }
                            }
                            const uint32_t col = oa + i;
                            if (kp.counts != nullptr) {
                                const uint32_t tot = valid ? __popc(acc & tail) : 0u;
                                if (tot) {
                                    if (kp.counts_in_smem) atomicAdd(cnt + col, tot);
                                    else atomicAdd(kp.counts + col, (unsigned long long)tot);
                                }
                            } else if (b8) {
                                sink_put(cp, sk, valid, col, acc, u, kp.num_shots, lane);
                            } else if (valid) {
                                cp.rows_out[(int64_t)col * cp.rows_stride + u] = acc;
                            }
                        }
                        break;
                    }
                    case K_OBS: {
                        if (!kp.do_dets) break;
                        uint32_t acc = 0u;
                        for (uint32_t j = (uint32_t)lane; j < count; j += 32) {
                            const uint32_t sidx = P[j];
                            if (sidx != NO_SLOT) acc ^= ring[sidx];
                        }
                        acc = __reduce_xor_sync(0xFFFFFFFFu, acc);
                        if (lane == 0) ring[oa] ^= acc;
                        break;
                    }
                    default: break;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
            }
            // the last, partial block of output columns
            if (live && b8 && sk.flushed * 32u < (uint32_t)cp.ncols_out)
                sink_flush(cp, sk, sk.flushed, u, kp.num_shots, lane);
        }
    }
    if (kp.counts_in_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x)
            if (cnt[i]) atomicAdd(kp.counts + i, (unsigned long long)cnt[i]);
    }
}

size_t col_warp_words(int num_qubits, int64_t num_slots) {
    return ((size_t)2 * num_qubits + (size_t)num_slots + 64 + 3) & ~(size_t)3;
}

size_t col_smem_bytes(int nw, size_t warp_words, uint32_t slot_bytes, int64_t counts_words) {
    const size_t cw = counts_words > 0 ? (((size_t)counts_words + 3) & ~(size_t)3) : 0;
    return (size_t)COL_SLOTS * slot_bytes + 2 * COL_SLOTS * 8 + cw * 4 + (size_t)nw * warp_words * 4;
}

cudaError_t set_frame_col_kernel_smem(size_t smem) {
    return cudaFuncSetAttribute(frame_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_frame_col_kernel(const KParams& kp, const ColParams& cp, int grid, size_t smem,
                                    cudaStream_t stream) {
    frame_col_kernel<<<grid, 32 * (cp.nw + 1), smem, stream>>>(kp, cp);
    return cudaGetLastError();
}

}  // namespace pfs
