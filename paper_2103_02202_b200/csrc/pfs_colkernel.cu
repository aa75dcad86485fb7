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

// V-word vectors: a lane's slice of one frame row (V consecutive 32-shot words).
template <int V> struct VV { uint32_t w[V]; };

template <int V> __device__ __forceinline__ VV<V> vload(const uint32_t* p) {
    VV<V> r;
    if constexpr (V == 4) { const uint4 t = *reinterpret_cast<const uint4*>(p); r.w[0] = t.x; r.w[1] = t.y; r.w[2] = t.z; r.w[3] = t.w; }
    else if constexpr (V == 2) { const uint2 t = *reinterpret_cast<const uint2*>(p); r.w[0] = t.x; r.w[1] = t.y; }
    else r.w[0] = *p;
    return r;
}
template <int V> __device__ __forceinline__ void vstore(uint32_t* p, const VV<V>& v) {
    if constexpr (V == 4) *reinterpret_cast<uint4*>(p) = make_uint4(v.w[0], v.w[1], v.w[2], v.w[3]);
    else if constexpr (V == 2) *reinterpret_cast<uint2*>(p) = make_uint2(v.w[0], v.w[1]);
    else *p = v.w[0];
}
template <int V> __device__ __forceinline__ VV<V> vxor(const VV<V>& a, const VV<V>& b) {
    VV<V> r;
#pragma unroll
    for (int i = 0; i < V; i++) r.w[i] = a.w[i] ^ b.w[i];
    return r;
}
template <int V> __device__ __forceinline__ VV<V> vzero() {
    VV<V> r;
#pragma unroll
    for (int i = 0; i < V; i++) r.w[i] = 0u;
    return r;
}

// Transpose a complete block B of 32 output columns held one per lane (bit s
// = shot s of word w) and store each shot's 4 bytes of its b8 row.
__device__ __forceinline__ void store_block(const ColParams& cp, uint32_t v, uint32_t B, int64_t shot0,
                                            int64_t num_shots, int lane) {
    if (B * 32u + (uint32_t)lane >= (uint32_t)cp.ncols_out) v = 0u;
    uint32_t t = transpose32_lane(v, lane);  // lane s: columns 32B.. of shot s
    if (cp.ref_words != nullptr) t ^= __ldg(cp.ref_words + B);
    const int64_t shot = shot0 + lane;
    if (shot < num_shots) {
        uint8_t* p = cp.b8_out + shot * cp.b8_pitch + (int64_t)B * 4;
        const int64_t nb = cp.b8_bytes - (int64_t)B * 4;
        if (cp.b8_aligned && nb >= 4) {
            *reinterpret_cast<uint32_t*>(p) = t;
        } else {
            for (int j = 0; j < 4 && j < nb; j++) p[j] = (uint8_t)(t >> (8 * j));
        }
    }
}

// Output sink of one warp for columns that arrive in arbitrary windows (the
// measurement records of M/MR ops): per word a two-block ring of column words;
// a block is transposed and stored once its last column arrived.
template <int V>
struct Sink {
    uint32_t* buf;      // V x 64 words (shared)
    uint32_t flushed;   // blocks already stored (warp-uniform)
};

template <int V>
__device__ __forceinline__ void sink_flush(const ColParams& cp, const Sink<V>& sk, uint32_t B, int64_t u,
                                           int64_t num_shots, int lane) {
    __syncwarp();
#pragma unroll
    for (int w = 0; w < V; w++)
        store_block(cp, sk.buf[w * 64 + (B & 1u) * 32u + (uint32_t)lane], B, u * 32 * V + 32 * w, num_shots, lane);
    __syncwarp();
}

// Warp-collective: lane-valid columns (a window of at most 32 consecutive
// columns, in increasing order across calls) enter the sink.
template <int V>
__device__ __forceinline__ void sink_put(const ColParams& cp, Sink<V>& sk, bool valid, uint32_t col,
                                         const VV<V>& v, int64_t u, int64_t num_shots, int lane) {
    if (valid)
#pragma unroll
        for (int w = 0; w < V; w++) sk.buf[w * 64 + ((col >> 5) & 1u) * 32u + (col & 31u)] = v.w[w];
    const uint32_t cend = __reduce_max_sync(0xFFFFFFFFu, valid ? col + 1u : 0u);
    while ((sk.flushed + 1u) * 32u <= cend) {
        sink_flush<V>(cp, sk, sk.flushed, u, num_shots, lane);
        sk.flushed++;
    }
}

// Gate rules on a word column's frame: x plane X[q*V..], z plane Z[q*V..]
// (stabsim/frame_sim.py:64-72, rules gates.py:326-348; all XORs read old values).
template <uint32_t CODE, int V>
__device__ __forceinline__ void rule2(uint32_t* X, uint32_t* Z, uint2 q, const VV<V>& x0, const VV<V>& x1,
                                      const VV<V>& z0, const VV<V>& z1) {
    const uint32_t a = q.x * V, b = q.y * V;
    if (CODE == R_CX) {
        vstore<V>(X + b, vxor<V>(x1, x0)); vstore<V>(Z + a, vxor<V>(z0, z1));
    } else if (CODE == R_CZ) {
        vstore<V>(Z + a, vxor<V>(z0, x1)); vstore<V>(Z + b, vxor<V>(z1, x0));
    } else if (CODE == R_CY) {
        vstore<V>(X + b, vxor<V>(x1, x0)); vstore<V>(Z + a, vxor<V>(z0, vxor<V>(x1, z1)));
        vstore<V>(Z + b, vxor<V>(z1, x0));
    } else {  // SWAP
        vstore<V>(X + a, x1); vstore<V>(X + b, x0); vstore<V>(Z + a, z1); vstore<V>(Z + b, z0);
    }
}

template <uint32_t CODE, int V>
__device__ __forceinline__ void rule1(uint32_t* X, uint32_t* Z, uint32_t q, const VV<V>& x, const VV<V>& z) {
    const uint32_t a = q * V;
    if (CODE == R_SWAPXZ) { vstore<V>(X + a, z); vstore<V>(Z + a, x); }
    else if (CODE == R_ZXORX) vstore<V>(Z + a, vxor<V>(z, x));
    else vstore<V>(X + a, vxor<V>(x, z));  // R_XXORZ
}

// Lanes take the applications of one op (distinct qubits, so no two lanes
// touch one row): unguarded batches of U per lane, then the remainder.
template <uint32_t CODE, int V>
__device__ __forceinline__ void gate2(uint32_t* X, uint32_t* Z, const uint32_t* P, uint32_t count, int lane) {
    constexpr int U = V == 4 ? 2 : 4;
    const uint2* P2 = reinterpret_cast<const uint2*>(P);
    uint32_t i = (uint32_t)lane;
    for (; i + 32u * (U - 1) < count; i += 32u * U) {
        uint2 q[U];
        VV<V> x0[U], x1[U], z0[U], z1[U];
#pragma unroll
        for (int t = 0; t < U; t++) q[t] = P2[i + 32u * t];
#pragma unroll
        for (int t = 0; t < U; t++) {
            x0[t] = vload<V>(X + q[t].x * V); x1[t] = vload<V>(X + q[t].y * V);
            z0[t] = vload<V>(Z + q[t].x * V); z1[t] = vload<V>(Z + q[t].y * V);
        }
#pragma unroll
        for (int t = 0; t < U; t++) rule2<CODE, V>(X, Z, q[t], x0[t], x1[t], z0[t], z1[t]);
    }
    for (; i < count; i += 32u) {
        const uint2 q = P2[i];
        rule2<CODE, V>(X, Z, q, vload<V>(X + q.x * V), vload<V>(X + q.y * V), vload<V>(Z + q.x * V),
                       vload<V>(Z + q.y * V));
    }
}

template <uint32_t CODE, int V>
__device__ __forceinline__ void gate1(uint32_t* X, uint32_t* Z, const uint32_t* P, uint32_t count, int lane) {
    constexpr int U = 4;
    uint32_t i = (uint32_t)lane;
    for (; i + 32u * (U - 1) < count; i += 32u * U) {
        uint32_t q[U];
        VV<V> x[U], z[U];
#pragma unroll
        for (int t = 0; t < U; t++) q[t] = P[i + 32u * t];
#pragma unroll
        for (int t = 0; t < U; t++) { x[t] = vload<V>(X + q[t] * V); z[t] = vload<V>(Z + q[t] * V); }
#pragma unroll
        for (int t = 0; t < U; t++) rule1<CODE, V>(X, Z, q[t], x[t], z[t]);
    }
    for (; i < count; i += 32u) {
        const uint32_t q = P[i];
        rule1<CODE, V>(X, Z, q, vload<V>(X + q * V), vload<V>(Z + q * V));
    }
}

// ring entry: V words in shared (RING_SMEM) or global memory
template <int V, bool RS> __device__ __forceinline__ VV<V> ring_load(const uint32_t* p) {
    if constexpr (RS) return vload<V>(p);
    VV<V> r;
    if constexpr (V == 4) { const uint4 t = __ldcg(reinterpret_cast<const uint4*>(p)); r.w[0] = t.x; r.w[1] = t.y; r.w[2] = t.z; r.w[3] = t.w; }
    else if constexpr (V == 2) { const uint2 t = __ldcg(reinterpret_cast<const uint2*>(p)); r.w[0] = t.x; r.w[1] = t.y; }
    else r.w[0] = __ldcg(p);
    return r;
}

}  // namespace

template <int V, bool RING_SMEM, int MAXW>
__global__ void __launch_bounds__(32 * (MAXW + 1), 1)
frame_col_kernel(const __grid_constant__ KParams kp, const __grid_constant__ ColParams cp) {
    extern __shared__ __align__(16) uint8_t smem8[];
    constexpr uint32_t K = COL_SLOTS;
    constexpr uint32_t T = 32u * V;  // shots per word column unit (the RNG tile)
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
                    if (seq >= K) mbar_wait_backoff(empty + s, ((seq / K) - 1u) & 1u);
                    bulk_load(slots + s * SB, cp.stream + (size_t)bi.x * 4, bi.y, full + s);
                }
            }
        }
    } else {
        // ---------------- consumers: one V-word column (T shots) per warp ----------------
        uint32_t* const X = reinterpret_cast<uint32_t*>(smem8 + K * SB + 2 * K * 8) + cnt_words +
                            (size_t)warp * cp.warp_words;
        uint32_t* const Z = X + (size_t)n * V;
        // record ring (V words per slot): after the frame, or (large circuits)
        // a per-warp region in global memory so more columns fit shared memory
        uint32_t* const ring = RING_SMEM ? Z + (size_t)n * V
                                         : kp.ring_global + ((size_t)blockIdx.x * NW + warp) * kp.num_slots * V;
        Sink<V> sk{RING_SMEM ? ring + (size_t)kp.num_slots * V : Z + (size_t)n * V, 0u};
        uint32_t* const wscr = sk.buf + 64 * V;
        uint32_t* const sl = kp.noise_scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * NZ_MAX_LIST;
        const bool b8 = cp.b8_out != nullptr;
        uint32_t seq = 0;
        for (int64_t p = 0; p < passes; p++) {
            const int64_t u = first + p * per_pass + warp;  // local column unit
            const bool live = u < cp.n_units;
            const uint32_t g = (uint32_t)(kp.tile_offset + (uint64_t)u);  // global RNG tile
            uint32_t tail[V];  // valid shots of each word
#pragma unroll
            for (int w = 0; w < V; w++) {
                const int64_t rem = kp.num_shots - (u * T + 32 * w);
                tail[w] = rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
            }
            sk.flushed = 0u;
            if (live) {
                // ---- FrameBatch.__init__: x = 0, z = coin rows 0..n-1 (frame_sim.py:36-39) ----
                const uint32_t k1 = coin_k1((uint32_t)n);
                for (uint32_t kb = 0; kb < k1; kb += 32) {
                    const uint32_t k = kb + (uint32_t)lane;
                    if (k >= k1 || !coin_group_live(k, 0u, (uint32_t)n)) continue;
                    const uint32_t live = init_live_rows(kp, k, (uint32_t)n);
                    uint32_t o[V][4];
#pragma unroll
                    for (int w = 0; w < V; w++) {
                        o[w][0] = o[w][1] = o[w][2] = o[w][3] = 0u;
                        if (live) coin_group<V>(kp, k, (uint32_t)w, g, u, 0u, (uint32_t)n, o[w]);
                    }
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        const uint32_t e = coin_row0(k) + 32u * r;
                        if (e >= (uint32_t)n) continue;
                        VV<V> zv;
#pragma unroll
                        for (int w = 0; w < V; w++) zv.w[w] = ((live >> r) & 1u) ? o[w][r] : 0u;
                        const uint32_t row = __ldg(kp.row_of + e);  // qubit e's frame row
                        vstore<V>(X + row * V, vzero<V>());
                        vstore<V>(Z + row * V, zv);
                    }
                }
                for (int i = lane; i < kp.num_obs; i += 32) vstore<V>(ring + (size_t)i * V, vzero<V>());
                __syncwarp();
            }
            for (int32_t bi = 0; bi < nblk; bi++, seq++) {
                const uint32_t s = seq % K;
                mbar_wait_sleep(full + s, (seq / K) & 1u);
                const uint32_t* const hb = reinterpret_cast<const uint32_t*>(slots + s * SB);
                if (live) {
                    const uint4 h4 = *reinterpret_cast<const uint4*>(hb);
                    const uint32_t kcf = h4.x, count = h4.y, oa = h4.z, ob = h4.w;
                    const uint32_t kind = kcf & 0xFFu, code = (kcf >> 8) & 0xFFu, flags = kcf >> 16;
                    const uint32_t hw = COL_HEAD_WORDS + (kind == K_NOISE ? COL_NP_WORDS : 0u);
                    const uint32_t* const P = hb + hw;  // every block is staged (build_col_stream)
                    switch (kind) {
                    case K_GATE:
                        switch (code) {
                            case R_SWAPXZ: gate1<R_SWAPXZ, V>(X, Z, P, count, lane); break;
                            case R_ZXORX: gate1<R_ZXORX, V>(X, Z, P, count, lane); break;
                            case R_XXORZ: gate1<R_XXORZ, V>(X, Z, P, count, lane); break;
                            case R_CX: gate2<R_CX, V>(X, Z, P, count, lane); break;
                            case R_CZ: gate2<R_CZ, V>(X, Z, P, count, lane); break;
                            case R_CY: gate2<R_CY, V>(X, Z, P, count, lane); break;
                            default: gate2<R_SWAP, V>(X, Z, P, count, lane); break;
                        }
                        break;
                    case K_M: case K_MR: case K_R: {
                        // lanes take coin groups: V Philox blocks = four coin rows
                        // 32 apart, so a warp pass covers 128 consecutive rows
                        const uint32_t lo = ob, hi = ob + (kind == K_MR ? 2u : 1u) * count;
                        const uint32_t k1 = coin_k1(hi);
                        const bool emit = cp.records != 0;
                        for (uint32_t kb = coin_k0(lo); kb < k1; kb += 32) {
                            const uint32_t k = kb + (uint32_t)lane;
                            const bool kl = k < k1 && coin_group_live(k, lo, hi);
                            uint2 qsv[4];
                            uint32_t live = 0u;
#pragma unroll
                            for (int r = 0; r < 4; r++) {
                                const uint32_t e = coin_row0(k) + 32u * r;
                                qsv[r] = make_uint2(0u, NO_SLOT);
                                if (!kl || e < lo || e >= hi) continue;
                                const uint32_t rel = e - lo;
                                if (kind == K_R) qsv[r].x = P[rel];
                                else if (kind == K_M || (rel & 1u))
                                    qsv[r] = reinterpret_cast<const uint2*>(P)[kind == K_MR ? rel >> 1 : rel];
                                else continue;
                                if (!(qsv[r].x & COIN_DEAD)) live |= 1u << r;  // dead rows: z never read
                                qsv[r].x &= ~COIN_DEAD;
                            }
                            uint32_t o[V][4];
#pragma unroll
                            for (int w = 0; w < V; w++) {
                                o[w][0] = o[w][1] = o[w][2] = o[w][3] = 0u;
                                if (live) coin_group<V>(kp, k, (uint32_t)w, g, u, lo, hi, o[w]);
                            }
#pragma unroll
                            for (int r = 0; r < 4; r++) {
                                const uint32_t e = coin_row0(k) + 32u * r;
                                const bool in = kl && e >= lo && e < hi;
                                const uint32_t rel = e - lo;
                                const bool rec = in && kind != K_R && (kind == K_M || (rel & 1u));
                                const uint32_t j = kind == K_MR ? rel >> 1 : rel;
                                VV<V> cv, xv = vzero<V>();
#pragma unroll
                                for (int w = 0; w < V; w++) cv.w[w] = ((live >> r) & 1u) ? o[w][r] : 0u;
                                if (in) {
                                    const uint32_t qv = qsv[r].x * V;
                                    if (kind == K_R) {
                                        vstore<V>(X + qv, vzero<V>());
                                        vstore<V>(Z + qv, cv);
                                    } else if (rec) {
                                        xv = vload<V>(X + qv);
                                        if (kp.do_dets && qsv[r].y != NO_SLOT) vstore<V>(ring + (size_t)qsv[r].y * V, xv);
                                        if (kind == K_M) {
                                            if ((live >> r) & 1u) vstore<V>(Z + qv, vxor<V>(vload<V>(Z + qv), cv));
                                        } else {
                                            vstore<V>(X + qv, vzero<V>());
                                            vstore<V>(Z + qv, cv);
                                        }
                                    }
                                }
                                if (emit) {
                                    if (b8) {
                                        sink_put<V>(cp, sk, rec, oa + j, xv, u, kp.num_shots, lane);
                                    } else if (rec) {
#pragma unroll
                                        for (int w = 0; w < V; w++)
                                            cp.rows_out[(int64_t)(oa + j) * cp.rows_stride + u * V + w] = xv.w[w];
                                    }
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
                                const uint32_t qv = P[j] * V;
                                const uint32_t* mrow = kp.masks + (int64_t)(oa + 2 * j) * kp.inject_words + u * V;
#pragma unroll
                                for (int w = 0; w < V; w++) {
                                    const uint32_t mx = __ldg(mrow + w), mz = __ldg(mrow + kp.inject_words + w);
                                    if (flags & F_DUP) {
                                        if (mx) atomicXor(X + qv + w, mx);
                                        if (mz) atomicXor(Z + qv + w, mz);
                                    } else {
                                        X[qv + w] ^= mx;
                                        Z[qv + w] ^= mz;
                                    }
                                }
                            }
                            break;
                        }
                        const NoiseParam np = *reinterpret_cast<const NoiseParam*>(hb + COL_HEAD_WORDS);
                        if (np.flags & NZ_NONE) break;
                        noise_op_warp(kp, np, ob, g, wscr, sl, lane, [&](uint32_t trial, uint32_t pick) {
                            const uint32_t app = trial / T, sh = trial % T;
                            const uint32_t wd = sh >> 5, bit = 1u << (sh & 31u);
                            uint32_t xm, zm;
                            pattern_of(code, pick, xm, zm);
                            const uint32_t q0 = P[app * ar] * V + wd;
                            if (xm & 1u) atomicXor(X + q0, bit);
                            if (zm & 1u) atomicXor(Z + q0, bit);
                            if (ar == 2) {
                                const uint32_t q1 = P[app * 2 + 1] * V + wd;
                                if (xm & 2u) atomicXor(X + q1, bit);
                                if (zm & 2u) atomicXor(Z + q1, bit);
                            }
                        });
                        break;
                    }
                    case K_DET: {
                        if (!kp.do_dets) break;
                        // iterations follow 32-column output blocks: lane = column & 31
                        const uint32_t cend = oa + count;
                        for (uint32_t B = oa >> 5; B * 32u < cend; B++) {
                            const uint32_t col = B * 32u + (uint32_t)lane;
                            const bool valid = col >= oa && col < cend;
                            const uint32_t i = col - oa;
                            VV<V> acc = vzero<V>();
                            if (valid) {
                                if (code == 2) {
                                    const uint2 sv = reinterpret_cast<const uint2*>(P)[i];
                                    if (sv.x != NO_SLOT) acc = ring_load<V, RING_SMEM>(ring + (size_t)sv.x * V);
                                    if (sv.y != NO_SLOT) acc = vxor<V>(acc, ring_load<V, RING_SMEM>(ring + (size_t)sv.y * V));
                                } else if (code) {
                                    for (uint32_t e = 0; e < code; e++) {
                                        const uint32_t sidx = P[i * code + e];
                                        if (sidx != NO_SLOT) acc = vxor<V>(acc, ring_load<V, RING_SMEM>(ring + (size_t)sidx * V));
                                    }
                                } else {
                                    const uint32_t e0 = P[i], e1 = P[i + 1];
                                    for (uint32_t e = e0; e < e1; e++) {
                                        const uint32_t sidx = P[count + 1 + e];
                                        if (sidx != NO_SLOT) acc = vxor<V>(acc, ring_load<V, RING_SMEM>(ring + (size_t)sidx * V));
                                    }
                                }
                            }
                            if (kp.counts != nullptr) {
                                uint32_t tot = 0u;
                                if (valid)
#pragma unroll
                                    for (int w = 0; w < V; w++) tot += __popc(acc.w[w] & tail[w]);
                                if (tot) {
                                    if (kp.counts_in_smem) atomicAdd(cnt + col, tot);
                                    else atomicAdd(kp.counts + col, (unsigned long long)tot);
                                }
                            } else if (b8) {
                                // columns of this block from earlier ops wait in the carry buffer
                                const bool whole = B * 32u >= oa && B * 32u + 32u <= cend;
                                const uint32_t bend = min(B * 32u + 32u, (uint32_t)cp.ncols_out);
#pragma unroll
                                for (int w = 0; w < V; w++) {
                                    uint32_t v = acc.w[w];
                                    if (!whole && !valid) v = sk.buf[w * 32 + lane];
                                    if (bend <= cend) store_block(cp, v, B, u * T + 32 * w, kp.num_shots, lane);
                                    else sk.buf[w * 32 + lane] = v;
                                }
                            } else if (valid) {
#pragma unroll
                                for (int w = 0; w < V; w++) cp.rows_out[(int64_t)col * cp.rows_stride + u * V + w] = acc.w[w];
                            }
                        }
                        break;
                    }
                    case K_OBS: {
                        if (!kp.do_dets) break;
                        VV<V> acc = vzero<V>();
                        for (uint32_t j = (uint32_t)lane; j < count; j += 32) {
                            const uint32_t sidx = P[j];
                            if (sidx != NO_SLOT) acc = vxor<V>(acc, ring_load<V, RING_SMEM>(ring + (size_t)sidx * V));
                        }
#pragma unroll
                        for (int w = 0; w < V; w++) acc.w[w] = __reduce_xor_sync(0xFFFFFFFFu, acc.w[w]);
                        if (lane == 0) vstore<V>(ring + (size_t)oa * V, vxor<V>(ring_load<V, RING_SMEM>(ring + (size_t)oa * V), acc));
                        break;
                    }
                    default: break;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
            }
            // measurement records: the last, partial block of columns
            if (live && b8 && cp.records && sk.flushed * 32u < (uint32_t)cp.ncols_out)
                sink_flush<V>(cp, sk, sk.flushed, u, kp.num_shots, lane);
        }
    }
    if (kp.counts_in_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < kp.num_cols; i += blockDim.x)
            if (cnt[i]) atomicAdd(kp.counts + i, (unsigned long long)cnt[i]);
    }
}

size_t col_warp_words(int num_qubits, int64_t num_slots, bool ring_smem, int V) {
    return ((size_t)V * (2 * (size_t)num_qubits + (ring_smem ? (size_t)num_slots : 0) + 64) + 32 * NZ_MAX_LIST + 3) &
           ~(size_t)3;
}

size_t col_smem_bytes(int nw, size_t warp_words, uint32_t slot_bytes, int64_t counts_words) {
    const size_t cw = counts_words > 0 ? (((size_t)counts_words + 3) & ~(size_t)3) : 0;
    return (size_t)COL_SLOTS * slot_bytes + 2 * COL_SLOTS * 8 + cw * 4 + (size_t)nw * warp_words * 4;
}

template <int V, bool RS>
static cudaError_t col_attr(size_t smem) {
    return cudaFuncSetAttribute(frame_col_kernel<V, RS, col_max_warps(V, RS)>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t set_frame_col_kernel_smem(size_t smem) {
    cudaError_t e;
    if ((e = col_attr<1, true>(smem)) != cudaSuccess) return e;
    if ((e = col_attr<1, false>(smem)) != cudaSuccess) return e;
    if ((e = col_attr<2, true>(smem)) != cudaSuccess) return e;
    if ((e = col_attr<2, false>(smem)) != cudaSuccess) return e;
    if ((e = col_attr<4, true>(smem)) != cudaSuccess) return e;
    return col_attr<4, false>(smem);
}

template <int V, bool RS>
static void col_launch(const KParams& kp, const ColParams& cp, int grid, size_t smem, cudaStream_t st) {
    frame_col_kernel<V, RS, col_max_warps(V, RS)><<<grid, 32 * (cp.nw + 1), smem, st>>>(kp, cp);
}

cudaError_t launch_frame_col_kernel(const KParams& kp, const ColParams& cp, int V, bool ring_smem, int grid,
                                    size_t smem, cudaStream_t stream) {
    switch (V * 2 + (ring_smem ? 1 : 0)) {
        case 3: col_launch<1, true>(kp, cp, grid, smem, stream); break;
        case 2: col_launch<1, false>(kp, cp, grid, smem, stream); break;
        case 5: col_launch<2, true>(kp, cp, grid, smem, stream); break;
        case 4: col_launch<2, false>(kp, cp, grid, smem, stream); break;
        case 9: col_launch<4, true>(kp, cp, grid, smem, stream); break;
        case 8: col_launch<4, false>(kp, cp, grid, smem, stream); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace pfs
