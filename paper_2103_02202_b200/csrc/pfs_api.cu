// C-ABI of libpfs.so (include/pfs.h): program handles, device upload, the
// sampling driver (chunked, double-buffered D2H pipeline for host outputs).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "pfs_internal.h"

using namespace pfs;

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(PFS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
    } while (0)

constexpr size_t kSmemBudget = 227 * 1024;  // B200 opt-in max dynamic shared memory / CTA

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t reserve(size_t count) {
        if (count <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) n = count;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};
}  // namespace

struct pfs_program {
    HostProgram hp;
    pfs_options opts{};
    LaunchCfg cfg{};   // frame_kernel (cooperative); cfg.W is the program's tile width
    LaunchCfg wcfg{};  // frame_warp_kernel (wcfg.kernel == 0: not eligible)
    int warp_desc_smem = 0;
    int device = -1;
    int num_sms = 0;
    size_t smem_optin = kSmemBudget;
    DevBuf<DOp> d_ops;
    DevBuf<uint32_t> d_targets, d_det_ptr, d_det_terms, d_ring;
    DevBuf<NoiseParam> d_noise;
    DevBuf<uint64_t> d_noise_tab;
    DevBuf<uint32_t> d_pregen, d_noise_off, d_noise_ch, d_init_dead, d_row_of;
    DevBuf<uint64_t> d_hits;
    DevBuf<uint32_t> d_ncnt;
    DevBuf<long long> d_clock;
    DevBuf<uint32_t> d_nscratch;
    DevBuf<uint32_t> d_rows[2];
    DevBuf<uint8_t> d_b8[2];
    DevBuf<uint32_t> d_coins, d_masks;
    DevBuf<uint8_t> d_ref;
    DevBuf<unsigned long long> d_counts;
    // column kernel (KERNEL_COL): op-block stream, block table, packed reference bits
    bool colk = false;
    // error-model detector sampler (KERNEL_DEM)
    bool demk = false;
    bool dem_global = false;  // output column words in global memory (too many for shared)
    bool dem_per_warp = false;  // dem_warp_kernel
    DemModel dem;
    DevBuf<uint32_t> d_comp_base, d_cols, d_items;
    DevBuf<unsigned long long> d_comp_words;
    int dem_grid = 0;
    bool col_ring_smem = true;
    int col_v = 1;      // words per lane (tile = 32 col_v shots)
    int col_nw = 0;
    size_t col_smem = 0;
    int col_grid = 0;
    ColStream cs;
    DevBuf<uint32_t> d_cstream;
    DevBuf<uint2> d_binfo;
    DevBuf<uint32_t> d_refw;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev[10] = {};
    // noise/frame pipeline: noise_kernel of sub-chunk i+1 on noise_stream while
    // frame_kernel of sub-chunk i runs; two hit-list buffers
    cudaStream_t noise_stream = nullptr;   // low priority
    cudaStream_t frame_stream = nullptr;   // high priority: frame CTAs claim freed SMs first
    cudaStream_t tr_stream = nullptr;      // low priority: per-sub-chunk transposes
    int pipe_default = 1;
    cudaEvent_t pev[7] = {};  // [0] entry, [1..2] noise done, [3..4] frame done, [5] frame end, [6] transposes end
    DevBuf<uint64_t> d_hits2;
    DevBuf<uint32_t> d_ncnt2;
    double last_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t last_launches = 0;
};

static bool desc_fits(const HostProgram& hp) { return hp.ops.size() * sizeof(DOp) <= (size_t)DESC_SMEM_MAX; }

// per-group hit counts, descriptor copy
static size_t fixed_smem(const HostProgram& hp, int groups) {
    return (size_t)hp.num_noise * 4 * groups + 16 + (desc_fits(hp) ? hp.ops.size() * sizeof(DOp) : 0);
}

// Cooperative-kernel groups per CTA (named barriers 1..kMaxGroups).
constexpr int kMaxGroups = 8;

// Warp-private kernel: a warp's word column (x/z per qubit, record ring, hit
// counts) must fit shared memory several times over; descriptors join it when
// they fit without costing a warp.
static void choose_warp_layout(pfs_program* pg) {
    const HostProgram& hp = pg->hp;
    const size_t budget = pg->smem_optin;
    const size_t per = warp_kernel_smem_per_warp(hp.num_qubits, hp.num_slots, hp.num_noise);
    const size_t desc = hp.ops.size() * sizeof(DOp);
    const int max_w = WARP_KERNEL_MAX_THREADS / 32;
    int nw_g = (int)std::min<size_t>(max_w, budget / per);
    int nw_s = desc <= budget ? (int)std::min<size_t>(max_w, (budget - desc) / per) : 0;
    pg->wcfg = LaunchCfg{};
    // opt-in (pfs_options.kernel = 2): measured slower than the cooperative
    // kernel on the d=25 headline circuit
    if (pg->opts.kernel != KERNEL_WARP || std::max(nw_g, nw_s) < 4) return;
    const bool ds = nw_s >= nw_g;
    const int nw = ds ? nw_s : nw_g;
    pg->warp_desc_smem = ds ? 1 : 0;
    pg->wcfg.kernel = KERNEL_WARP;
    pg->wcfg.threads = 32 * nw;
    pg->wcfg.groups = 1;
    pg->wcfg.ring_smem = true;
    pg->wcfg.smem_bytes = (ds ? desc : 0) + (size_t)nw * per;
}

// Column kernel: staged op blocks up to kColSlotCap bytes; every consumer warp
// holds 2n + slots + 64 words.  Chosen automatically when at least
// kColMinWarps word columns fit one CTA (or forced with options.kernel = 3).
constexpr uint32_t kColSlotCap = 16384;
constexpr int kColMinWarps = 4;
constexpr bool kColAuto = false;  // auto layout picks the column kernel
// noise/frame pipeline sub-chunks per launch (pfs_options.pipeline overrides):
// noise_kernel of sub-chunk i+1 (16 KB shared, 8 warps) runs in the room a
// 640-thread frame CTA leaves on its SM while frame_kernel works on sub-chunk i
constexpr int kPipeChunks = 6;
constexpr int kPipeFrameThreads = 640;
constexpr int DEM_WARPS_HOST = 16;  // dem_kernel's warps (DEM_WARPS)

static uint32_t col_max_block_bytes(const HostProgram& hp) {
    uint32_t mx = 16;
    for (const DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF, code = (o.kcf >> 8) & 0xFF;
        uint64_t w = COL_HEAD_WORDS;
        switch (kind) {
            case K_GATE: w += (uint64_t)o.count * (code >= R_CX ? 2 : 1); break;
            case K_M: case K_MR: w += 2ull * o.count; break;
            case K_R: case K_OBS: w += o.count; break;
            case K_NOISE: w += COL_NP_WORDS + (uint64_t)o.count * (code == CH_DEP2 ? 2 : 1); break;
            case K_DET:
                w += code ? (uint64_t)o.count * code
                          : (uint64_t)o.count + 1 + (hp.det_ptr[o.a + o.count] - hp.det_ptr[o.a]);
                break;
            default: break;
        }
        const uint64_t b = (w * 4 + 15) & ~15ull;
        if (b > kColSlotCap) return 0;  // an op too large to stage: not eligible
        mx = std::max<uint32_t>(mx, (uint32_t)b);
    }
    return mx;
}

static bool choose_col_layout(pfs_program* pg) {
    const HostProgram& hp = pg->hp;
    const pfs_options& o = pg->opts;
    pg->colk = false;
    if (o.kernel != 0 && o.kernel != KERNEL_COL) return false;
    if (o.kernel == 0 && !kColAuto) return false;
    if (o.words_per_tile != 0 && o.words_per_tile != 1 && o.words_per_tile != 2 && o.words_per_tile != 4)
        return false;
    const uint32_t sb = col_max_block_bytes(hp);
    if (sb == 0) return false;
    // candidates (V words per lane, record ring in shared or global memory):
    // most shots in flight per SM (columns x 32 V), preferring wider lanes (fewer
    // instructions per shot) and a shared-memory ring on ties
    int best_nw = 0, best_v = 1;
    bool best_rs = true;
    int64_t best_score = -1;
    for (int V = 4; V >= 1; V >>= 1) {
        if (o.words_per_tile > 0 && V != o.words_per_tile) continue;
        for (int rs = 1; rs >= 0; rs--) {
            if (o.ring_in_smem == 0 && rs) continue;
            if (o.ring_in_smem == 1 && !rs) continue;
            const size_t ww = col_warp_words(hp.num_qubits, std::max<int64_t>(hp.num_slots, 1), rs != 0, V);
            const size_t fixed = col_smem_bytes(0, ww, sb, 0);
            if (fixed >= pg->smem_optin) continue;
            int nw = (int)std::min<size_t>(col_max_warps(V, rs != 0), (pg->smem_optin - fixed) / (ww * 4));
            if (o.threads > 0) nw = std::min(nw, std::max(1, o.threads / 32 - 1));
            if (nw < 1) continue;
            // warps keep latency hidden: below kColMinWarps a column counts half
            const int64_t eff = nw >= kColMinWarps ? nw : nw / 2;
            const int64_t score = eff * 32 * V * 16 + V * 2 + rs;
            if (score > best_score) { best_score = score; best_nw = nw; best_v = V; best_rs = rs != 0; }
        }
    }
    if (best_nw < (o.kernel == KERNEL_COL ? 1 : kColMinWarps)) return false;
    pg->colk = true;
    pg->col_nw = best_nw;
    pg->col_v = best_v;
    pg->col_ring_smem = best_rs;
    pg->col_smem = col_smem_bytes(best_nw, col_warp_words(hp.num_qubits, std::max<int64_t>(hp.num_slots, 1), best_rs, best_v),
                                  sb, 0);
    return true;
}

static void choose_layout(pfs_program* pg) {
    const HostProgram& hp = pg->hp;
    pfs_options o = pg->opts;
    if (pg->opts.kernel == KERNEL_DEM) {
        // error-model sampler: RNG tiles of one word (32 shots), no frame
        pg->demk = true;
        pg->wcfg = LaunchCfg{};
        pg->cfg = LaunchCfg{};
        pg->cfg.W = 1;
        pg->cfg.groups = 1;
        pg->cfg.threads = 32 * DEM_WARPS_HOST;
        pg->cfg.smem_bytes = dem_smem_bytes(DEM_WARPS_HOST, hp.num_cols, false);
        if (pg->cfg.smem_bytes > kSmemBudget) {  // d=100: a million columns
            pg->dem_global = true;
            pg->cfg.smem_bytes = dem_smem_bytes(DEM_WARPS_HOST, 0, false);
        } else if (dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, true) <= 96 * 1024) {
            pg->dem_per_warp = true;  // small circuits: a tile per warp
            pg->cfg.smem_bytes = dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, false);
        }
        pg->cfg.kernel = 0;
        return;
    }
    if (choose_col_layout(pg)) {
        // the program's tile is one word: RNG counters per 32-shot column
        pg->wcfg = LaunchCfg{};
        pg->cfg = LaunchCfg{};
        pg->cfg.W = pg->col_v;
        pg->cfg.groups = 1;
        pg->cfg.threads = 32 * (pg->col_nw + 1);
        pg->cfg.ring_smem = pg->col_ring_smem;
        pg->cfg.smem_bytes = pg->col_smem;
        pg->cfg.kernel = 0;
        return;
    }
    choose_warp_layout(pg);
    // the warp-private kernel takes 8-word tiles (hit lists shared by 8 warps)
    // unless the caller fixes W; the cooperative kernel then uses the same W
    if (pg->wcfg.kernel && o.words_per_tile <= 0) o.words_per_tile = 8;
    const size_t budget = pg->smem_optin;
    auto frame = [&](int W) { return frame_smem_bytes(hp.num_qubits, W); };
    auto ring = [&](int W) { return (size_t)hp.num_slots * W * 4; };
    auto need = [&](int W, int G, bool rs) {
        return G * (frame(W) + (rs ? ring(W) : 0)) + fixed_smem(hp, G);
    };
    auto fits = [&](int W, int G, bool rs) { return need(W, G, rs) <= budget; };
    int W = 0, G = 1;
    bool rs = false;
    if (o.words_per_tile > 0) {
        W = o.words_per_tile;
        G = o.groups > 0 ? o.groups : (fits(W, 2, false) ? 2 : 1);
        if (pg->wcfg.kernel && !fits(W, G, false)) G = 1;
        if (o.ring_in_smem == 1) rs = true;
        else if (o.ring_in_smem == 0) rs = false;
        else rs = fits(W, G, true);
    } else {
        // candidates: (W, groups, ring placement); prefer more shots in flight
        // per SM (G*W), then two groups (latency overlap), then a shared-memory ring
        int best_score = -1;
        for (int g = 1; g <= 2; g++) {
            if (o.groups > 0 && g != o.groups) continue;
            for (int w = 32; w >= 1; w >>= 1) {
                for (int r = 1; r >= 0; r--) {
                    if (o.ring_in_smem == 0 && r) continue;
                    if (o.ring_in_smem == 1 && !r) continue;
                    if (!fits(w, g, r)) continue;
                    const int score = (g * w) * 4 + (g == 2 ? 2 : 0) + r;
                    if (score > best_score) { best_score = score; W = w; G = g; rs = r; }
                }
            }
        }
    }
    G = std::min(G, kMaxGroups);
    pg->cfg.W = W;
    pg->cfg.groups = G;
    pg->cfg.ring_smem = rs;
    pg->cfg.smem_bytes = W > 0 ? need(W, G, rs) : 0;
    // default threads: all 768 without sampled noise; with it, 640 so that a
    // noise_kernel CTA fits beside the frame CTA (pipelined launch_tiles)
    // (measured: d=25, two groups, 12.46 -> 11.83 ms per 2^20 shots; a one-group
    // layout loses more frame-kernel speed with 640 threads than it hides:
    // d=100 80.8 -> 87.1 ms, so it keeps 768 threads and no pipeline)
    const bool pipelined = hp.num_noise > 0 && (o.pipeline > 1 || (o.pipeline == 0 && G >= 2));
    pg->pipe_default = pipelined ? kPipeChunks : 1;
    int threads = o.threads > 0 ? std::min(o.threads, FRAME_MAX_THREADS)
                                : (pipelined ? kPipeFrameThreads : FRAME_MAX_THREADS);
    threads = (threads / (32 * G)) * 32 * G;  // whole warps per group
    pg->cfg.threads = threads;
    pg->cfg.kernel = KERNEL_COOP;
    if (pg->wcfg.kernel) {
        pg->wcfg.W = W;
        if (!fits(W, G, rs)) pg->cfg.kernel = 0;  // counts mode runs on the warp kernel too
    }
}

extern "C" {

int pfs_version(void) { return 1; }

int pfs_measure_smem_bandwidth(int device, double* gbs) {
    if (!gbs) return fail(PFS_E_INVALID, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(PFS_E_NODEVICE, "no CUDA device available");
    CUDA_TRY(smem_probe(device, gbs));
    return PFS_OK;
}
const char* pfs_last_error(void) { return g_last_error.c_str(); }

int pfs_program_create(const pfs_instr* instrs, int64_t n_instrs, const int32_t* targets,
                       int64_t n_targets, const double* noise_p, int64_t n_noise,
                       const int64_t* det_ptr, const int64_t* det_idx, int64_t n_columns,
                       int64_t n_observables, int32_t num_qubits, int64_t num_measurements,
                       int64_t num_coin_rows, int64_t num_noise_rows,
                       const pfs_options* options_or_null, pfs_program** out) {
    if (!out) return fail(PFS_E_INVALID, "out is null");
    *out = nullptr;
    pfs_program* pg = new (std::nothrow) pfs_program();
    if (!pg) return fail(PFS_E_NOMEM, "out of host memory");
    if (options_or_null) pg->opts = *options_or_null;
    try {
        pg->hp = compile_program(instrs, n_instrs, targets, n_targets, noise_p, n_noise, det_ptr,
                                 det_idx, n_columns, n_observables, num_qubits, num_measurements,
                                 num_coin_rows, num_noise_rows);
    } catch (const std::invalid_argument& e) {
        delete pg;
        return fail(PFS_E_INVALID, e.what());
    } catch (const std::bad_alloc&) {
        delete pg;
        return fail(PFS_E_NOMEM, "out of host memory");
    }
    choose_layout(pg);
    if (pg->opts.schedule_only && pg->cfg.W < 1) pg->cfg.W = pg->opts.words_per_tile > 0 ? pg->opts.words_per_tile : 1;
    if (pg->demk) {
        try {
            pg->dem = build_dem(instrs, n_instrs, targets, det_ptr, det_idx, n_columns, num_qubits,
                                num_measurements, n_noise);
        } catch (const std::invalid_argument& e) {
            delete pg;
            return fail(PFS_E_INVALID, e.what());
        }
        if (!pg->dem.coin_dependent.empty()) {
            const std::string why = pg->dem.coin_dependent;
            delete pg;
            return fail(PFS_E_INVALID, "error-model sampler: " + why + " (use the frame sampler)");
        }
        if (pg->cfg.smem_bytes > kSmemBudget) {
            delete pg;
            return fail(PFS_E_INVALID, "error-model sampler: too many output columns for one CTA");
        }
    }
    if (!pg->opts.schedule_only && !pg->wcfg.kernel && !pg->colk && !pg->demk &&
        (pg->cfg.W < 1 || pg->cfg.smem_bytes > kSmemBudget)) {
        delete pg;
        return fail(PFS_E_INVALID, "frame table of " + std::to_string(num_qubits) +
                                       " qubits does not fit one CTA's shared memory");
    }
    // mean hits per noise chunk: 2 measured fastest (fewer count draws, rare
    // duplicate-position redraws; counts above NZ_MAX_LIST ~1e-10 of chunks)
    const double th = pg->opts.noise_target_hits > 0 ? pg->opts.noise_target_hits : 2.0;
    try {
        // warp kernel: 8-byte x/z rows, 16 lanes per shared-memory wavefront
        permute_rows(pg->hp);
        reorder_for_banks(pg->hp, pg->wcfg.kernel ? 2 : pg->cfg.W);
        dedup_operands(pg->hp);
        build_noise_schedule(pg->hp, 32 * pg->cfg.W, th);
        if (pg->colk) pg->cs = build_col_stream(pg->hp, kColSlotCap);
        if (pg->demk) {  // every tile's noise chunks as (ordinal, chunk) work items
            pg->dem.items.clear();
            for (int64_t o = 0; o < pg->hp.num_noise; o++) {
                const NoiseParam& np = pg->hp.noise[o];
                if (np.flags & NZ_NONE) continue;
                for (uint32_t r = 0; r < np.nchunks; r++) { pg->dem.items.push_back((uint32_t)o); pg->dem.items.push_back(r); }
            }
        }
    } catch (const std::invalid_argument& e) {
        delete pg;
        return fail(PFS_E_INVALID, e.what());
    }
    *out = pg;
    return PFS_OK;
}

int pfs_program_info(const pfs_program* pg, pfs_info* o) {
    if (!pg || !o) return fail(PFS_E_INVALID, "null argument");
    std::memset(o, 0, sizeof(*o));
    const HostProgram& hp = pg->hp;
    o->num_qubits = hp.num_qubits;
    o->words_per_tile = pg->cfg.W;
    o->groups = pg->cfg.groups;
    o->kernel = pg->demk ? KERNEL_DEM : pg->colk ? KERNEL_COL : pg->wcfg.kernel ? KERNEL_WARP : KERNEL_COOP;
    o->warps_per_cta = pg->colk ? pg->col_nw : pg->wcfg.kernel ? pg->wcfg.threads / 32 : 0;
    o->tile_shots = 32 * pg->cfg.W;
    o->threads = pg->cfg.threads;
    o->ring_in_smem = pg->cfg.ring_smem ? 1 : 0;
    o->smem_bytes = (int32_t)pg->cfg.smem_bytes;
    if (pg->wcfg.kernel) {  // row-producing modes run the warp-private kernel
        o->threads = pg->wcfg.threads;
        o->ring_in_smem = 1;
        o->smem_bytes = (int32_t)pg->wcfg.smem_bytes;
        o->groups = 1;
    }
    o->num_measurements = hp.num_meas;
    o->num_columns = hp.num_cols;
    o->num_observables = hp.num_obs;
    o->num_ops = (int64_t)hp.ops.size();
    o->num_barriers = hp.num_barriers;
    o->num_slots = hp.num_slots;
    o->num_noise = hp.num_noise;
    o->bframe_bits = hp.bframe_bits;
    o->num_coin_rows = hp.num_coin_rows;
    o->num_noise_rows = hp.num_noise_rows;
    o->noise_tab_len = (int64_t)hp.noise_tab.size();
    o->hit_capacity = hp.hit_capacity;
    o->pregen_chunks = hp.pregen_chunks;
    return PFS_OK;
}

int pfs_program_noise_schedule(const pfs_program* pg, uint32_t* params, int64_t n_params,
                               uint64_t* tab, int64_t n_tab) {
    if (!pg) return fail(PFS_E_INVALID, "null argument");
    const HostProgram& hp = pg->hp;
    if (n_params != hp.num_noise * 12 || n_tab != (int64_t)hp.noise_tab.size())
        return fail(PFS_E_INVALID, "size mismatch");
    if (n_params && !params) return fail(PFS_E_INVALID, "null params");
    if (n_tab && !tab) return fail(PFS_E_INVALID, "null table");
    if (n_params) std::memcpy(params, hp.noise.data(), n_params * 4);
    if (n_tab) std::memcpy(tab, hp.noise_tab.data(), n_tab * 8);
    return PFS_OK;
}

int pfs_program_last_timing(const pfs_program* pg, double* ms, int n) {
    if (!pg || !ms) return fail(PFS_E_INVALID, "null argument");
    for (int i = 0; i < n && i < 6; i++) ms[i] = pg->last_ms[i];
    return PFS_OK;
}

int64_t pfs_program_last_launches(const pfs_program* pg) { return pg ? pg->last_launches : -1; }

void pfs_program_destroy(pfs_program* pg) {
    if (!pg) return;
    if (pg->device >= 0) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(pg->device);
        pg->d_ops.release(); pg->d_targets.release(); pg->d_det_ptr.release();
        pg->d_det_terms.release(); pg->d_ring.release(); pg->d_noise.release();
        pg->d_noise_tab.release(); pg->d_pregen.release(); pg->d_hits.release();
        pg->d_noise_off.release(); pg->d_noise_ch.release(); pg->d_ncnt.release(); pg->d_init_dead.release();
        pg->d_row_of.release();
        pg->d_nscratch.release(); pg->d_clock.release();
        for (int i = 0; i < 2; i++) { pg->d_rows[i].release(); pg->d_b8[i].release(); }
        pg->d_coins.release(); pg->d_masks.release(); pg->d_ref.release(); pg->d_counts.release();
        pg->d_cstream.release(); pg->d_binfo.release(); pg->d_refw.release();
        pg->d_comp_base.release(); pg->d_cols.release(); pg->d_items.release();
        pg->d_comp_words.release();
        pg->d_hits2.release(); pg->d_ncnt2.release();
        if (pg->copy_stream) cudaStreamDestroy(pg->copy_stream);
        if (pg->noise_stream) cudaStreamDestroy(pg->noise_stream);
        if (pg->frame_stream) cudaStreamDestroy(pg->frame_stream);
        if (pg->tr_stream) cudaStreamDestroy(pg->tr_stream);
        for (auto& e : pg->ev) if (e) cudaEventDestroy(e);
        for (auto& e : pg->pev) if (e) cudaEventDestroy(e);
        if (prev >= 0) cudaSetDevice(prev);
    }
    delete pg;
}

}  // extern "C"

template <typename T>
static cudaError_t upload(DevBuf<T>& b, const std::vector<T>& v) {
    cudaError_t e = b.reserve(v.size());
    if (e != cudaSuccess || v.empty()) return e;
    return cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

static int ensure_device(pfs_program* pg, int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(PFS_E_NODEVICE, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(PFS_E_INVALID, "bad device index");
    CUDA_TRY(cudaSetDevice(device));
    if (pg->device == device) return PFS_OK;
    if (pg->device >= 0) return fail(PFS_E_INVALID, "program is bound to another device");
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(PFS_E_NODEVICE, "libpfs is built for sm_100a (B200) only");
    pg->num_sms = prop.multiProcessorCount;
    pg->smem_optin = prop.sharedMemPerBlockOptin;
    if (pg->opts.schedule_only)
        return fail(PFS_E_INVALID, "schedule-only program");
    if (pg->demk ? pg->cfg.smem_bytes > pg->smem_optin : pg->colk ? pg->col_smem > pg->smem_optin
                 : pg->wcfg.kernel ? pg->wcfg.smem_bytes > pg->smem_optin
                                   : pg->cfg.smem_bytes > pg->smem_optin)
        return fail(PFS_E_INVALID, "frame tile exceeds this device's shared memory");
    const HostProgram& hp = pg->hp;
    CUDA_TRY(upload(pg->d_ops, hp.ops));
    CUDA_TRY(upload(pg->d_targets, hp.targets));
    CUDA_TRY(upload(pg->d_det_ptr, hp.det_ptr));
    CUDA_TRY(upload(pg->d_det_terms, hp.det_terms));
    CUDA_TRY(upload(pg->d_noise, hp.noise));
    CUDA_TRY(upload(pg->d_noise_tab, hp.noise_tab));
    CUDA_TRY(upload(pg->d_pregen, hp.pregen_ops));
    CUDA_TRY(upload(pg->d_noise_off, hp.noise_off));
    CUDA_TRY(upload(pg->d_noise_ch, hp.noise_ch));
    CUDA_TRY(upload(pg->d_init_dead, hp.init_dead));
    CUDA_TRY(upload(pg->d_row_of, hp.row_of));
    auto grid_of = [&](const LaunchCfg& c) {
        int per_sm = pg->opts.ctas_per_sm;
        if (per_sm <= 0) {
            size_t per = c.smem_bytes + 1024;
            per_sm = (int)std::max<size_t>(1, (prop.sharedMemPerMultiprocessor) / per);
            per_sm = std::min(per_sm, std::max(1, prop.maxThreadsPerMultiProcessor / c.threads));
        }
        return pg->num_sms * per_sm;
    };
    if (pg->cfg.kernel && pg->cfg.smem_bytes <= pg->smem_optin) {
        CUDA_TRY(set_frame_kernel_smem(pg->cfg));
        pg->cfg.grid = grid_of(pg->cfg);
    } else {
        pg->cfg.kernel = 0;
    }
    if (pg->wcfg.kernel) {
        CUDA_TRY(set_frame_warp_kernel_smem(pg->wcfg));
        pg->wcfg.grid = grid_of(pg->wcfg);
    }
    if (pg->demk) {
        CUDA_TRY(upload(pg->d_comp_base, pg->dem.comp_base));
        CUDA_TRY(upload(pg->d_cols, pg->dem.cols));
        CUDA_TRY(upload(pg->d_comp_words, pg->dem.comp_words));
        CUDA_TRY(upload(pg->d_items, pg->dem.items));
        CUDA_TRY(set_dem_kernel_smem(pg->smem_optin));
        int per_sm = pg->opts.ctas_per_sm;
        if (per_sm <= 0) {
            per_sm = (int)std::max<size_t>(1, prop.sharedMemPerMultiprocessor / (pg->cfg.smem_bytes + 1024));
            per_sm = std::min(per_sm, std::max(1, prop.maxThreadsPerMultiProcessor / (32 * DEM_WARPS_HOST)));
        }
        pg->dem_grid = pg->num_sms * per_sm;
    }
    if (pg->colk) {
        CUDA_TRY(upload(pg->d_cstream, pg->cs.words));
        std::vector<uint2> bi(pg->cs.n_blocks);
        for (int64_t i = 0; i < pg->cs.n_blocks; i++) bi[i] = make_uint2(pg->cs.binfo[2 * i], pg->cs.binfo[2 * i + 1]);
        CUDA_TRY(upload(pg->d_binfo, bi));
        CUDA_TRY(set_frame_col_kernel_smem(pg->smem_optin));
        int per_sm = pg->opts.ctas_per_sm;
        if (per_sm <= 0) {
            per_sm = (int)std::max<size_t>(1, prop.sharedMemPerMultiprocessor / (pg->col_smem + 1024));
            per_sm = std::min(per_sm, std::max(1, prop.maxThreadsPerMultiProcessor / (32 * (pg->col_nw + 1))));
        }
        pg->col_grid = pg->num_sms * per_sm;
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&pg->copy_stream, cudaStreamNonBlocking));
    {
        int least = 0, greatest = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        CUDA_TRY(cudaStreamCreateWithPriority(&pg->noise_stream, cudaStreamNonBlocking, least));
        CUDA_TRY(cudaStreamCreateWithPriority(&pg->tr_stream, cudaStreamNonBlocking, least));
        CUDA_TRY(cudaStreamCreateWithPriority(&pg->frame_stream, cudaStreamNonBlocking, greatest));
    }
    for (auto& e : pg->ev) CUDA_TRY(cudaEventCreate(&e));
    for (auto& e : pg->pev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pg->device = device;
    return PFS_OK;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Run nt tiles: noise_kernel (per-tile hit lists) then frame_kernel, in
// sub-chunks bounded by the hit-list buffer budget.  kp describes tile 0 of
// the range (tile_offset, output and inject pointers, num_shots).
// Shot-major b8 transposition of the launch's tile-major scratch, handed to a
// pipelined launch_tiles so that each sub-chunk's transpose overlaps the next
// sub-chunk's frame kernel (done = true when it was issued there).
struct TransposeJob {
    const uint32_t* rows = nullptr;  // [tile][row][W] scratch of tile 0 of the launch
    int64_t R = 0;
    const uint8_t* xor_bits = nullptr;
    uint8_t* dst = nullptr;          // row of shot 0 of the launch
    int64_t pitch = 0;
    bool done = false;
};

static int launch_tiles(pfs_program* pg, KParams kp, const LaunchCfg& cfg, int64_t nt, bool injected,
                        cudaStream_t st, bool time_noise, ColParams cp = ColParams{},
                        TransposeJob* tj = nullptr) {
    const HostProgram& hp = pg->hp;
    if (pg->demk) {
        // error-model sampler: noise hits XOR their output signatures, one launch
        DemParams dp{};
        dp.comp_base = pg->d_comp_base.p;
        dp.cols = pg->d_cols.p;
        dp.comp_words = pg->d_comp_words.p;
        dp.b8_out = cp.b8_out;
        dp.b8_pitch = cp.b8_pitch;
        dp.b8_bytes = cp.b8_bytes;
        dp.rows_out = cp.rows_out;
        dp.rows_stride = cp.rows_stride;
        dp.items = reinterpret_cast<const uint2*>(pg->d_items.p);
        dp.n_items = (int32_t)(pg->dem.items.size() / 2);
        dp.warps = DEM_WARPS_HOST;
        kp.n_tiles = nt;
        dp.per_warp = pg->dem_per_warp ? 1 : 0;
        const size_t smem = pg->dem_global ? dem_smem_bytes(DEM_WARPS_HOST, 0, false)
                          : pg->dem_per_warp ? dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, kp.counts_in_smem != 0)
                                             : dem_smem_bytes(DEM_WARPS_HOST, hp.num_cols, kp.counts_in_smem != 0);
        const int grid = (int)std::min<int64_t>(pg->dem_grid,
                                                pg->dem_per_warp ? (nt + DEM_WARPS_HOST - 1) / DEM_WARPS_HOST : nt);
        if (pg->dem_global) {
            // column words of every tile accumulate in the tile-major scratch
            // [tile][col] (kp.ev_out), transposed afterwards like the frame path
            if (!kp.ev_out) return fail(PFS_E_INVALID, "error-model sampler at this size: b8 / rows outputs only");
            if (kp.out_row_stride == 1)
                CUDA_TRY(cudaMemsetAsync(kp.ev_out, 0, (size_t)nt * hp.num_cols * 4, st));
            else
                CUDA_TRY(cudaMemset2DAsync(kp.ev_out, (size_t)kp.out_row_stride * 4, 0, (size_t)nt * 4,
                                           (size_t)hp.num_cols, st));
            dp.b8_out = nullptr;
            dp.rows_out = nullptr;
        }
        CUDA_TRY(launch_dem_kernel(kp, dp, pg->dem_global, grid, smem, st));
        pg->last_launches++;
        return PFS_OK;
    }
    if (pg->colk) {
        // column kernel: one launch, noise sampled inline, outputs written directly
        cp.stream = pg->d_cstream.p;
        cp.binfo = pg->d_binfo.p;
        cp.n_blocks = (int32_t)pg->cs.n_blocks;
        cp.slot_bytes = (int32_t)std::max<uint32_t>(pg->cs.slot_bytes, 16u);
        cp.nw = pg->col_nw;
        cp.warp_words = (int32_t)col_warp_words(hp.num_qubits, std::max<int64_t>(hp.num_slots, 1), pg->col_ring_smem,
                                                pg->col_v);
        if (!pg->col_ring_smem) {
            CUDA_TRY(pg->d_ring.reserve((size_t)std::max<int64_t>(hp.num_slots, 1) * pg->col_grid * cp.nw * pg->col_v));
            kp.ring_global = pg->d_ring.p;
        }
        cp.n_units = nt;
        kp.n_tiles = nt;
        const size_t smem = col_smem_bytes(cp.nw, cp.warp_words, cp.slot_bytes,
                                           kp.counts_in_smem ? hp.num_cols : 0);
        const int grid = (int)std::min<int64_t>(pg->col_grid, (nt + cp.nw - 1) / cp.nw);
        CUDA_TRY(launch_frame_col_kernel(kp, cp, pg->col_v, pg->col_ring_smem, grid, smem, st));
        pg->last_launches++;
        return PFS_OK;
    }
    const int W = cfg.W;
    const int64_t T = 32 * W;
    const bool pregen = !injected && !hp.pregen_ops.empty() && !(pg->opts.debug_skip & 2);
    int64_t sub = nt;
    // pipeline depth: sub-chunks per launch_tiles call (1 = noise, then frame)
    const int pipe = pg->opts.pipeline > 0 ? pg->opts.pipeline : cfg.kernel == KERNEL_COOP ? pg->pipe_default : 1;
    const int64_t per_wave = (int64_t)cfg.grid * std::max(cfg.groups, 1);
    const bool piped = pregen && !time_noise && pipe > 1 && nt >= 2 * per_wave;
    if (pregen) {
        const int64_t per_tile = hp.hit_capacity * 8 + hp.num_noise * 4;
        const int64_t budget = (int64_t)(piped ? 768 : 1536) << 20;
        sub = std::max<int64_t>(cfg.grid, budget / std::max<int64_t>(per_tile, 1));
        if (piped)  // whole waves of tiles per sub-chunk
            sub = std::min(sub, ((nt + pipe - 1) / pipe + per_wave - 1) / per_wave * per_wave);
        sub = std::min(sub, nt);
        CUDA_TRY(pg->d_hits.reserve((size_t)std::max<int64_t>(hp.hit_capacity, 1) * sub));
        CUDA_TRY(pg->d_ncnt.reserve((size_t)std::max<int64_t>(hp.num_noise, 1) * sub));
        if (piped) {
            CUDA_TRY(pg->d_hits2.reserve((size_t)std::max<int64_t>(hp.hit_capacity, 1) * sub));
            CUDA_TRY(pg->d_ncnt2.reserve((size_t)std::max<int64_t>(hp.num_noise, 1) * sub));
            CUDA_TRY(cudaEventRecord(pg->pev[0], st));  // everything before this call
            CUDA_TRY(cudaStreamWaitEvent(pg->noise_stream, pg->pev[0], 0));
            CUDA_TRY(cudaStreamWaitEvent(pg->frame_stream, pg->pev[0], 0));
            if (tj) CUDA_TRY(cudaStreamWaitEvent(pg->tr_stream, pg->pev[0], 0));
        }
    }
    cudaStream_t fst = piped ? pg->frame_stream : st;
    int64_t it = 0;
    for (int64_t s0 = 0; s0 < nt; s0 += sub, it++) {
        const int64_t ns = std::min(sub, nt - s0);
        KParams k2 = kp;
        k2.n_tiles = ns;
        k2.tile_offset = kp.tile_offset + (uint64_t)s0;
        k2.num_shots = std::min<int64_t>(kp.num_shots - s0 * T, ns * T);
        if (k2.rec_out) k2.rec_out += s0 * kp.out_tile_stride;
        if (k2.ev_out) k2.ev_out += s0 * kp.out_tile_stride;
        if (k2.coins) k2.coins += s0 * W;
        if (k2.masks) k2.masks += s0 * W;
        if (piped) {
            const int b = (int)(it & 1);
            cudaStream_t nst = pg->noise_stream;
            k2.hits_global = b ? pg->d_hits2.p : pg->d_hits.p;
            k2.ncnt_global = b ? pg->d_ncnt2.p : pg->d_ncnt.p;
            if (it >= 2) CUDA_TRY(cudaStreamWaitEvent(nst, pg->pev[3 + b], 0));  // buffer b consumed
            CUDA_TRY(cudaMemsetAsync(k2.ncnt_global, 0, (size_t)hp.num_noise * ns * 4, nst));
            CUDA_TRY(launch_noise_kernel(W, k2, ns, nst));
            CUDA_TRY(cudaEventRecord(pg->pev[1 + b], nst));
            CUDA_TRY(cudaStreamWaitEvent(fst, pg->pev[1 + b], 0));
            pg->last_launches++;
        } else if (pregen) {
            k2.hits_global = pg->d_hits.p;
            k2.ncnt_global = pg->d_ncnt.p;
            CUDA_TRY(cudaMemsetAsync(pg->d_ncnt.p, 0, (size_t)hp.num_noise * ns * 4, st));
            if (time_noise && s0 == 0) CUDA_TRY(cudaEventRecord(pg->ev[8], st));
            CUDA_TRY(launch_noise_kernel(W, k2, ns, st));
            if (time_noise && s0 == 0) CUDA_TRY(cudaEventRecord(pg->ev[9], st));
            pg->last_launches++;
        }
        LaunchCfg lc = cfg;
        k2.groups = cfg.groups;
        if (cfg.kernel == KERNEL_WARP) {
            const int64_t nw = cfg.threads / 32;
            lc.grid = (int)std::min<int64_t>(cfg.grid, (ns * W + nw - 1) / nw);
            CUDA_TRY(launch_frame_warp_kernel(lc, k2, fst));
        } else {
            lc.grid = (int)std::min<int64_t>(cfg.grid, (ns + cfg.groups - 1) / cfg.groups);
            CUDA_TRY(launch_frame_kernel(lc, k2, fst));
        }
        pg->last_launches++;
        if (piped) {
            CUDA_TRY(cudaEventRecord(pg->pev[3 + (it & 1)], fst));
            if (tj) {
                CUDA_TRY(cudaStreamWaitEvent(pg->tr_stream, pg->pev[3 + (it & 1)], 0));
                CUDA_TRY(launch_tiles_to_b8(tj->rows + s0 * kp.out_tile_stride, tj->R, W, ns, k2.num_shots,
                                            tj->xor_bits, tj->dst + s0 * T * tj->pitch, tj->pitch,
                                            pg->tr_stream, false));
                pg->last_launches++;
            }
        }
    }
    if (piped) {  // the caller's stream resumes after the last frame launch and transpose
        CUDA_TRY(cudaEventRecord(pg->pev[5], fst));
        CUDA_TRY(cudaStreamWaitEvent(st, pg->pev[5], 0));
        if (tj) {
            CUDA_TRY(cudaEventRecord(pg->pev[6], pg->tr_stream));
            CUDA_TRY(cudaStreamWaitEvent(st, pg->pev[6], 0));
            tj->done = true;
        }
    }
    return PFS_OK;
}

extern "C" int pfs_run(pfs_program* pg, int device, uint64_t seed, uint64_t shot_offset,
                       int64_t num_shots, int mode, const uint8_t* ref_bits,
                       const uint32_t* inject_coins, const uint32_t* inject_noise,
                       int64_t inject_row_words, void* out, int64_t out_bytes,
                       int64_t out_pitch, void* stream_v) {
    if (!pg) return fail(PFS_E_INVALID, "program is null");
    if (num_shots < 1) return fail(PFS_E_INVALID, "num_shots must be >= 1");
    if (mode < PFS_MODE_FLIPS || mode > PFS_MODE_DETECTORS_ROWS) return fail(PFS_E_INVALID, "bad mode");
    if (!out) return fail(PFS_E_INVALID, "out is null");
    const HostProgram& hp = pg->hp;
    const int W = pg->cfg.W;
    const int64_t T = 32 * W;
    if (shot_offset % T) return fail(PFS_E_INVALID, "shot_offset must be a multiple of the tile size " + std::to_string(T));
    if ((inject_coins == nullptr) != (inject_noise == nullptr))
        return fail(PFS_E_INVALID, "injected mode needs both coin and noise-mask rows");
    const bool injected = inject_coins != nullptr;
    if (injected && inject_row_words < (num_shots + 31) / 32)
        return fail(PFS_E_INVALID, "inject_row_words smaller than ceil(num_shots/32)");
    if (mode == PFS_MODE_SAMPLES && !ref_bits && hp.num_meas > 0)
        return fail(PFS_E_INVALID, "SAMPLES mode needs the reference sample");
    const bool rows_meas = mode == PFS_MODE_FLIPS || mode == PFS_MODE_SAMPLES || mode == PFS_MODE_FLIPS_ROWS;
    const bool b8 = mode <= PFS_MODE_DETECTORS;
    const int64_t R = rows_meas ? hp.num_meas : hp.num_cols;
    const int64_t nbytes = (R + 7) / 8;
    if (out_pitch == 0) out_pitch = nbytes;
    if (b8 && out_pitch < nbytes) return fail(PFS_E_INVALID, "out_pitch smaller than ceil(R/8)");
    const int64_t used_words = (num_shots + 31) / 32;
    int64_t need;
    if (b8) need = (num_shots - 1) * out_pitch + nbytes;
    else if (mode == PFS_MODE_COUNTS) need = hp.num_cols * 8;
    else need = R * used_words * 4;
    if (out_bytes < need) return fail(PFS_E_INVALID, "output buffer too small: need " + std::to_string(need) + " bytes");

    if (pg->demk && injected)
        return fail(PFS_E_INVALID, "the error-model sampler draws its own noise (no injected masks)");
    if (pg->demk && pg->dem_global && mode == PFS_MODE_COUNTS)
        return fail(PFS_E_INVALID, "error-model sampler: counts need the output columns in shared memory");
    if (pg->demk && rows_meas)
        return fail(PFS_E_INVALID, "the error-model sampler produces detection events only (use the frame sampler "
                                   "for measurement records)");
    int rc = ensure_device(pg, device);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream_v;
    const bool dev_out = is_device_ptr(out);
    const bool timing = pg->opts.timing != 0;
    pg->last_launches = 0;
    for (double& m : pg->last_ms) m = 0;
    if (timing) CUDA_TRY(cudaEventRecord(pg->ev[0], st));

    // ---- inputs: injected rows and reference bits (H2D) ----
    const int64_t n_tiles_all = (num_shots + T - 1) / T;
    const int64_t words_all = n_tiles_all * W;
    if (injected) {
        // rows padded to whole tiles
        auto up_rows = [&](DevBuf<uint32_t>& b, const uint32_t* src, int64_t rows) -> cudaError_t {
            cudaError_t e = b.reserve((size_t)std::max<int64_t>(rows, 1) * words_all);
            if (e != cudaSuccess || rows == 0) return e;
            if (is_device_ptr(src)) {
                e = cudaMemsetAsync(b.p, 0, (size_t)rows * words_all * 4, st);
                if (e != cudaSuccess) return e;
                return cudaMemcpy2DAsync(b.p, words_all * 4, src, inject_row_words * 4, used_words * 4,
                                         rows, cudaMemcpyDeviceToDevice, st);
            }
            e = cudaMemsetAsync(b.p, 0, (size_t)rows * words_all * 4, st);
            if (e != cudaSuccess) return e;
            return cudaMemcpy2DAsync(b.p, words_all * 4, src, inject_row_words * 4, used_words * 4,
                                     rows, cudaMemcpyHostToDevice, st);
        };
        CUDA_TRY(up_rows(pg->d_coins, inject_coins, hp.num_coin_rows));
        CUDA_TRY(up_rows(pg->d_masks, inject_noise, hp.num_noise_rows));
    }
    const uint8_t* d_ref = nullptr;
    if (mode == PFS_MODE_SAMPLES && hp.num_meas > 0) {
        CUDA_TRY(pg->d_ref.reserve(hp.num_meas));
        CUDA_TRY(cudaMemcpyAsync(pg->d_ref.p, ref_bits, hp.num_meas,
                                 is_device_ptr(ref_bits) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        d_ref = pg->d_ref.p;
        if (pg->colk) {
            // reference bits packed LSB-first into words (XORed per 32-column block)
            std::vector<uint32_t> rw((hp.num_meas + 31) / 32, 0u);
            std::vector<uint8_t> rb(hp.num_meas);
            if (is_device_ptr(ref_bits)) CUDA_TRY(cudaMemcpy(rb.data(), ref_bits, hp.num_meas, cudaMemcpyDeviceToHost));
            else std::memcpy(rb.data(), ref_bits, hp.num_meas);
            for (int64_t m = 0; m < hp.num_meas; m++) if (rb[m] & 1) rw[m >> 5] |= 1u << (m & 31);
            CUDA_TRY(pg->d_refw.reserve(rw.size()));
            CUDA_TRY(cudaMemcpyAsync(pg->d_refw.p, rw.data(), rw.size() * 4, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaStreamSynchronize(st));
        }
    }
    if (timing) CUDA_TRY(cudaEventRecord(pg->ev[1], st));

    KParams kp{};
    kp.ops = pg->d_ops.p;
    kp.targets = pg->d_targets.p;
    kp.det_ptr = pg->d_det_ptr.p;
    kp.det_terms = pg->d_det_terms.p;
    kp.noise = pg->d_noise.p;
    kp.noise_tab = pg->d_noise_tab.p;
    kp.pregen_ops = pg->d_pregen.p;
    kp.hit_capacity = hp.hit_capacity;
    kp.num_noise = (int32_t)hp.num_noise;
    kp.num_pregen = (int32_t)hp.pregen_ops.size();
    kp.pregen_chunks = (int32_t)hp.pregen_chunks;
    kp.noise_off = pg->d_noise_off.p;
    kp.noise_ch = pg->d_noise_ch.p;
    kp.init_dead = pg->d_init_dead.p;
    kp.row_of = pg->d_row_of.p;
    kp.first_pregen = hp.first_pregen;
    kp.first_cap_base = hp.first_cap_base;

    kp.coins = injected ? pg->d_coins.p : nullptr;
    kp.masks = injected ? pg->d_masks.p : nullptr;
    kp.inject_words = words_all;
    kp.seed = seed;
    kp.n_ops = (int32_t)hp.ops.size();
    kp.num_qubits = hp.num_qubits;
    kp.num_slots = (int32_t)hp.num_slots;
    kp.num_obs = (int32_t)hp.num_obs;
    kp.num_cols = (int32_t)hp.num_cols;
    kp.do_dets = rows_meas ? 0 : 1;
    kp.debug_skip = pg->opts.debug_skip;
    // frame kernel: warp-private when eligible (counts mode keeps the cooperative
    // kernel's shared-memory counters when it has one)
    const bool coop_counts = mode == PFS_MODE_COUNTS && pg->cfg.kernel && pg->opts.kernel != KERNEL_WARP;
    LaunchCfg cfg = (!pg->wcfg.kernel || coop_counts) ? pg->cfg : pg->wcfg;
    const bool warpk = cfg.kernel == KERNEL_WARP;
    kp.desc_in_smem = warpk ? pg->warp_desc_smem : (desc_fits(hp) ? 1 : 0);
    CUDA_TRY(pg->d_nscratch.reserve(pg->demk ? (size_t)pg->dem_grid * 32 * DEM_WARPS_HOST * NZ_MAX_LIST
                                    : pg->colk ? (size_t)pg->col_grid * 32 * (pg->col_nw + 1) * NZ_MAX_LIST
                                               : (size_t)cfg.grid * cfg.threads * NZ_MAX_LIST));
    kp.noise_scratch = pg->d_nscratch.p;
    if (pg->opts.debug_skip & 64) {  // op-boundary clock trace of the first tile
        CUDA_TRY(pg->d_clock.reserve(hp.ops.size() * 9 + 1));
        kp.op_clock = pg->d_clock.p;
    }

    if (!warpk && !cfg.ring_smem && !pg->colk && !pg->demk) {
        CUDA_TRY(pg->d_ring.reserve((size_t)std::max<int64_t>(hp.num_slots, 1) * W * cfg.grid * cfg.groups));
        kp.ring_global = pg->d_ring.p;
    }

    if (mode == PFS_MODE_COUNTS) {
        unsigned long long* cptr;
        if (dev_out) cptr = (unsigned long long*)out;
        else { CUDA_TRY(pg->d_counts.reserve(std::max<int64_t>(hp.num_cols, 1))); cptr = pg->d_counts.p; }
        if (hp.num_cols > 0) CUDA_TRY(cudaMemsetAsync(cptr, 0, hp.num_cols * 8, st));
        kp.counts = cptr;
        const size_t extra = (size_t)hp.num_cols * 4;
        kp.counts_in_smem = (!warpk && cfg.smem_bytes + extra <= pg->smem_optin) ? 1 : 0;
        if (pg->demk) {
            kp.counts_in_smem = (pg->dem_per_warp ? dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, true)
                                                  : dem_smem_bytes(DEM_WARPS_HOST, hp.num_cols, true)) <= pg->smem_optin;
        } else if (pg->colk) {
            kp.counts_in_smem = col_smem_bytes(pg->col_nw, col_warp_words(hp.num_qubits, std::max<int64_t>(hp.num_slots, 1), pg->col_ring_smem, pg->col_v),
                                               std::max<uint32_t>(pg->cs.slot_bytes, 16u), hp.num_cols) <= pg->smem_optin;
        } else if (kp.counts_in_smem) {
            cfg.smem_bytes += extra;
            CUDA_TRY(set_frame_kernel_smem(cfg));
        }
        // per-CTA u32 counters: bound shots per launch so no counter can overflow
        const int64_t max_tiles = std::max<int64_t>(1, ((int64_t)1 << 30) / T) *
                                  (pg->demk ? pg->dem_grid : pg->colk ? pg->col_grid : cfg.grid);
        for (int64_t t0 = 0; t0 < n_tiles_all; t0 += max_tiles) {
            const int64_t nt = std::min(max_tiles, n_tiles_all - t0);
            kp.n_tiles = nt;
            kp.tile_offset = shot_offset / T + t0;
            kp.num_shots = std::min<int64_t>(num_shots - t0 * T, nt * T);
            if (injected) { kp.coins = pg->d_coins.p + t0 * W; kp.masks = pg->d_masks.p + t0 * W; }
            int rc2 = launch_tiles(pg, kp, cfg, nt, injected, st, false);
            if (rc2) return rc2;
        }
        if (timing) CUDA_TRY(cudaEventRecord(pg->ev[2], st));
        if (!dev_out && hp.num_cols > 0)
            CUDA_TRY(cudaMemcpyAsync(out, cptr, hp.num_cols * 8, cudaMemcpyDeviceToHost, st));
        if (timing) CUDA_TRY(cudaEventRecord(pg->ev[4], st));
        if (!dev_out || timing) CUDA_TRY(cudaStreamSynchronize(st));
        if (timing) {
            float a = 0, b = 0, c = 0;
            cudaEventElapsedTime(&a, pg->ev[1], pg->ev[2]);
            cudaEventElapsedTime(&b, pg->ev[0], pg->ev[1]);
            cudaEventElapsedTime(&c, pg->ev[0], pg->ev[4]);
            pg->last_ms[0] = a; pg->last_ms[2] = b; pg->last_ms[4] = c;
        }
        return PFS_OK;
    }

    // ---- row-producing modes ----
    // Device output: one pass straight into the caller's buffer when possible.
    // Host output: chunks of tiles, kernels on `st`, D2H on copy_stream, double-buffered.
    const int64_t dev_pitch = b8 ? ((nbytes + 31) / 32) * 32 : 0;
    int64_t chunk_tiles = n_tiles_all;
    if (!dev_out) {
        const bool fused = pg->colk || (pg->demk && !pg->dem_global);  // no tile-major scratch
        const int64_t bytes_per_tile = (fused && b8 ? 0 : R * W * 4) + (b8 ? T * dev_pitch : 0);
        const int64_t target = (int64_t)256 << 20;
        chunk_tiles = std::max<int64_t>(1, target / std::max<int64_t>(bytes_per_tile, 1));
        chunk_tiles = std::max<int64_t>(chunk_tiles, pg->demk ? (int64_t)pg->dem_grid * 2 * (pg->dem_per_warp ? DEM_WARPS_HOST : 1)
                                                   : pg->colk ? (int64_t)pg->col_grid * pg->col_nw
                                                                  : (int64_t)cfg.grid);  // keep every SM busy
        chunk_tiles = std::min(chunk_tiles, n_tiles_all);
    }
    const bool direct_rows = dev_out && !b8;  // *_ROWS into the caller's buffer
    const int n_chunks = (int)((n_tiles_all + chunk_tiles - 1) / chunk_tiles);
    const int nbuf = dev_out ? 1 : std::min(2, n_chunks);
    const int64_t chunk_words = chunk_tiles * W;
    for (int b = 0; b < nbuf; b++) {
        // (+ padding to whole 8-word groups: the word-major transpose reads
        // narrow tiles in groups of 8 words)
        if (!direct_rows && !((pg->colk || (pg->demk && !pg->dem_global)) && b8)) CUDA_TRY(pg->d_rows[b].reserve((size_t)std::max<int64_t>(R, 1) * ((chunk_words + 7) & ~7ll)));
        if (b8 && !dev_out) CUDA_TRY(pg->d_b8[b].reserve((size_t)chunk_tiles * T * dev_pitch));
    }
    if (timing) CUDA_TRY(cudaEventRecord(pg->ev[1], st));
    float frame_ms = 0, tr_ms = 0;
    for (int ci = 0; ci < n_chunks; ci++) {
        const int b = ci % nbuf;
        const int64_t t0 = (int64_t)ci * chunk_tiles;
        const int64_t nt = std::min(chunk_tiles, n_tiles_all - t0);
        const int64_t shots0 = t0 * T;
        const int64_t nshots = std::min<int64_t>(num_shots - shots0, nt * T);
        if (!dev_out && ci >= 2) CUDA_TRY(cudaStreamWaitEvent(st, pg->ev[6 + b], 0));  // buffer free
        uint32_t* rows = direct_rows ? (uint32_t*)out : pg->d_rows[b].p;
        const int64_t row_words = direct_rows ? used_words : chunk_words;
        // b8: tile-major scratch ([tile][row][W]; warp kernel [tile][W][row])
        kp.out_row_stride = b8 ? (warpk ? 1 : W) : row_words;
        kp.out_word_stride = (b8 && warpk) ? R : 1;
        kp.out_tile_stride = b8 ? R * W : W;
        kp.rec_out = rows_meas ? rows : nullptr;
        kp.ev_out = rows_meas ? nullptr : rows;
        kp.n_tiles = nt;
        kp.tile_offset = shot_offset / T + t0;
        kp.num_shots = nshots;
        if (injected) { kp.coins = pg->d_coins.p + t0 * W; kp.masks = pg->d_masks.p + t0 * W; }
        ColParams cpx{};
        if (pg->colk || pg->demk) {
            cpx.records = rows_meas ? 1 : 0;
            cpx.ncols_out = (int32_t)R;
            if (b8) {
                cpx.b8_out = dev_out ? (uint8_t*)out + shots0 * out_pitch : pg->d_b8[b].p;
                cpx.b8_pitch = dev_out ? out_pitch : dev_pitch;
                cpx.b8_bytes = nbytes;
                cpx.b8_aligned = ((reinterpret_cast<uintptr_t>(cpx.b8_out) | (uintptr_t)cpx.b8_pitch) & 3u) == 0;
                cpx.ref_words = mode == PFS_MODE_SAMPLES ? pg->d_refw.p : nullptr;
            } else {
                cpx.rows_out = rows;
                cpx.rows_stride = row_words;
            }
        }
        if (!pg->colk && !pg->demk && direct_rows && (used_words % W) != 0) {
            // the last tile would write past the caller's rows: stage through scratch
            CUDA_TRY(pg->d_rows[0].reserve((size_t)std::max<int64_t>(R, 1) * chunk_words));
            rows = pg->d_rows[0].p;
            kp.out_row_stride = chunk_words;
            kp.out_word_stride = 1;
            kp.out_tile_stride = W;
            kp.rec_out = rows_meas ? rows : nullptr;
            kp.ev_out = rows_meas ? nullptr : rows;
        }
        if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[2], st));
        TransposeJob tj;
        const bool wm = warpk || W == 1;
        const bool tj_ok = b8 && !pg->colk && !pg->demk && !wm && kp.out_row_stride == W;
        if (tj_ok) {
            tj.rows = rows;
            tj.R = R;
            tj.xor_bits = mode == PFS_MODE_SAMPLES ? d_ref : nullptr;
            tj.dst = dev_out ? (uint8_t*)out + shots0 * out_pitch : pg->d_b8[b].p;
            tj.pitch = dev_out ? out_pitch : dev_pitch;
        }
        {
            int rc2 = launch_tiles(pg, kp, cfg, nt, injected, st, timing && ci == 0, cpx, tj_ok ? &tj : nullptr);
            if (rc2) return rc2;
        }
        if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[3], st));
        if (b8 && (pg->colk || (pg->demk && !pg->dem_global))) {
            if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[5], st));
        } else if (b8 && tj.done) {
            if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[5], st));
        } else if (b8) {
            uint8_t* dst = dev_out ? (uint8_t*)out + shots0 * out_pitch : pg->d_b8[b].p;
            const int64_t pitch = dev_out ? out_pitch : dev_pitch;
            // word-major tiles narrower than 8 words are contiguous word columns:
            // transpose them as 8-word tiles (256-shot blocks per CTA)
            // one-word tiles ([tile][row][1] = [tile][1][row]) are word-major too:
            // transpose them as 8-word tiles, like the warp kernel's
            const int tw = (wm && W < 8) ? 8 : W;
            const int64_t ntw = (nt * W + tw - 1) / tw;
            CUDA_TRY(launch_tiles_to_b8(rows, R, tw, ntw, nshots,
                                        mode == PFS_MODE_SAMPLES ? d_ref : nullptr, dst, pitch, st, wm));
            pg->last_launches++;
            if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[5], st));
        } else if (direct_rows && rows != (uint32_t*)out) {
            CUDA_TRY(cudaMemcpy2DAsync(out, used_words * 4, rows, kp.out_row_stride * 4, used_words * 4, R,
                                       cudaMemcpyDeviceToDevice, st));
        }
        if (timing && ci == 0) {
            CUDA_TRY(cudaStreamSynchronize(st));
            cudaEventElapsedTime(&frame_ms, pg->ev[2], pg->ev[3]);
            if (!pg->colk && !pg->demk && !injected && !hp.pregen_ops.empty() && !(pg->opts.debug_skip & 2)) {
                float nz = 0;
                cudaEventElapsedTime(&nz, pg->ev[8], pg->ev[9]);
                pg->last_ms[5] = nz;
                frame_ms -= nz;  // [0] = frame kernel alone, [5] = noise kernel
            }
            if (b8) cudaEventElapsedTime(&tr_ms, pg->ev[3], pg->ev[5]);
        }
        if (!dev_out) {
            CUDA_TRY(cudaEventRecord(pg->ev[4], st));
            CUDA_TRY(cudaStreamWaitEvent(pg->copy_stream, pg->ev[4], 0));
            if (b8) {
                CUDA_TRY(cudaMemcpy2DAsync((uint8_t*)out + shots0 * out_pitch, out_pitch, pg->d_b8[b].p,
                                           dev_pitch, nbytes, nshots, cudaMemcpyDeviceToHost,
                                           pg->copy_stream));
            } else {
                const int64_t cw = (nshots + 31) / 32;
                CUDA_TRY(cudaMemcpy2DAsync((uint32_t*)out + shots0 / 32, used_words * 4, rows,
                                           chunk_words * 4, cw * 4, R, cudaMemcpyDeviceToHost,
                                           pg->copy_stream));
            }
            CUDA_TRY(cudaEventRecord(pg->ev[6 + b], pg->copy_stream));
        }
    }
    if (!dev_out) {
        CUDA_TRY(cudaStreamSynchronize(pg->copy_stream));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    if (timing) {
        CUDA_TRY(cudaEventRecord(pg->ev[4], st));
        CUDA_TRY(cudaStreamSynchronize(st));
        float h2d = 0, tot = 0;
        cudaEventElapsedTime(&h2d, pg->ev[0], pg->ev[1]);
        cudaEventElapsedTime(&tot, pg->ev[0], pg->ev[4]);
        pg->last_ms[0] = frame_ms;
        pg->last_ms[1] = tr_ms;
        pg->last_ms[2] = h2d;
        pg->last_ms[4] = tot;
    }
    return PFS_OK;
}

// detector_events (stabsim/io_formats.py:208-227) on already-sampled flips.
extern "C" int pfs_detector_events(int device, const uint8_t* flips_b8, int64_t num_shots,
                                   int64_t num_results, int64_t in_pitch, const int64_t* det_ptr,
                                   const int64_t* det_idx, int64_t num_dets, uint8_t* out_b8,
                                   int64_t out_bytes, int64_t out_pitch, void* stream_v) {
    if (num_shots < 0 || num_results < 0 || num_dets < 0) return fail(PFS_E_INVALID, "negative size");
    if (num_shots == 0 || num_dets == 0) return PFS_OK;
    if (!flips_b8 || !det_ptr || !out_b8) return fail(PFS_E_INVALID, "null argument");
    const int64_t nb_in = (num_results + 7) / 8, nb_out = (num_dets + 7) / 8;
    if (in_pitch == 0) in_pitch = nb_in;
    if (out_pitch == 0) out_pitch = nb_out;
    if (in_pitch < nb_in || out_pitch < nb_out) return fail(PFS_E_INVALID, "pitch too small");
    if (out_bytes < (num_shots - 1) * out_pitch + nb_out) return fail(PFS_E_INVALID, "output buffer too small");
    for (int64_t d = 0; d < num_dets; d++) {
        if (det_ptr[d + 1] < det_ptr[d]) return fail(PFS_E_INVALID, "det_ptr not monotone");
        for (int64_t e = det_ptr[d]; e < det_ptr[d + 1]; e++)
            if (det_idx[e] < 0 || det_idx[e] >= num_results)
                return fail(PFS_E_INVALID, "detector " + std::to_string(d) + " references measurement " +
                                               std::to_string(det_idx[e]) + ", have " + std::to_string(num_results));
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PFS_E_NODEVICE, "no CUDA device available");
    CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream_v;
    const int64_t words = (num_shots + 31) / 32;
    const int64_t nnz = det_ptr[num_dets];
    const bool in_dev = is_device_ptr(flips_b8), out_dev = is_device_ptr(out_b8);
    uint8_t *d_in = nullptr, *d_out = nullptr;
    uint32_t *d_rows = nullptr, *d_ev = nullptr;
    int64_t *d_ptr = nullptr, *d_idx = nullptr;
    auto cleanup = [&]() {
        if (!in_dev && d_in) cudaFree(d_in);
        if (!out_dev && d_out) cudaFree(d_out);
        cudaFree(d_rows); cudaFree(d_ev); cudaFree(d_ptr); cudaFree(d_idx);
    };
#define DE_TRY(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) { cleanup(); \
        return fail(PFS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); } } while (0)
    if (in_dev) d_in = const_cast<uint8_t*>(flips_b8);
    else {
        DE_TRY(cudaMalloc(&d_in, (size_t)num_shots * in_pitch));
        DE_TRY(cudaMemcpyAsync(d_in, flips_b8, (size_t)num_shots * in_pitch, cudaMemcpyHostToDevice, st));
    }
    if (out_dev) d_out = out_b8;
    else DE_TRY(cudaMalloc(&d_out, (size_t)num_shots * out_pitch));
    DE_TRY(cudaMalloc(&d_rows, (size_t)std::max<int64_t>(num_results, 1) * words * 4));
    DE_TRY(cudaMalloc(&d_ev, (size_t)num_dets * words * 4));
    DE_TRY(cudaMalloc(&d_ptr, (size_t)(num_dets + 1) * 8));
    DE_TRY(cudaMalloc(&d_idx, (size_t)std::max<int64_t>(nnz, 1) * 8));
    DE_TRY(cudaMemcpyAsync(d_ptr, det_ptr, (size_t)(num_dets + 1) * 8, cudaMemcpyHostToDevice, st));
    if (nnz) DE_TRY(cudaMemcpyAsync(d_idx, det_idx, (size_t)nnz * 8, cudaMemcpyHostToDevice, st));
    DE_TRY(launch_detector_events(d_in, in_pitch, num_shots, num_results, d_ptr, d_idx, num_dets, d_rows,
                                  d_ev, d_out, out_pitch, st));
    if (!out_dev)
        DE_TRY(cudaMemcpyAsync(out_b8, d_out, (size_t)(num_shots - 1) * out_pitch + nb_out, cudaMemcpyDeviceToHost, st));
    DE_TRY(cudaStreamSynchronize(st));
#undef DE_TRY
    cleanup();
    return PFS_OK;
}

// write_table (stabsim/io_formats.py:198-201) on the GPU for 01 / hits / r8.
extern "C" int pfs_write_format(int device, const uint8_t* b8, int64_t in_pitch, int64_t num_shots,
                                int64_t num_results, int fmt, uint8_t* out, int64_t out_capacity,
                                int64_t* out_len, void* stream_v) {
    if (!out_len) return fail(PFS_E_INVALID, "out_len is null");
    *out_len = 0;
    if (fmt != 0 && fmt != 2 && fmt != 3) return fail(PFS_E_INVALID, "device writers: fmt 0 (01), 2 (hits), 3 (r8)");
    if (num_shots < 0 || num_results < 0) return fail(PFS_E_INVALID, "negative size");
    const int64_t nb = (num_results + 7) / 8;
    if (in_pitch == 0) in_pitch = nb;
    if (in_pitch < nb) return fail(PFS_E_INVALID, "pitch too small");
    if (num_shots == 0) return PFS_OK;
    if (!b8) return fail(PFS_E_INVALID, "null input");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PFS_E_NODEVICE, "no CUDA device available");
    CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream_v;
    const bool in_dev = is_device_ptr(b8);
    const uint8_t* d_in = b8;
    uint8_t* tmp_in = nullptr;
    if (!in_dev) {
        CUDA_TRY(cudaMalloc(&tmp_in, (size_t)num_shots * in_pitch));
        CUDA_TRY(cudaMemcpyAsync(tmp_in, b8, (size_t)(num_shots - 1) * in_pitch + nb, cudaMemcpyHostToDevice, st));
        d_in = tmp_in;
    }
    int64_t len = 0;
    cudaError_t e = write_format(d_in, in_pitch, num_shots, num_results, fmt, nullptr, 0, &len, st);
    uint8_t* d_out = nullptr;
    if (e == cudaSuccess && out && out_capacity >= len && len > 0) {
        const bool out_dev = is_device_ptr(out);
        if (out_dev) d_out = out;
        else e = cudaMalloc(&d_out, (size_t)len);
        if (e == cudaSuccess) e = write_format(d_in, in_pitch, num_shots, num_results, fmt, d_out, len, &len, st);
        if (e == cudaSuccess && !out_dev) e = cudaMemcpyAsync(out, d_out, (size_t)len, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (!out_dev && d_out) cudaFree(d_out);
    }
    if (tmp_in) { cudaStreamSynchronize(st); cudaFree(tmp_in); }
    CUDA_TRY(e);
    *out_len = len;
    if (out && out_capacity < len) return fail(PFS_E_INVALID, "output buffer too small: need " + std::to_string(len) + " bytes");
    return PFS_OK;
}

// Profiling: the per-op clock64 trace recorded by the last pfs_run with
// options.debug_skip bit 6 (CTA 0, group 0, first tile).
extern "C" int pfs_program_op_clock(pfs_program* pg, long long* out, int64_t n) {
    if (!pg || !out) return fail(PFS_E_INVALID, "null argument");
    if (!pg->d_clock.p) return fail(PFS_E_INVALID, "no clock trace (set debug_skip bit 6)");
    const int64_t m = std::min<int64_t>(n, (int64_t)pg->hp.ops.size() * 9);
    CUDA_TRY(cudaMemcpy(out, pg->d_clock.p, m * sizeof(long long), cudaMemcpyDeviceToHost));
    return PFS_OK;
}

// Profiling: the device op list (kind|code|flags, count) for interpreting traces.
extern "C" int pfs_program_ops(const pfs_program* pg, uint32_t* out, int64_t n) {
    if (!pg || !out) return fail(PFS_E_INVALID, "null argument");
    const int64_t m = std::min<int64_t>(n, (int64_t)pg->hp.ops.size());
    for (int64_t i = 0; i < m; i++) { out[2 * i] = pg->hp.ops[i].kcf; out[2 * i + 1] = pg->hp.ops[i].count; }
    return PFS_OK;
}
