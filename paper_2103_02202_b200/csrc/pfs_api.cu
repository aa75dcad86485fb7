// C-ABI of libpfs.so (include/pfs.h): program handles, device upload, the
// sampling driver (sub-chunk pipeline of frame kernel and shot-major
// transposes; chunked, double-buffered D2H for host outputs).
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

// One compiled flavour of the program (PM_EVENTS or PM_RECORDS) and its
// device copies.
struct Flavour {
    HostProgram hp;
    LaunchCfg cfg{};
    bool desc_smem = false;
    DevBuf<DOp> ops;
    DevBuf<SOp> sops;
    DevBuf<uint32_t> arena;
    DevBuf<uint32_t> targets, det_ptr, det_terms, ring, init_dead, row_of, noise_ch, noise_rowb;
    DevBuf<NoiseParam> noise;
    DevBuf<unsigned long long> noise_tab;
    DevBuf<uint32_t> fused, hit_items;  // pre-sampled fused noise (noise_kernel)
    void release() {
        ops.release(); sops.release(); arena.release(); targets.release(); det_ptr.release(); det_terms.release(); ring.release();
        init_dead.release(); row_of.release(); noise_ch.release(); noise_rowb.release();
        noise.release(); noise_tab.release(); fused.release(); hit_items.release();
    }
};
}  // namespace

struct pfs_program {
    Flavour fl[2];  // [PM_EVENTS], [PM_RECORDS]
    pfs_options opts{};
    int device = -1;
    int num_sms = 0;
    size_t smem_optin = kSmemBudget;
    DevBuf<long long> d_clock;
    DevBuf<uint32_t> d_nscratch;
    DevBuf<uint32_t> d_rows[2];
    DevBuf<uint8_t> d_b8[2];
    DevBuf<uint32_t> d_coins, d_masks;
    DevBuf<uint8_t> d_ref;
    DevBuf<unsigned long long> d_counts;
    DevBuf<unsigned long long> d_hits;  // noise_kernel hit entries of one sub-chunk of tiles
    DevBuf<uint32_t> d_spans;           // their per-warp spans (uint2) and per-tile fill counters
    DevBuf<uint32_t> d_fill;
    int noise_grid = 0;
    // error-model detector sampler (KERNEL_DEM)
    bool demk = false;
    bool dem_global = false;    // output column words in global memory (too many for shared)
    bool dem_per_warp = false;  // dem_warp_kernel
    DemModel dem;
    DevBuf<uint32_t> d_comp_base, d_cols, d_items;
    DevBuf<unsigned long long> d_comp_words;
    int dem_grid = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev[10] = {};
    // sub-chunk pipeline: the frame kernel of sub-chunk i+1 (high priority)
    // runs while the shot-major transpose of sub-chunk i (low priority) drains
    cudaStream_t frame_stream = nullptr;
    cudaStream_t tr_stream = nullptr;
    int pipe_default = 1;
    cudaEvent_t pev[4] = {};  // [0] entry, [1] frame sub-chunk done, [2] frame end, [3] transposes end
    double last_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t last_launches = 0;
};

// Cooperative-kernel groups per CTA (named barriers 1..kMaxGroups).
constexpr int kMaxGroups = 8;
// sub-chunks per launch of the frame / transpose pipeline (pfs_options.pipeline overrides)
constexpr int kPipeChunks = 6;
constexpr int kPipeFrameThreads = FRAME_MAX_THREADS;
constexpr int DEM_WARPS_HOST = 16;  // dem_kernel's warps (DEM_WARPS)
constexpr double kStandaloneHits = 2.0;  // mean hits per noise chunk (standalone / error-model)
constexpr double kFusedHits = 2.0;       // mean hits per fused noise chunk (noise_kernel: count per chunk, then hit-parallel)
constexpr int64_t kHitBufBytes = (int64_t)256 << 20;  // hit lists of one sub-chunk of tiles

static bool desc_fits(const HostProgram& hp) {
    return hp.ops.size() * sizeof(SOp) <= (size_t)DESC_SMEM_MAX;
}

// per-warp noise scratch, descriptors + threshold tables (when they fit), alignment slack
static size_t fixed_smem(const HostProgram& hp) {
    return 16 + (size_t)(FRAME_MAX_THREADS / 32) * WSCR * 4 +
           (desc_fits(hp) ? hp.ops.size() * sizeof(SOp) : 0);
}

// Outputs of the kernels that write final layouts directly (dem_kernel).
struct OutParams {
    uint8_t* b8_out = nullptr;   // shot-major rows or null
    int64_t b8_pitch = 0;
    int64_t b8_bytes = 0;        // ceil(R / 8)
    uint32_t* rows_out = nullptr;  // *_ROWS modes: [R][rows_stride] words, or null
    int64_t rows_stride = 0;
};

static size_t flavour_smem(const HostProgram& hp, int W, int G, bool rs) {
    return G * (frame_smem_bytes(hp.num_qubits, W) + (rs ? (size_t)hp.num_slots * W * 4 : 0)) + fixed_smem(hp);
}

// Tile width W, groups G and ring placement, chosen on the event flavour (it
// has the ring); the record flavour runs the same tiles without one.  The
// threshold tables are not known yet (they depend on W): reserve room for them.
static void choose_layout(pfs_program* pg) {
    const HostProgram& hp = pg->fl[PM_EVENTS].hp;
    pfs_options o = pg->opts;
    LaunchCfg& cfg = pg->fl[PM_EVENTS].cfg;
    if (pg->opts.kernel == KERNEL_DEM) {
        // error-model sampler: RNG tiles of one word (32 shots), no frame
        pg->demk = true;
        cfg = LaunchCfg{};
        cfg.W = 1;
        cfg.groups = 1;
        cfg.threads = 32 * DEM_WARPS_HOST;
        cfg.smem_bytes = dem_smem_bytes(DEM_WARPS_HOST, hp.num_cols, false);
        if (cfg.smem_bytes > kSmemBudget) {  // d=100: a million columns
            pg->dem_global = true;
            cfg.smem_bytes = dem_smem_bytes(DEM_WARPS_HOST, 0, false);
        } else if (dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, true) <= 96 * 1024) {
            pg->dem_per_warp = true;  // small circuits: a tile per warp
            cfg.smem_bytes = dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, false);
        }
        cfg.kernel = 0;
        pg->fl[PM_RECORDS].cfg = cfg;
        return;
    }
    const size_t budget = pg->smem_optin - 2048;  // room for the threshold tables
    auto fits = [&](int W, int G, bool rs) { return flavour_smem(hp, W, G, rs) <= budget; };
    int W = 0, G = 1;
    bool rs = false;
    if (o.words_per_tile > 0) {
        W = o.words_per_tile;
        G = o.groups > 0 ? o.groups : (fits(W, 2, false) ? 2 : 1);
        if (o.ring_in_smem == 1) rs = true;
        else if (o.ring_in_smem == 0) rs = false;
        else rs = fits(W, G, true);
    } else {
        // candidates: (W, groups, ring placement); prefer more shots in flight
        // per SM (G*W), then a shared-memory ring, then two groups (latency overlap)
        int best_score = -1;
        for (int g = 1; g <= (o.groups > 0 ? o.groups : 2); g++) {
            if (o.groups > 0 && g != o.groups) continue;
            for (int w = 32; w >= 1; w >>= 1) {
                for (int r = 1; r >= 0; r--) {
                    if (o.ring_in_smem == 0 && r) continue;
                    if (o.ring_in_smem == 1 && !r) continue;
                    if (!fits(w, g, r)) continue;
                    const int score = (g * w) * 8 + r * 4 + (g == 2 ? 2 : 0);
                    if (score > best_score) { best_score = score; W = w; G = g; rs = r; }
                }
            }
        }
    }
    G = std::min(G, kMaxGroups);
    cfg.W = W;
    cfg.groups = G;
    cfg.ring_smem = rs;
    const bool pipelined = o.pipeline > 1 || (o.pipeline == 0 && G >= 2);
    pg->pipe_default = pipelined ? kPipeChunks : 1;
    int threads = o.threads > 0 ? std::min(o.threads, FRAME_MAX_THREADS)
                                : (pipelined ? kPipeFrameThreads : FRAME_MAX_THREADS);
    threads = (threads / (32 * G)) * 32 * G;  // whole warps per group
    cfg.threads = threads;
    cfg.kernel = KERNEL_COOP;
    pg->fl[PM_RECORDS].cfg = cfg;
    pg->fl[PM_RECORDS].cfg.ring_smem = true;  // no ring: nothing to place
}

extern "C" {

int pfs_version(void) { return 2; }

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
    if (pg->opts.kernel != 0 && pg->opts.kernel != KERNEL_COOP && pg->opts.kernel != KERNEL_DEM) {
        delete pg;
        return fail(PFS_E_INVALID, "options.kernel must be 0 (auto), 1 (frame sampler) or 4 (error-model sampler)");
    }
    const bool dem = pg->opts.kernel == KERNEL_DEM;
    try {
        for (int m = 0; m < (dem ? 1 : 2); m++)
            pg->fl[m].hp = compile_program(instrs, n_instrs, targets, n_targets, noise_p, n_noise, det_ptr,
                                           det_idx, n_columns, n_observables, num_qubits, num_measurements,
                                           num_coin_rows, num_noise_rows, m);
    } catch (const std::invalid_argument& e) {
        delete pg;
        return fail(PFS_E_INVALID, e.what());
    } catch (const std::bad_alloc&) {
        delete pg;
        return fail(PFS_E_NOMEM, "out of host memory");
    }
    choose_layout(pg);
    LaunchCfg& cfg = pg->fl[PM_EVENTS].cfg;
    if (pg->opts.schedule_only && cfg.W < 1) cfg.W = pg->opts.words_per_tile > 0 ? pg->opts.words_per_tile : 1;
    if (dem) {
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
        if (cfg.smem_bytes > kSmemBudget) {
            delete pg;
            return fail(PFS_E_INVALID, "error-model sampler: too many output columns for one CTA");
        }
    }
    if (!pg->opts.schedule_only && !dem &&
        (cfg.W < 1 || flavour_smem(pg->fl[PM_EVENTS].hp, cfg.W, cfg.groups, cfg.ring_smem) > kSmemBudget)) {
        delete pg;
        return fail(PFS_E_INVALID, "frame table of " + std::to_string(num_qubits) +
                                       " qubits does not fit one CTA's shared memory");
    }
    const double th = pg->opts.noise_target_hits > 0 ? pg->opts.noise_target_hits : kStandaloneHits;
    const double thf = pg->opts.fused_target_milli > 0 ? pg->opts.fused_target_milli / 1000.0 : kFusedHits;
    try {
        const int W = cfg.W;
        const int V = W >= 4 ? 4 : W;
        for (int m = 0; m < (dem ? 1 : 2); m++) {
            HostProgram& hp = pg->fl[m].hp;
            // the error-model kernel's chunks span whole 32-shot tiles
            build_noise_schedule(hp, 32 * W, dem ? 32 : 32 * V, th, dem ? th : thf);
            // row placement needs the warps' application ranges, hence the chunk
            // geometry; it rewrites every op's targets, so it runs before
            // identical operand blocks are shared
            permute_rows(hp, (dem || W >= 32) ? 1 : 128 / (W * 4),
                         dem ? 0 : cfg.threads / std::max(1, cfg.groups) / 32);
            dedup_operands(hp);
            if (!dem) {
                const int wpg = cfg.threads / std::max(1, cfg.groups) / 32;
                if (pg->opts.presample_noise >= 0) build_hit_lists(hp, 32 * W, wpg);
                lower_stream(hp, W, wpg);
            }
            Flavour& f = pg->fl[m];
            if (m == PM_RECORDS) f.cfg = cfg, f.cfg.ring_smem = true;
            f.desc_smem = desc_fits(hp);
            if (!dem) f.cfg.smem_bytes = flavour_smem(hp, W, cfg.groups, f.cfg.ring_smem && m == PM_EVENTS);
        }
        if (dem) {  // every tile's noise chunks as (ordinal, chunk) work items
            const HostProgram& hp = pg->fl[PM_EVENTS].hp;
            pg->dem.items.clear();
            for (int64_t o = 0; o < hp.num_noise; o++) {
                const NoiseParam& np = hp.noise[o];
                if (np.zone == NZONE_NONE) continue;
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
    const HostProgram& hp = pg->fl[PM_EVENTS].hp;
    const LaunchCfg& cfg = pg->fl[PM_EVENTS].cfg;
    o->num_qubits = hp.num_qubits;
    o->words_per_tile = cfg.W;
    o->groups = cfg.groups;
    o->kernel = pg->demk ? KERNEL_DEM : KERNEL_COOP;
    o->warps_per_cta = 0;
    o->tile_shots = 32 * cfg.W;
    o->threads = cfg.threads;
    o->ring_in_smem = cfg.ring_smem ? 1 : 0;
    o->smem_bytes = (int32_t)cfg.smem_bytes;
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
    o->live_coin_rows = hp.live_coin_rows;
    o->record_ops = pg->demk ? 0 : (int64_t)pg->fl[PM_RECORDS].hp.ops.size();
    int64_t fused = 0;
    for (uint32_t f : hp.noise_fused) fused += f ? 1 : 0;
    o->fused_noise = fused;
    return PFS_OK;
}

int pfs_program_noise_schedule(const pfs_program* pg, uint32_t* params, int64_t n_params,
                               uint64_t* tab, int64_t n_tab) {
    if (!pg) return fail(PFS_E_INVALID, "null argument");
    const HostProgram& hp = pg->fl[PM_EVENTS].hp;
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
        for (Flavour& f : pg->fl) f.release();
        pg->d_nscratch.release(); pg->d_clock.release();
        for (int i = 0; i < 2; i++) { pg->d_rows[i].release(); pg->d_b8[i].release(); }
        pg->d_coins.release(); pg->d_masks.release(); pg->d_ref.release(); pg->d_counts.release();
        pg->d_comp_base.release(); pg->d_cols.release(); pg->d_items.release();
        pg->d_comp_words.release();
        pg->d_hits.release(); pg->d_spans.release(); pg->d_fill.release();
        if (pg->copy_stream) cudaStreamDestroy(pg->copy_stream);
        if (pg->frame_stream) cudaStreamDestroy(pg->frame_stream);
        if (pg->tr_stream) cudaStreamDestroy(pg->tr_stream);
        for (auto& e : pg->ev) if (e) cudaEventDestroy(e);
        for (auto& e : pg->pev) if (e) cudaEventDestroy(e);
        if (prev >= 0) cudaSetDevice(prev);
    }
    delete pg;
}

}  // extern "C"

template <typename T, typename U>
static cudaError_t upload(DevBuf<T>& b, const std::vector<U>& v) {
    static_assert(sizeof(T) == sizeof(U), "element size");
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
    for (int m = 0; m < 2; m++) {
        Flavour& f = pg->fl[m];
        if (pg->demk && m == PM_RECORDS) break;
        if (f.cfg.smem_bytes > pg->smem_optin)
            return fail(PFS_E_INVALID, "frame tile exceeds this device's shared memory");
        const HostProgram& hp = f.hp;
        CUDA_TRY(upload(f.ops, hp.ops));
        CUDA_TRY(upload(f.sops, hp.sops));
        CUDA_TRY(upload(f.arena, hp.arena));
        CUDA_TRY(upload(f.targets, hp.targets));
        CUDA_TRY(upload(f.det_ptr, hp.det_ptr));
        CUDA_TRY(upload(f.det_terms, hp.det_terms));
        CUDA_TRY(upload(f.noise, hp.noise));
        CUDA_TRY(upload(f.noise_tab, hp.noise_tab));
        CUDA_TRY(upload(f.noise_ch, hp.noise_ch));
        CUDA_TRY(upload(f.noise_rowb, hp.noise_rowb));
        CUDA_TRY(upload(f.init_dead, hp.init_dead));
        CUDA_TRY(upload(f.row_of, hp.row_of));
        CUDA_TRY(upload(f.fused, hp.fused_info));
        CUDA_TRY(upload(f.hit_items, hp.hit_items));
        if (!pg->demk) {
            // the attribute is per kernel instance, shared by both flavours and
            // counts mode: allow the device maximum once
            LaunchCfg all = f.cfg;
            all.smem_bytes = pg->smem_optin;
            CUDA_TRY(set_frame_kernel_smem(all));
            int per_sm = pg->opts.ctas_per_sm;
            if (per_sm <= 0) {
                per_sm = (int)std::max<size_t>(1, prop.sharedMemPerMultiprocessor / (f.cfg.smem_bytes + 1024));
                per_sm = std::min(per_sm, std::max(1, prop.maxThreadsPerMultiProcessor / f.cfg.threads));
            }
            f.cfg.grid = pg->num_sms * per_sm;
        }
    }
    if (pg->demk) {
        CUDA_TRY(upload(pg->d_comp_base, pg->dem.comp_base));
        CUDA_TRY(upload(pg->d_cols, pg->dem.cols));
        CUDA_TRY(upload(pg->d_comp_words, pg->dem.comp_words));
        CUDA_TRY(upload(pg->d_items, pg->dem.items));
        CUDA_TRY(set_dem_kernel_smem(pg->smem_optin));
        int per_sm = pg->opts.ctas_per_sm;
        if (per_sm <= 0) {
            per_sm = (int)std::max<size_t>(1, prop.sharedMemPerMultiprocessor / (pg->fl[0].cfg.smem_bytes + 1024));
            per_sm = std::min(per_sm, std::max(1, prop.maxThreadsPerMultiProcessor / (32 * DEM_WARPS_HOST)));
        }
        pg->dem_grid = pg->num_sms * per_sm;
    }
    pg->noise_grid = pg->num_sms * std::max(1, prop.maxThreadsPerMultiProcessor / (NK_WARPS * 32));
    CUDA_TRY(cudaStreamCreateWithFlags(&pg->copy_stream, cudaStreamNonBlocking));
    {
        int least = 0, greatest = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
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

// Shot-major b8 transposition of a launch's tile-major scratch, handed to a
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

// Run nt tiles of flavour f.  kp describes tile 0 of the range (tile_offset,
// output and inject pointers, num_shots).  With a transpose job and a
// pipeline depth > 1 the tiles go in sub-chunks of whole waves: frame kernels
// on the high-priority stream, each sub-chunk's transpose on the low-priority
// one behind it.
static int launch_tiles(pfs_program* pg, const Flavour& f, KParams kp, const LaunchCfg& cfg, int64_t nt,
                        cudaStream_t st, bool serial, OutParams cp = OutParams{}, TransposeJob* tj = nullptr) {
    const HostProgram& hp = f.hp;
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
    const int W = cfg.W;
    const int64_t T = 32 * W;
    const int pipe = pg->opts.pipeline > 0 ? pg->opts.pipeline : pg->pipe_default;
    const int64_t per_wave = (int64_t)cfg.grid * std::max(cfg.groups, 1);
    const bool piped = tj != nullptr && !serial && pipe > 1 && nt >= 2 * per_wave;
    // pre-sampled fused noise: noise_kernel fills the hit lists of a sub-chunk
    // of tiles ahead of its frame kernel (same stream), lists bounded by kHitBufBytes
    const bool lists = !hp.hit_items.empty() && kp.masks == nullptr && !(pg->opts.debug_skip & 2);
    int64_t sub = nt;
    if (lists) {
        const int64_t cap_tiles = std::max<int64_t>(per_wave, kHitBufBytes / (hp.hit_block * 8) / per_wave * per_wave);
        sub = std::min(nt, cap_tiles);
        CUDA_TRY(pg->d_hits.reserve((size_t)sub * hp.hit_block));
        CUDA_TRY(pg->d_spans.reserve((size_t)sub * hp.num_noise * hp.list_warps * 2));
        CUDA_TRY(pg->d_fill.reserve((size_t)sub * 2));
        kp.fused = reinterpret_cast<const uint4*>(f.fused.p);
        kp.hit_items = reinterpret_cast<const uint2*>(f.hit_items.p);
        kp.hit_block = hp.hit_block;
        kp.list_warps = hp.list_warps;
        kp.n_items = (int32_t)(hp.hit_items.size() / 2);
    }
    if (piped) {
        sub = std::min(sub, ((nt + pipe - 1) / pipe + per_wave - 1) / per_wave * per_wave);  // whole waves per sub-chunk
        CUDA_TRY(cudaEventRecord(pg->pev[0], st));  // everything before this call
        CUDA_TRY(cudaStreamWaitEvent(pg->frame_stream, pg->pev[0], 0));
        CUDA_TRY(cudaStreamWaitEvent(pg->tr_stream, pg->pev[0], 0));
    }
    cudaStream_t fst = piped ? pg->frame_stream : st;
    for (int64_t s0 = 0; s0 < nt; s0 += sub) {
        const int64_t ns = std::min(sub, nt - s0);
        KParams k2 = kp;
        k2.n_tiles = ns;
        k2.tile_offset = kp.tile_offset + (uint64_t)s0;
        k2.num_shots = std::min<int64_t>(kp.num_shots - s0 * T, ns * T);
        if (k2.rec_out) k2.rec_out += s0 * kp.out_tile_stride;
        if (k2.ev_out) k2.ev_out += s0 * kp.out_tile_stride;
        if (k2.coins) k2.coins += s0 * W;
        if (k2.masks) k2.masks += s0 * W;
        LaunchCfg lc = cfg;
        k2.groups = cfg.groups;
        lc.grid = (int)std::min<int64_t>(cfg.grid, (ns + cfg.groups - 1) / cfg.groups);
        if (lists) {
            const bool tm = serial && pg->opts.timing;
            k2.hits_global = pg->d_hits.p;
            k2.spans_global = reinterpret_cast<uint2*>(pg->d_spans.p);
            k2.fill_global = pg->d_fill.p;
            if (tm) CUDA_TRY(cudaEventRecord(pg->ev[8], fst));
            CUDA_TRY(cudaMemsetAsync(pg->d_fill.p, 0, (size_t)ns * 8, fst));
            const int64_t items = ns * k2.n_items;
            const int ng = (int)std::min<int64_t>(pg->noise_grid, (items + NK_WARPS - 1) / NK_WARPS);
            CUDA_TRY(launch_noise_kernel(W, k2, ng, fst));
            pg->last_launches++;
            if (tm) {
                CUDA_TRY(cudaEventRecord(pg->ev[9], fst));
                CUDA_TRY(cudaEventSynchronize(pg->ev[9]));
                float ms = 0;
                cudaEventElapsedTime(&ms, pg->ev[8], pg->ev[9]);
                pg->last_ms[5] += ms;
            }
        }
        CUDA_TRY(launch_frame_kernel(lc, k2, fst));
        pg->last_launches++;
        if (piped) {
            CUDA_TRY(cudaEventRecord(pg->pev[1], fst));
            CUDA_TRY(cudaStreamWaitEvent(pg->tr_stream, pg->pev[1], 0));
            CUDA_TRY(launch_tiles_to_b8(tj->rows + s0 * kp.out_tile_stride, tj->R, W, ns, k2.num_shots,
                                        tj->xor_bits, tj->dst + s0 * T * tj->pitch, tj->pitch, pg->tr_stream, false));
            pg->last_launches++;
        }
    }
    if (piped) {  // the caller's stream resumes after the last frame launch and transpose
        CUDA_TRY(cudaEventRecord(pg->pev[2], fst));
        CUDA_TRY(cudaStreamWaitEvent(st, pg->pev[2], 0));
        CUDA_TRY(cudaEventRecord(pg->pev[3], pg->tr_stream));
        CUDA_TRY(cudaStreamWaitEvent(st, pg->pev[3], 0));
        tj->done = true;
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
    const bool rows_meas = mode == PFS_MODE_FLIPS || mode == PFS_MODE_SAMPLES || mode == PFS_MODE_FLIPS_ROWS;
    if (pg->demk && rows_meas)
        return fail(PFS_E_INVALID, "the error-model sampler produces detection events only (use the frame sampler "
                                   "for measurement records)");
    const Flavour& fl = pg->fl[rows_meas ? PM_RECORDS : PM_EVENTS];
    const HostProgram& hp = fl.hp;
    const int W = fl.cfg.W;
    const int64_t T = 32 * W;
    if (shot_offset % T) return fail(PFS_E_INVALID, "shot_offset must be a multiple of the tile size " + std::to_string(T));
    if (shot_offset / T + (uint64_t)((num_shots + T - 1) / T) < shot_offset / T)
        return fail(PFS_E_INVALID, "shot range overflows the 64-bit tile index");
    if ((inject_coins == nullptr) != (inject_noise == nullptr))
        return fail(PFS_E_INVALID, "injected mode needs both coin and noise-mask rows");
    const bool injected = inject_coins != nullptr;
    if (injected && inject_row_words < (num_shots + 31) / 32)
        return fail(PFS_E_INVALID, "inject_row_words smaller than ceil(num_shots/32)");
    if (mode == PFS_MODE_SAMPLES && !ref_bits && hp.num_meas > 0)
        return fail(PFS_E_INVALID, "SAMPLES mode needs the reference sample");
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
            e = cudaMemsetAsync(b.p, 0, (size_t)rows * words_all * 4, st);
            if (e != cudaSuccess) return e;
            return cudaMemcpy2DAsync(b.p, words_all * 4, src, inject_row_words * 4, used_words * 4, rows,
                                     is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
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
    }
    if (timing) CUDA_TRY(cudaEventRecord(pg->ev[1], st));

    KParams kp{};
    kp.ops = fl.ops.p;
    kp.sops = fl.sops.p;
    kp.arena = fl.arena.p;
    kp.first_span = hp.first_span;
    kp.all_presampled = hp.all_presampled ? 1 : 0;
    kp.targets = fl.targets.p;
    kp.det_ptr = fl.det_ptr.p;
    kp.det_terms = fl.det_terms.p;
    kp.noise = fl.noise.p;
    kp.noise_tab = fl.noise_tab.p;
    kp.noise_ch = fl.noise_ch.p;
    kp.noise_rowb = fl.noise_rowb.p;
    kp.init_dead = fl.init_dead.p;
    kp.row_of = fl.row_of.p;
    kp.num_noise = (int32_t)hp.num_noise;
    kp.tab_len = (int32_t)hp.noise_tab.size();
    kp.coins = injected ? pg->d_coins.p : nullptr;
    kp.masks = injected ? pg->d_masks.p : nullptr;
    kp.inject_words = words_all;
    kp.seed = seed;
    kp.n_ops = (int32_t)hp.ops.size();
    kp.num_qubits = hp.num_qubits;
    kp.num_slots = (int32_t)hp.num_slots;
    kp.num_obs = hp.mode == PM_EVENTS ? (int32_t)hp.num_obs : 0;  // accumulators live in the event ring
    kp.num_cols = (int32_t)hp.num_cols;
    kp.debug_skip = pg->opts.debug_skip;
    LaunchCfg cfg = fl.cfg;
    kp.desc_in_smem = fl.desc_smem ? 1 : 0;
    CUDA_TRY(pg->d_nscratch.reserve(pg->demk ? (size_t)pg->dem_grid * 32 * DEM_WARPS_HOST * NZ_MAX_LIST
                                             : (size_t)cfg.grid * cfg.threads * NZ_MAX_LIST));
    kp.noise_scratch = pg->d_nscratch.p;
    if (pg->opts.debug_skip & 64) {  // op-boundary clock trace of the first tile
        CUDA_TRY(pg->d_clock.reserve(hp.ops.size() * 12 + 1));
        CUDA_TRY(cudaMemsetAsync(pg->d_clock.p, 0, (hp.ops.size() * 12 + 1) * sizeof(long long), st));
        kp.op_clock = pg->d_clock.p;
    }

    if (!cfg.ring_smem && !pg->demk && hp.num_slots > 0) {
        Flavour& fw = const_cast<Flavour&>(fl);
        CUDA_TRY(fw.ring.reserve((size_t)hp.num_slots * W * cfg.grid * cfg.groups));
        kp.ring_global = fw.ring.p;
    }

    if (mode == PFS_MODE_COUNTS) {
        unsigned long long* cptr;
        if (dev_out) cptr = (unsigned long long*)out;
        else { CUDA_TRY(pg->d_counts.reserve(std::max<int64_t>(hp.num_cols, 1))); cptr = pg->d_counts.p; }
        if (hp.num_cols > 0) CUDA_TRY(cudaMemsetAsync(cptr, 0, hp.num_cols * 8, st));
        kp.counts = cptr;
        const size_t extra = (size_t)hp.num_cols * 4;
        kp.counts_in_smem = (cfg.smem_bytes + extra <= pg->smem_optin) ? 1 : 0;
        if (pg->demk) {
            kp.counts_in_smem = (pg->dem_per_warp ? dem_warp_smem_bytes(DEM_WARPS_HOST, hp.num_cols, true)
                                                  : dem_smem_bytes(DEM_WARPS_HOST, hp.num_cols, true)) <= pg->smem_optin;
        } else if (kp.counts_in_smem) {
            cfg.smem_bytes += extra;
        }
        // per-CTA u32 counters: bound shots per launch so no counter can overflow
        const int64_t max_tiles = std::max<int64_t>(1, ((int64_t)1 << 30) / T) * (pg->demk ? pg->dem_grid : cfg.grid);
        for (int64_t t0 = 0; t0 < n_tiles_all; t0 += max_tiles) {
            const int64_t nt = std::min(max_tiles, n_tiles_all - t0);
            kp.n_tiles = nt;
            kp.tile_offset = shot_offset / T + t0;
            kp.num_shots = std::min<int64_t>(num_shots - t0 * T, nt * T);
            if (injected) { kp.coins = pg->d_coins.p + t0 * W; kp.masks = pg->d_masks.p + t0 * W; }
            int rc2 = launch_tiles(pg, fl, kp, cfg, nt, st, true);
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
    const bool dem_direct = pg->demk && !pg->dem_global;  // dem_kernel writes b8 itself: no scratch
    int64_t chunk_tiles = n_tiles_all;
    if (!dev_out) {
        const int64_t bytes_per_tile = (dem_direct && b8 ? 0 : R * W * 4) + (b8 ? T * dev_pitch : 0);
        const int64_t target = (int64_t)256 << 20;
        chunk_tiles = std::max<int64_t>(1, target / std::max<int64_t>(bytes_per_tile, 1));
        chunk_tiles = std::max<int64_t>(chunk_tiles, pg->demk ? (int64_t)pg->dem_grid * 2 * (pg->dem_per_warp ? DEM_WARPS_HOST : 1)
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
        if (!direct_rows && !(dem_direct && b8))
            CUDA_TRY(pg->d_rows[b].reserve((size_t)std::max<int64_t>(R, 1) * ((chunk_words + 7) & ~7ll)));
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
        // b8: tile-major scratch [tile][row][W]
        kp.out_row_stride = b8 ? W : row_words;
        kp.out_tile_stride = b8 ? R * W : W;
        kp.rec_out = rows_meas ? rows : nullptr;
        kp.ev_out = rows_meas ? nullptr : rows;
        kp.n_tiles = nt;
        kp.tile_offset = shot_offset / T + t0;
        kp.num_shots = nshots;
        if (injected) { kp.coins = pg->d_coins.p + t0 * W; kp.masks = pg->d_masks.p + t0 * W; }
        OutParams cpx{};
        if (pg->demk) {
            if (b8) {
                cpx.b8_out = dev_out ? (uint8_t*)out + shots0 * out_pitch : pg->d_b8[b].p;
                cpx.b8_pitch = dev_out ? out_pitch : dev_pitch;
                cpx.b8_bytes = nbytes;
            } else {
                cpx.rows_out = rows;
                cpx.rows_stride = row_words;
            }
        }
        if (!pg->demk && direct_rows && (used_words % W) != 0) {
            // the last tile would write past the caller's rows: stage through scratch
            CUDA_TRY(pg->d_rows[0].reserve((size_t)std::max<int64_t>(R, 1) * chunk_words));
            rows = pg->d_rows[0].p;
            kp.out_row_stride = chunk_words;
            kp.out_tile_stride = W;
            kp.rec_out = rows_meas ? rows : nullptr;
            kp.ev_out = rows_meas ? nullptr : rows;
        }
        if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[2], st));
        TransposeJob tj;
        const bool wm = W == 1;
        const bool tj_ok = b8 && !pg->demk && !wm && kp.out_row_stride == W;
        if (tj_ok) {
            tj.rows = rows;
            tj.R = R;
            tj.xor_bits = mode == PFS_MODE_SAMPLES ? d_ref : nullptr;
            tj.dst = dev_out ? (uint8_t*)out + shots0 * out_pitch : pg->d_b8[b].p;
            tj.pitch = dev_out ? out_pitch : dev_pitch;
        }
        {
            int rc2 = launch_tiles(pg, fl, kp, cfg, nt, st, timing && ci == 0, cpx, tj_ok ? &tj : nullptr);
            if (rc2) return rc2;
        }
        if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[3], st));
        if ((b8 && dem_direct) || (b8 && tj.done)) {
            if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[5], st));
        } else if (b8) {
            uint8_t* dst = dev_out ? (uint8_t*)out + shots0 * out_pitch : pg->d_b8[b].p;
            const int64_t pitch = dev_out ? out_pitch : dev_pitch;
            // one-word tiles ([tile][row][1] = [tile][1][row]) are word-major:
            // transpose them as 8-word tiles (256-shot blocks per CTA)
            const int tw = (wm && W < 8) ? 8 : W;
            const int64_t ntw = (nt * W + tw - 1) / tw;
            CUDA_TRY(launch_tiles_to_b8(rows, R, tw, ntw, nshots, mode == PFS_MODE_SAMPLES ? d_ref : nullptr, dst,
                                        pitch, st, wm));
            pg->last_launches++;
            if (timing && ci == 0) CUDA_TRY(cudaEventRecord(pg->ev[5], st));
        } else if (direct_rows && rows != (uint32_t*)out) {
            CUDA_TRY(cudaMemcpy2DAsync(out, used_words * 4, rows, kp.out_row_stride * 4, used_words * 4, R,
                                       cudaMemcpyDeviceToDevice, st));
        }
        if (timing && ci == 0) {
            CUDA_TRY(cudaStreamSynchronize(st));
            cudaEventElapsedTime(&frame_ms, pg->ev[2], pg->ev[3]);
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
        pg->last_ms[0] = frame_ms - pg->last_ms[5];  // frame kernels only (noise_kernel: [5])
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
    // a pitched input spans (num_shots - 1) * in_pitch + nb_in bytes
    const size_t in_span = (size_t)(num_shots - 1) * in_pitch + nb_in;
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
        DE_TRY(cudaMemcpyAsync(d_in, flips_b8, in_span, cudaMemcpyHostToDevice, st));
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
    const int64_t m = std::min<int64_t>(n, (int64_t)pg->fl[PM_EVENTS].hp.ops.size() * 12);
    CUDA_TRY(cudaMemcpy(out, pg->d_clock.p, m * sizeof(long long), cudaMemcpyDeviceToHost));
    return PFS_OK;
}

// Profiling: the event program's device op list (kind|code|flags, count).
extern "C" int pfs_program_ops(const pfs_program* pg, uint32_t* out, int64_t n) {
    if (!pg || !out) return fail(PFS_E_INVALID, "null argument");
    const HostProgram& hp = pg->fl[PM_EVENTS].hp;
    const int64_t m = std::min<int64_t>(n, (int64_t)hp.ops.size());
    for (int64_t i = 0; i < m; i++) { out[2 * i] = hp.ops[i].kcf; out[2 * i + 1] = hp.ops[i].count; }
    return PFS_OK;
}

// Test tooling: raw tables of a compiled flavour (include/pfs.h).
extern "C" int64_t pfs_program_dump(const pfs_program* pg, int flavour, int what, uint32_t* out, int64_t n) {
    if (!pg || flavour < 0 || flavour > 1) return fail(PFS_E_INVALID, "bad argument");
    const HostProgram& hp = pg->fl[flavour].hp;
    const uint32_t* src = nullptr;
    int64_t words = 0;
    switch (what) {
        case 0: src = reinterpret_cast<const uint32_t*>(hp.ops.data()); words = (int64_t)hp.ops.size() * 8; break;
        case 1: src = hp.targets.data(); words = (int64_t)hp.targets.size(); break;
        case 2: src = hp.det_ptr.data(); words = (int64_t)hp.det_ptr.size(); break;
        case 3: src = hp.det_terms.data(); words = (int64_t)hp.det_terms.size(); break;
        case 4: src = reinterpret_cast<const uint32_t*>(hp.sops.data()); words = (int64_t)hp.sops.size() * 12; break;
        case 5: src = hp.arena.data(); words = (int64_t)hp.arena.size(); break;
        case 6: src = hp.fused_info.data(); words = (int64_t)hp.fused_info.size(); break;
        case 7: src = hp.row_of.data(); words = (int64_t)hp.row_of.size(); break;
        default: return fail(PFS_E_INVALID, "unknown table");
    }
    if (out && n > 0 && words > 0) std::memcpy(out, src, (size_t)std::min(n, words) * 4);
    return words;
}
