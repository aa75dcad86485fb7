// Internal declarations shared by the host compiler (pfs_compile.cpp), the
// kernels (pfs_kernels.cu) and the C-ABI (pfs_api.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "pfs.h"

namespace pfs {

enum Kind : uint32_t { K_GATE = 0, K_M = 1, K_R = 2, K_MR = 3, K_NOISE = 4, K_DET = 5, K_OBS = 6 };
enum Rule : uint32_t { R_NONE = 0, R_SWAPXZ = 1, R_ZXORX = 2, R_XXORZ = 3, R_CX = 4, R_CZ = 5,
                       R_CY = 6, R_SWAP = 7 };
enum Channel : uint32_t { CH_XERR = 0, CH_YERR = 1, CH_ZERR = 2, CH_DEP1 = 3, CH_DEP2 = 4 };

// Device op flags
constexpr uint32_t F_BARRIER = 1u;   // __syncthreads() before this op
constexpr uint32_t F_DUP = 2u;       // noise op with repeated targets
constexpr uint32_t F_PREGEN = 4u;    // noise op whose hits come from the producer warps
constexpr uint32_t NO_SLOT = 0xFFFFFFFFu;
constexpr uint32_t COIN_DEAD = 0x80000000u;  // M/MR/R target word: the op's coin row is never read

constexpr uint32_t DOMAIN_COIN = 0x40000000u;
constexpr uint32_t DOMAIN_NOISE = 0x80000000u;

// Noise schedule flags
constexpr uint32_t NZ_NONE = 1u;     // p == 0: no hits
constexpr uint32_t NZ_ALL = 2u;      // p == 1: every trial hits
constexpr uint32_t NZ_PREGEN = 4u;   // hits generated in the tile's pre-pass into a hit list
constexpr int NZ_MAX_LIST = 16;
// frame kernel CTA size cap (launch bounds): 768 threads leaves 85 registers per
// thread, enough for the noise sampler without spills
constexpr int FRAME_MAX_THREADS = 768;
constexpr int WARP_KERNEL_MAX_THREADS = 1024;
constexpr int KERNEL_COOP = 1, KERNEL_WARP = 2;  // frame_warp_kernel: one word column per warp
// op descriptors are copied to shared memory when they take at most this much
constexpr int DESC_SMEM_MAX = 16384;      // distinct-position list; larger counts use selection sampling

// One device op (32 bytes).  See DESIGN.md §3.
//   GATE : count = apps, off -> targets (1 or 2 per app)
//   M/MR : count = targets, off -> (qubit, slot) pairs, a = rec_base, b = coin_base
//   R    : count = targets, off -> qubits, b = coin_base
//   NOISE: count = apps, off -> targets, a = noise_row_base, b = noise ordinal,
//          c = hit-list base, d/e = ordinal/hit-list base of the next
//          pre-generated noise op (NO_SLOT: none), for prefetching its hits
//   DET  : count = columns, a = first column (terms via det_ptr/det_terms)
//   OBS  : count = terms, off -> record slots, a = accumulator slot
struct DOp {
    uint32_t kcf;  // kind | code << 8 | flags << 16
    uint32_t count;
    uint32_t off;
    uint32_t a;
    uint32_t b;
    uint32_t c;
    uint32_t d;
    uint32_t e;
};
static_assert(sizeof(DOp) == 32, "DOp is 32 bytes");

// Per noise instruction sampling schedule for one tile: the
// op's trial space (apps x T shots, app-major) is cut into chunks of L trials;
// each chunk draws Binomial(len, p) hits by table inversion, then distinct
// uniform positions, then a uniform Pauli pattern per hit.
struct NoiseParam {
    uint32_t L;          // trials per chunk
    uint32_t nchunks;
    uint32_t last_len;   // trials in the last chunk
    uint32_t tab_full;   // offset of the Binomial(L, p) threshold table
    uint32_t len_full;
    uint32_t tab_last;   // Binomial(last_len, p) table
    uint32_t len_last;
    uint32_t cap_base;   // hit-list region of this op in the per-CTA scratch
    uint32_t cap;
    uint32_t flags;
    uint32_t npat;
    uint32_t chunk_base; // first pre-pass work item (32-chunk block) of this op
};
static_assert(sizeof(NoiseParam) == 48, "NoiseParam is 48 bytes");

struct HostProgram {
    int32_t num_qubits = 0;
    int64_t num_meas = 0;
    int64_t num_cols = 0;
    int64_t num_obs = 0;
    int64_t num_noise = 0;
    int64_t num_coin_rows = 0;
    int64_t num_noise_rows = 0;
    int64_t bframe_bits = 0;
    int64_t num_slots = 0;
    int64_t num_barriers = 0;
    std::vector<DOp> ops;
    std::vector<uint32_t> targets;
    std::vector<uint32_t> det_ptr;    // [num_cols + 1] into det_terms
    std::vector<uint32_t> det_terms;  // slots
    std::vector<uint32_t> init_dead;  // bitmap: qubits whose initial z coin is never read
    std::vector<uint32_t> row_of;     // frame row of each qubit (permute_rows)
    std::vector<double> noise_p;
    std::vector<uint32_t> noise_apps; // apps per noise ordinal
    std::vector<uint32_t> noise_arity;
    std::vector<uint32_t> noise_off;  // per ordinal: device target offset
    std::vector<uint32_t> noise_ch;   // per ordinal: channel
    // filled by build_noise_schedule once T is known
    std::vector<NoiseParam> noise;
    std::vector<uint64_t> noise_tab;
    std::vector<uint32_t> pregen_ops;   // noise ordinals with NZ_PREGEN, in order
    int64_t pregen_chunks = 0;          // total pre-pass work items (32-chunk blocks) per tile
    int64_t hit_capacity = 0;           // hit-list entries per CTA (per buffer)
    uint32_t first_pregen = NO_SLOT;
    uint32_t first_cap_base = 0;
};

// Host compiler: flat program -> device ops (splitting, merging, record-slot
// liveness allocation, barrier scheduling).  Throws std::invalid_argument.
HostProgram compile_program(const pfs_instr* instrs, int64_t n_instrs, const int32_t* targets,
                            int64_t n_targets, const double* noise_p, int64_t n_noise,
                            const int64_t* det_ptr, const int64_t* det_idx, int64_t n_cols,
                            int64_t n_obs, int32_t num_qubits, int64_t num_meas,
                            int64_t num_coin_rows, int64_t num_noise_rows);

void build_noise_schedule(HostProgram& hp, int tile_shots, double target_hits);
void permute_rows(HostProgram& hp);
void reorder_for_banks(HostProgram& hp, int W);
void dedup_operands(HostProgram& hp);

// Kernel launch plumbing (pfs_kernels.cu)
struct KParams {
    const DOp* ops;
    const uint32_t* targets;
    const uint32_t* det_ptr;
    const uint32_t* det_terms;
    const NoiseParam* noise;
    const uint64_t* noise_tab;
    const uint32_t* pregen_ops;
    const uint32_t* noise_off;   // per noise ordinal: offset of its targets
    const uint32_t* noise_ch;    // per noise ordinal: channel
    const uint32_t* coins;       // injected: [rows][inject_words]
    const uint32_t* masks;
    uint32_t* rec_out;           // [M][out_words] (flips rows) or null
    uint32_t* ev_out;            // [cols][out_words] or null
    unsigned long long* counts;  // [cols] or null
    uint32_t* ring_global;       // [grid][slots][W] when the ring is not in smem
    long long* op_clock;         // profiling: per-op clock64 of CTA 0's first tile, or null
    uint32_t* noise_scratch;     // [grid][threads][NZ_MAX_LIST] inline noise sampler scratch
    const uint32_t* init_dead;   // bitmap of qubits whose initial coin row is dead (skip its draw)
    const uint32_t* row_of;      // frame row of qubit q (initial coin row q goes to z row row_of[q])
    uint64_t* hits_global;       // [tiles][hit_capacity] pre-sampled noise hits (noise_kernel)
    uint32_t* ncnt_global;       // [tiles][num_noise] hits per noise op
    int64_t inject_words;
    int64_t out_row_stride;      // output word address = row * out_row_stride
    int64_t out_tile_stride;     //                     + tile * out_tile_stride + word
    int64_t out_word_stride;     // frame_warp_kernel: word w adds w * out_word_stride
    int64_t n_tiles;
    int64_t num_shots;           // shots of this launch (for tail masking)
    int64_t hit_capacity;
    uint64_t seed;
    uint64_t tile_offset;        // global index of local tile 0
    int32_t n_ops;
    int32_t num_qubits;
    int32_t num_slots;
    int32_t num_obs;
    int32_t num_cols;
    int32_t num_noise;
    int32_t num_pregen;
    int32_t pregen_chunks;
    int32_t counts_in_smem;
    int32_t do_dets;             // evaluate DET/OBS ops
    int32_t debug_skip;          // profiling ablations (pfs_options.debug_skip)
    int32_t groups;              // independent thread groups (tiles in flight) per CTA
    int32_t desc_in_smem;        // op descriptors copied to shared memory
    uint32_t first_pregen;       // first pre-generated noise ordinal (NO_SLOT: none)
    uint32_t first_cap_base;
};

struct LaunchCfg {
    int kernel;  // KERNEL_COOP (frame_kernel) or KERNEL_WARP (frame_warp_kernel)
    int W;
    int groups;
    bool ring_smem;
    int threads;
    int grid;
    size_t smem_bytes;
};

size_t frame_smem_bytes(int num_qubits, int W);
cudaError_t launch_frame_kernel(const LaunchCfg& cfg, const KParams& kp, cudaStream_t stream);
cudaError_t launch_noise_kernel(int W, const KParams& kp, int64_t n_tiles, cudaStream_t stream);
cudaError_t set_frame_kernel_smem(const LaunchCfg& cfg);
cudaError_t launch_frame_warp_kernel(const LaunchCfg& cfg, const KParams& kp, cudaStream_t stream);
cudaError_t set_frame_warp_kernel_smem(const LaunchCfg& cfg);
size_t warp_kernel_smem_per_warp(int num_qubits, int64_t num_slots, int64_t num_noise);
cudaError_t launch_rows_to_b8(const uint32_t* rows, int64_t num_rows, int64_t row_words,
                              int64_t num_shots, const uint8_t* xor_bits, uint8_t* out,
                              int64_t pitch, cudaStream_t stream);
cudaError_t smem_probe(int device, double* gbs);
cudaError_t launch_detector_events(const uint8_t* flips, int64_t in_pitch, int64_t num_shots,
                                   int64_t num_results, const int64_t* ptr, const int64_t* idx,
                                   int64_t num_dets, uint32_t* rows, uint32_t* ev, uint8_t* out,
                                   int64_t out_pitch, cudaStream_t st);
// tile-major [tile][row][W] (word_major: [tile][W][row]) bit tables -> shot-major
// b8 rows of `pitch` bytes
cudaError_t launch_tiles_to_b8(const uint32_t* tiles, int64_t num_rows, int W, int64_t n_tiles,
                               int64_t num_shots, const uint8_t* xor_bits, uint8_t* out,
                               int64_t pitch, cudaStream_t stream, bool word_major = false);

// ---------------------------------------------------------------- column kernel
// frame_col_kernel (pfs_colkernel.cu): every consumer warp owns one 32-shot
// word column (its own x/z planes and record ring in shared memory) for the
// whole circuit, so warps never wait for each other; the op stream is a byte
// stream of self-describing blocks that one producer warp bulk-copies (TMA)
// into a ring of shared-memory slots shared by the CTA's warps.
constexpr int KERNEL_COL = 3;
constexpr int COL_MAX_WARPS = 15;     // consumer warps per CTA (+1 producer; 128 registers per thread)
// one-word columns with the record ring in global memory: more, lighter warps
constexpr int col_max_warps(int V, bool ring_smem) { return (V == 1 && !ring_smem) ? 19 : COL_MAX_WARPS; }
#ifndef PFS_COL_SLOTS
#define PFS_COL_SLOTS 4
#endif
constexpr int COL_SLOTS = PFS_COL_SLOTS;  // op-block ring depth
constexpr uint32_t F_GLOBALP = 8u;    // block payload left in global memory (too big to stage)
constexpr uint32_t COL_HEAD_WORDS = 8;   // block header (CHead)
constexpr uint32_t COL_NP_WORDS = 12;    // NoiseParam after a noise op's header

// Block header, 32 bytes; payload words follow (after a NoiseParam for noise ops).
//   GATE: count apps, payload targets (1 or 2 per app)
//   M/MR: count targets, a = first record, b = first coin row, payload (qubit, slot) pairs
//   R   : count targets, b = first coin row, payload qubits
//   NOISE: count apps, a = first noise-mask row, b = noise ordinal, payload targets
//   DET : count columns, a = first column; code = k > 0: payload k slots per column;
//         code = 0: payload = count + 1 column offsets, then the slot terms
//   OBS : count terms, a = accumulator slot, payload slots
struct CHead {
    uint32_t kcf;
    uint32_t count;
    uint32_t a;
    uint32_t b;
    uint32_t pwords;   // payload words
    uint32_t goff;     // word offset of the payload in the global stream
    uint32_t r0, r1;
};
static_assert(sizeof(CHead) == 32, "CHead is 32 bytes");

struct ColStream {
    std::vector<uint32_t> words;     // blocks, each 16-byte aligned
    std::vector<uint32_t> binfo;     // per block: (16-byte offset, staged bytes) pairs
    uint32_t slot_bytes = 0;         // largest staged block
    int64_t n_blocks = 0;
};
ColStream build_col_stream(const HostProgram& hp, uint32_t slot_cap);

struct ColParams {
    const uint32_t* stream;
    const uint2* binfo;
    uint8_t* b8_out;             // shot-major output (b8 modes) or null
    int64_t b8_pitch;
    int64_t b8_bytes;            // ceil(R / 8)
    const uint32_t* ref_words;   // SAMPLES: reference bits packed LSB-first in words, or null
    uint32_t* rows_out;          // *_ROWS modes: [R][rows_stride] words, or null
    int64_t rows_stride;
    int64_t n_units;             // 32-shot words of this launch
    int32_t n_blocks;
    int32_t slot_bytes;
    int32_t nw;                  // consumer warps per CTA
    int32_t warp_words;          // shared-memory words per consumer warp
    int32_t records;             // 1: the output columns are measurement records
    int32_t ncols_out;           // R: output columns (records or detector columns)
    int32_t b8_aligned;          // b8 pitch and base allow 32-bit stores
};

size_t col_warp_words(int num_qubits, int64_t num_slots, bool ring_smem, int V);
size_t col_smem_bytes(int nw, size_t warp_words, uint32_t slot_bytes, int64_t counts_words);
cudaError_t launch_frame_col_kernel(const KParams& kp, const ColParams& cp, int V, bool ring_smem, int grid,
                                    size_t smem, cudaStream_t stream);
cudaError_t set_frame_col_kernel_smem(size_t smem);

// ---------------------------------------------------------------- error model
// Detector error model (pfs_dem.cpp): per noise ordinal o, application a and
// component k (x slot 0, z slot 0, x slot 1, z slot 1) the output columns a
// frame flip there reaches: cols[comp_ptr[i] .. comp_ptr[i + 1]) with
// i = comp_base[o] + 4 a + k.  coin_dependent != "": some collapse coin reaches
// an output, so the events are not a function of the noise draws alone.
constexpr int KERNEL_DEM = 4;
struct DemModel {
    std::vector<uint32_t> comp_base;
    std::vector<uint32_t> comp_ptr;
    std::vector<uint32_t> cols;
    // one 64-bit word per component: up to 3 columns inline (20 bits each,
    // count in bits 62-63), else count 0 and (offset into cols, n) = bits 0-31, 32-61
    std::vector<unsigned long long> comp_words;
    std::string coin_dependent;
    double mean_cols_per_comp = 0.0;
    std::vector<uint32_t> items;     // (ordinal, chunk) pairs of one tile (set once the schedule is built)
};
DemModel build_dem(const pfs_instr* ins, int64_t n_ins, const int32_t* targets, const int64_t* det_ptr,
                   const int64_t* det_idx, int64_t n_cols, int32_t num_qubits, int64_t num_meas,
                   int64_t n_noise);

struct DemParams {
    const uint32_t* comp_base;             // first component of each noise ordinal
    const uint32_t* cols;                  // CSR columns of long signatures
    const unsigned long long* comp_words;  // DemModel::comp_words
    uint8_t* b8_out;             // shot-major detection events, or null
    int64_t b8_pitch;
    int64_t b8_bytes;
    uint32_t* rows_out;          // DETECTORS_ROWS: [cols][rows_stride], or null
    int64_t rows_stride;
    const uint2* items;          // (noise ordinal, chunk) work items of one tile
    int32_t n_items;
    int32_t warps;
    int32_t per_warp;            // dem_warp_kernel: one 32-shot tile per warp (small circuits)
};
cudaError_t launch_dem_kernel(const KParams& kp, const DemParams& dp, bool global_cols, int grid, size_t smem,
                              cudaStream_t st);
cudaError_t set_dem_kernel_smem(size_t smem);
size_t dem_smem_bytes(int warps, int64_t num_cols, bool counts);
size_t dem_warp_smem_bytes(int warps, int64_t num_cols, bool counts);

// output writers (pfs_writers.cu): device b8 -> 01 (fmt 0), hits (2), r8 (3)
cudaError_t write_format(const uint8_t* in, int64_t pitch, int64_t shots, int64_t R, int fmt, uint8_t* out,
                         int64_t capacity, int64_t* out_len, cudaStream_t st);

}  // namespace pfs
