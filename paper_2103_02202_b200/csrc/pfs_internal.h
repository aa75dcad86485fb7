// Internal declarations shared by the host compiler (pfs_compile.cpp), the
// kernels (pfs_kernels.cu) and the C-ABI (pfs_api.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "pfs.h"

namespace pfs {

enum Kind : uint32_t { K_GATE = 0, K_M = 1, K_R = 2, K_MR = 3, K_NOISE = 4, K_DET = 5, K_OBS = 6,
                       K_SPILL = 7 };
enum Rule : uint32_t { R_NONE = 0, R_SWAPXZ = 1, R_ZXORX = 2, R_XXORZ = 3, R_CX = 4, R_CZ = 5,
                       R_CY = 6, R_SWAP = 7 };
enum Channel : uint32_t { CH_XERR = 0, CH_YERR = 1, CH_ZERR = 2, CH_DEP1 = 3, CH_DEP2 = 4 };

// Device op flags
constexpr uint32_t F_BARRIER = 1u;   // group barrier before this op
constexpr uint32_t F_DUP = 2u;       // noise op with repeated targets
constexpr uint32_t F_NOISE = 4u;     // fused noise (after a gate / reset, before a measurement)
constexpr uint32_t F_PRESAMPLED = 8u;  // stream op: the fused noise comes from noise_kernel's hit lists
constexpr uint32_t F_NOROWS = 16u;     // stream op: a measurement with no row work (dead coins, records stay
                                       // in their x rows, no record output): only its fused noise runs
constexpr uint32_t NO_SLOT = 0xFFFFFFFFu;
constexpr uint32_t COIN_DEAD = 0x80000000u;  // M/MR/R target word: the op's coin row reaches no output
constexpr uint32_t XROW = 0x80000000u;       // DET/OBS term: the record is the x row of this frame row

constexpr uint32_t DOMAIN_COIN = 0x40000000u;
constexpr uint32_t DOMAIN_NOISE = 0x80000000u;

// Noise chunk zones
constexpr uint32_t NZONE_TAB = 0u;   // Binomial(L, p) count by table inversion
constexpr uint32_t NZONE_NONE = 1u;  // p == 0: no hits
constexpr uint32_t NZONE_ALL = 2u;   // p == 1: every trial hits
constexpr int NZ_MAX_LIST = 16;      // distinct-position list; larger counts use selection sampling
constexpr int WSCR = 64;             // per-warp shared scratch of the warp-cooperative noise draws (words)
// frame kernel CTA size (launch bounds): 640 threads at 96 registers — the hot
// tile loop fits without spills, and 20 warps hide more of the op chain than 16
// at 128 registers (measured at d=25: 512 / 576 / 640 / 704 threads -> 6.83 /
// 7.85 / 6.55 / 8.08 ms per 2^20 shots)
#ifndef PFS_FRAME_MAX_THREADS
#define PFS_FRAME_MAX_THREADS 640
#endif
constexpr int FRAME_MAX_THREADS = PFS_FRAME_MAX_THREADS;
constexpr int KERNEL_COOP = 1;
// stream ops (+ threshold tables) are copied to shared memory when they take at most this much
constexpr int DESC_SMEM_MAX = 24576;

// Program flavours: detection events (DETECTORS / COUNTS / DETECTORS_ROWS) keep
// measurement records in the measured qubit's x row and a shared-memory ring,
// and skip coins that reach no detector; measurement records (FLIPS / SAMPLES /
// FLIPS_ROWS) store every record to the output and evaluate no detectors.
enum ProgMode : int { PM_EVENTS = 0, PM_RECORDS = 1 };

// One device op (32 bytes).  See DESIGN.md §3.
//   GATE : count = apps, off -> targets (1 or 2 per app); fused: a -> the
//          targets again, bank-ordered within each warp range of b applications
//   R    : count = targets, off -> (row, spill slot) pairs, b = first coin row
//   M/MR : count = targets, off -> (row, record slot) pairs, a = first record,
//          b = first coin row (MR: two per target, the second is the reset's)
//   NOISE: count = apps, off -> targets (standalone: hits applied with atomics)
//   DET  : count = columns, a = first column, code = k: terms of column a+i at
//          det_terms[off + k i ..]; code = 0: via det_ptr
//   OBS  : count = terms, off -> terms, a = accumulator slot
//   SPILL: count = targets, off -> (row, slot) pairs: ring[slot] = x[row]
// Noise (NOISE, or F_NOISE on GATE / R / M / MR): c = ordinal, d = geometry
// (lg L | lg cs << 5 | npat << 10 | channel << 14 | zone << 17), e = threshold
// table (offset | len << 24).
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

// Stream op (48 bytes): what frame_kernel reads per op (lower_stream, DESIGN.md
// §3).  Same index as the DOp it was lowered from (the rare general paths —
// inline noise draws, injected masks, CSR detectors — read the DOp).
//   GATE : arena[off ..]: one block of K * PI words per warp of the group
//          (PI = applications per warp pass = 32 / vectors per row); word =
//          row of target 0 | row of target 1 << 16, bank-ordered within the
//          warp's application range, STREAM_NOP padding
//   M / MR / R / SPILL: arena[off ..] = the (row | COIN_DEAD, slot) pairs; warp w
//          owns targets [w K, w K + K)
//   DET  : code = k > 0: arena[off + k i ..] = the k terms of column a + i
//   OBS  : arena[off ..] = terms
struct SOp {
    uint32_t kcf;        // kind | code << 8 | flags << 16 (DOp flags + F_PRESAMPLED)
    uint32_t count;
    uint32_t off;        // operand block in the arena (words)
    uint32_t K;          // GATE: passes per warp; collapses: targets per warp
    uint32_t a, b;       // as in DOp (first record / column / accumulator, first coin row)
    uint32_t span;       // F_PRESAMPLED: ordinal * list_warps (index of warp 0's span)
    uint32_t next_span;  // span index of the next F_PRESAMPLED op (this op's when it is the last)
    uint32_t r2;         // reserved
    uint32_t ordinal;    // noise ordinal (fused or standalone), else NO_SLOT
    uint32_t r0;         // GATE: applications per warp (the warp's share)
    uint32_t r1;         // reserved
};
static_assert(sizeof(SOp) == 48, "SOp is 48 bytes");
constexpr uint32_t STREAM_NOP = 0xFFFFFFFFu;
// Padding words of a gate block name dummy frame rows (rows num_qubits ..):
// no lane is predicated off; consecutive padding applications take different
// dummy rows so that they fall into different shared-memory bank groups.
constexpr int DUMMY_ROWS = 4;
// operand words of the next gate op a lane loads ahead (frame kernel GATE_AHEAD):
// every warp block of a gate op is padded to at least this many passes
#ifndef PFS_GATE_AHEAD
#define PFS_GATE_AHEAD 4
#endif
constexpr uint32_t GATE_AHEAD_PASSES = PFS_GATE_AHEAD;

// Per noise instruction sampling schedule for one tile, also
// exported to the parity oracle through pfs_program_noise_schedule.
struct NoiseParam {
    uint32_t L;        // trials per chunk (power of two)
    uint32_t cs;       // shots per chunk (power of two dividing T)
    uint32_t ca;       // applications per chunk (L / cs)
    uint32_t nchunks;  // ceil(apps / ca) * (T / cs)
    uint32_t apps;
    uint32_t tab;      // offset of the Binomial(L, p) thresholds in noise_tab
    uint32_t len;
    uint32_t zone;     // NZONE_*
    uint32_t npat;
    uint32_t ch;
    uint32_t fused;    // 1: applied inside the neighbouring gate / collapse op
    uint32_t reserved;
};
static_assert(sizeof(NoiseParam) == 48, "NoiseParam is 48 bytes");

struct HostProgram {
    int mode = PM_EVENTS;
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
    int64_t live_coin_rows = 0;       // coin rows that reach an output
    std::vector<DOp> ops;
    std::vector<uint32_t> targets;
    std::vector<uint32_t> det_ptr;    // [num_cols + 1] into det_terms
    std::vector<uint32_t> det_terms;  // ring slots, or XROW | frame row
    std::vector<uint32_t> init_dead;  // bitmap: qubits whose initial z coin reaches no output
    std::vector<uint32_t> row_of;     // frame row of each qubit (permute_rows)
    std::vector<double> noise_p;
    std::vector<uint32_t> noise_apps; // apps per noise ordinal
    std::vector<uint32_t> noise_ch;   // per ordinal: channel
    std::vector<uint32_t> noise_fused;  // per ordinal: applied inside a gate / collapse op
    std::vector<uint32_t> noise_rowb; // per ordinal: first injected noise-mask row
    // filled by build_noise_schedule once the tile geometry is known
    std::vector<NoiseParam> noise;
    std::vector<uint64_t> noise_tab;
    // pre-sampled hit lists of fused noise (build_hit_lists): per ordinal
    // (K = applications per consumer warp, 1 = pre-sampled, 0, targets
    // offset | PAIRS), and the noise_kernel work items of one tile
    std::vector<uint32_t> fused_info;   // 4 per ordinal (zeros: drawn by the frame kernel)
    std::vector<uint32_t> hit_items;    // 2 per item: ordinal, first | last consumer warp << 16
    // stream form of the ops for one tile geometry (lower_stream)
    std::vector<SOp> sops;
    std::vector<uint32_t> arena;
    uint32_t first_span = NO_SLOT;      // span index of the first F_PRESAMPLED op
    bool all_presampled = false;        // every noise op with p > 0 is fused and pre-sampled
    int64_t hit_block = 0;              // hit-entry capacity of one tile
    int32_t list_warps = 0;             // consumer warps per group
};
constexpr uint32_t FUSED_PAIRS = 0x80000000u;  // fused_info[3]: targets are (row, slot) pairs
constexpr int NK_WARPS = 8;                    // noise_kernel warps per CTA
constexpr int NK_SCR = 384;                    // noise_kernel hit entries staged per warp

// Host compiler: flat program -> device ops (splitting, noise fusion, merging,
// record homes and ring-slot liveness, coin relevance, barrier scheduling).
// Throws std::invalid_argument.
HostProgram compile_program(const pfs_instr* instrs, int64_t n_instrs, const int32_t* targets,
                            int64_t n_targets, const double* noise_p, int64_t n_noise,
                            const int64_t* det_ptr, const int64_t* det_idx, int64_t n_cols,
                            int64_t n_obs, int32_t num_qubits, int64_t num_meas,
                            int64_t num_coin_rows, int64_t num_noise_rows, int mode);

// tile_shots T, vector_shots S (shots one kernel item owns), expected hits per
// chunk of standalone and of fused noise instructions
void build_noise_schedule(HostProgram& hp, int tile_shots, int vector_shots, double target_hits,
                          double fused_target_hits);
void permute_rows(HostProgram& hp, int bank_classes, int warps_per_group);
void build_hit_lists(HostProgram& hp, int tile_shots, int warps_per_group);
void lower_stream(HostProgram& hp, int W, int warps_per_group);
void dedup_operands(HostProgram& hp);

// Kernel launch plumbing (pfs_kernels.cu)
struct KParams {
    const DOp* ops;
    const SOp* sops;             // stream ops (same indices as ops)
    const uint32_t* arena;       // their operand blocks
    uint32_t first_span;         // span index of the first pre-sampled op (NO_SLOT: none)
    const uint32_t* targets;
    const uint32_t* det_ptr;
    const uint32_t* det_terms;
    const NoiseParam* noise;
    const unsigned long long* noise_tab;
    const uint32_t* noise_ch;    // per noise ordinal: channel (error-model kernel)
    const uint32_t* noise_rowb;  // per noise ordinal: first injected mask row (x, z per target)
    const uint32_t* coins;       // injected: [rows][inject_words]
    const uint32_t* masks;
    uint32_t* rec_out;           // records: [M] rows (see out_*_stride) or null
    uint32_t* ev_out;            // events: [cols] rows or null
    unsigned long long* counts;  // [cols] or null
    uint32_t* ring_global;       // [grid][groups][slots][W] when the ring is not in smem
    long long* op_clock;         // profiling: per-op clock64 of CTA 0's first tile, or null
    uint32_t* noise_scratch;     // [grid][threads][NZ_MAX_LIST] general-path noise scratch
    const uint32_t* init_dead;   // bitmap of qubits whose initial coin row is dead (skip its draw)
    const uint32_t* row_of;      // frame row of qubit q (initial coin row q goes to z row row_of[q])
    int64_t inject_words;
    int64_t out_row_stride;      // output word address = row * out_row_stride
    int64_t out_tile_stride;     //                     + tile * out_tile_stride + word
    int64_t n_tiles;
    int64_t num_shots;           // shots of this launch (for tail masking)
    uint64_t seed;
    uint64_t tile_offset;        // global index of local tile 0
    int32_t n_ops;
    int32_t num_qubits;
    int32_t num_slots;
    int32_t num_obs;
    int32_t num_cols;
    int32_t num_noise;
    int32_t counts_in_smem;
    int32_t debug_skip;          // profiling ablations (pfs_options.debug_skip)
    int32_t groups;              // independent thread groups (tiles in flight) per CTA
    int32_t desc_in_smem;        // op descriptors + threshold tables copied to shared memory
    int32_t tab_len;             // threshold table entries
    // pre-sampled fused noise (noise_kernel): per ordinal (K, 1, 0, off | PAIRS)
    const uint4* fused;
    unsigned long long* hits_global;  // [tiles][hit_block] entries
    uint2* spans_global;              // [tiles][num_noise][list_warps] (begin, end) in the tile's
                                      // block (begin NO_SLOT: the warp draws inline)
    uint32_t* fill_global;            // [tiles][2]: entries used (noise_kernel allocation), overflow mark
    int32_t all_presampled;           // every noise instruction is fused and pre-sampled (hot frame loop)
    const uint2* hit_items;           // noise_kernel items of one tile
    int64_t hit_block;
    int32_t list_warps;
    int32_t n_items;
};

struct LaunchCfg {
    int kernel;  // KERNEL_COOP (frame_kernel); 0 = not runnable
    int W;
    int groups;
    bool ring_smem;
    int threads;
    int grid;
    size_t smem_bytes;
};

size_t frame_smem_bytes(int num_qubits, int W);
cudaError_t launch_frame_kernel(const LaunchCfg& cfg, const KParams& kp, cudaStream_t stream);
cudaError_t set_frame_kernel_smem(const LaunchCfg& cfg);
cudaError_t launch_noise_kernel(int W, const KParams& kp, int grid, cudaStream_t stream);
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
