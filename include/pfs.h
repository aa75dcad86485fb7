/*
 * pfs.h — C-ABI of the B200 bulk Pauli-frame sampler (libpfs.so).
 *
 * The reference (stabsim, pure Python) has no native FFI; this ABI is what its
 * Python entry points would bind through ctypes to replace the hot path:
 *
 *   pfs_program_create   replaces  compile_frame_program     stabsim/frame_sim.py:170-189
 *                        (plus the record/detector bookkeeping of circuit.detector_sets,
 *                         stabsim/circuit.py:247-256)
 *   pfs_run (FLIPS)      replaces  collect_flips             stabsim/frame_sim.py:208-229
 *                        (FrameBatch + _run_batch + _transpose_flips, frame_sim.py:26-239)
 *   pfs_run (SAMPLES)    replaces  sample_batch              stabsim/frame_sim.py:242-258
 *   pfs_run (DETECTORS)  replaces  collect_flips + detector_events
 *                                                            stabsim/io_formats.py:208-227
 *   pfs_run (COUNTS)     new: per-column event counts (no output I/O; BASELINE config 3)
 *   pfs_last_error       error text (the reference raises ValueError, frame_sim.py:30-31,
 *                        211-212, 247-250; the ctypes shim re-raises it)
 *
 * All arguments are plain pointers and sizes.  Return value: 0 on success, a
 * negative PFS_E* code on failure with a thread-local message in pfs_last_error().
 * Threading: a program handle is bound to one device; do not run one handle on two
 * streams concurrently.  Ownership: the caller owns every input and output buffer;
 * the handle owns its device copies.
 */
#ifndef PFS_H
#define PFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat instruction row (int32 x 8), produced by paper_2103_02202_b200/program.py.
 * kind: 0 gate (code = frame rule), 1 M, 2 R, 3 MR, 4 noise (code = channel),
 *       5 DETECTOR (aux = column), 6 OBSERVABLE_INCLUDE (aux = column,
 *       targets = absolute record indices). */
typedef struct pfs_instr {
    int32_t kind, code, n_targets, tgt_off, rec_base, coin_base, noise_row_base, aux;
} pfs_instr;

typedef struct pfs_options {
    int32_t words_per_tile;   /* W: 32-shot words per CTA tile (0 = auto)          */
    int32_t ring_in_smem;     /* -1 auto, 0 global-memory record ring, 1 shared     */
    int32_t threads;          /* threads per CTA (0 = auto)                         */
    int32_t ctas_per_sm;      /* persistent grid = SMs x this (0 = auto)            */
    double noise_target_hits; /* expected hits per geometric-walk chunk (0 = 1.0)   */
    int32_t timing;           /* 1: record per-kernel CUDA-event times in pfs_run  */
    int32_t debug_skip;       /* profiling ablations only (wrong results!): bit0 noise
                                 apply, bit1 noise pre-pass, bit2 coin RNG, bit3 detectors,
                                 bit4 gates, bit5 collapses */
    int32_t presample_noise;  /* fused noise drawn by noise_kernel into per-warp hit
                                 lists ahead of the frame kernel: 0 auto (on), -1 off
                                 (drawn inline by the frame kernel)                 */
    int32_t schedule_only;    /* 1: compile without the shared-memory fit check (the
                                 program exposes info / noise schedule, cannot run)  */
    int32_t groups;           /* independent tiles in flight per CTA (0 = auto)     */
    int32_t kernel;           /* 0 auto = 1: frame sampler (frame_kernel, a CTA's
                                 threads share one tile); 4: error-model detector
                                 sampler (dem_kernel, detection events only)        */
    int32_t pipeline;         /* frame / transpose pipeline: sub-chunks per launch
                                 whose shot-major transpose overlaps the next
                                 sub-chunk's frame kernel (0 = auto, 1 = off)        */
    int32_t fused_target_milli; /* expected hits x 1000 per noise chunk of a noise
                                 instruction fused into its gate / collapse op
                                 (0 = 1000)                                         */
} pfs_options;

typedef struct pfs_info {
    int32_t num_qubits;
    int32_t words_per_tile;   /* W */
    int32_t tile_shots;       /* T = 32 W */
    int32_t threads;
    int32_t ring_in_smem;
    int32_t smem_bytes;       /* dynamic shared memory per CTA */
    int64_t num_measurements;
    int64_t num_columns;      /* detectors + observables */
    int64_t num_observables;
    int64_t num_ops;          /* device ops after splitting/merging */
    int64_t num_barriers;     /* __syncthreads between ops per tile */
    int64_t num_slots;        /* record ring slots (incl. observable accumulators) */
    int64_t num_noise;
    int64_t bframe_bits;      /* algorithmic frame bits per shot */
    int64_t num_coin_rows;
    int64_t num_noise_rows;
    int64_t noise_tab_len;    /* uint64 entries of the Binomial threshold tables   */
    int64_t live_coin_rows;   /* coin rows that reach an output (event program)      */
    int64_t record_ops;       /* device ops of the measurement-record program        */
    int64_t groups;           /* independent tiles in flight per CTA                */
    int64_t kernel;           /* 1 frame sampler, 4 error-model sampler              */
    int64_t warps_per_cta;    /* reserved (0)                                        */
    int64_t fused_noise;      /* noise instructions applied inside gate / collapse ops */
} pfs_info;

enum pfs_mode {
    PFS_MODE_FLIPS = 0,          /* shot-major b8 measurement flips                 */
    PFS_MODE_SAMPLES = 1,        /* shot-major b8 flips XOR reference sample         */
    PFS_MODE_DETECTORS = 2,      /* shot-major b8 detection events (+ observables)  */
    PFS_MODE_COUNTS = 3,         /* uint64 event count per column                   */
    PFS_MODE_FLIPS_ROWS = 4,     /* measurement-major uint32 rows [M][ceil(S/32)]   */
    PFS_MODE_DETECTORS_ROWS = 5  /* column-major uint32 rows [D][ceil(S/32)]        */
};

enum pfs_error {
    PFS_OK = 0,
    PFS_E_INVALID = -1,   /* bad argument (maps to ValueError)   */
    PFS_E_CUDA = -2,      /* CUDA runtime failure                */
    PFS_E_NOMEM = -3,     /* host/device allocation failure      */
    PFS_E_NODEVICE = -4   /* no CUDA device / extension unusable */
};

int pfs_program_create(const pfs_instr* instrs, int64_t n_instrs,
                       const int32_t* targets, int64_t n_targets,
                       const double* noise_p, int64_t n_noise,
                       const int64_t* det_ptr, const int64_t* det_idx,
                       int64_t n_columns, int64_t n_observables,
                       int32_t num_qubits, int64_t num_measurements,
                       int64_t num_coin_rows, int64_t num_noise_rows,
                       const pfs_options* options_or_null, struct pfs_program** out);

int pfs_program_info(const struct pfs_program* prog, pfs_info* out);

/* The per-tile noise sampling schedule, for the parity oracle:
 * params = num_noise x 12 uint32 (L, nchunks, last_len, tab_full, len_full,
 * tab_last, len_last, cap_base, cap, flags, npat, chunk_base), tab = the
 * Binomial threshold tables (noise_tab_len uint64). */
int pfs_program_noise_schedule(const struct pfs_program* prog, uint32_t* params,
                               int64_t n_params, uint64_t* tab, int64_t n_tab);

/*
 * Sample num_shots shots [shot_offset, shot_offset + num_shots) on `device`.
 * shot_offset must be a multiple of the tile size T (pfs_info.tile_shots); the
 * counter-based RNG is keyed by (seed, global tile, event), so results do not
 * depend on how a shot range is split across calls or GPUs.
 *
 * ref_bits: uint8[num_measurements] reference sample (SAMPLES only).
 * inject_coins / inject_noise: both NULL (Philox mode) or both set (injected
 * mode): uint32 rows [num_coin_rows | num_noise_rows][inject_row_words], shot s
 * of a row at bit s%32 of word s/32.
 * out: host or device pointer (detected).  b8 modes write num_shots rows of
 * out_pitch bytes (out_pitch >= ceil(R/8); 0 = exactly ceil(R/8));
 * COUNTS writes uint64[num_columns]; *_ROWS write rows of ceil(num_shots/32) words.
 * stream: cudaStream_t (NULL = legacy default stream).  Host outputs are complete
 * when pfs_run returns; device outputs are complete in stream order.
 */
int pfs_run(struct pfs_program* prog, int device, uint64_t seed, uint64_t shot_offset,
            int64_t num_shots, int mode, const uint8_t* ref_bits,
            const uint32_t* inject_coins, const uint32_t* inject_noise,
            int64_t inject_row_words, void* out, int64_t out_bytes, int64_t out_pitch,
            void* stream);

/* Per-kernel times (ms) of the last pfs_run when options.timing = 1 (first
 * chunk): [0] frame program kernel, [1] transpose kernel, [2] H2D, [3] D2H,
 * [4] total, [5] noise sampling kernel. */
int pfs_program_last_timing(const struct pfs_program* prog, double* ms, int n);

/* Number of this library's kernel launches made by the last pfs_run. */
int64_t pfs_program_last_launches(const struct pfs_program* prog);

/* detector_events (stabsim/io_formats.py:208-227) for flips that were already
 * sampled: flips_b8 = shot-major b8 rows (in_pitch bytes, 0 = ceil(M/8)),
 * detectors as CSR (det_ptr[num_dets+1], det_idx = record indices); writes
 * shot-major b8 events.  Host or device buffers; synchronous. */
int pfs_detector_events(int device, const uint8_t* flips_b8, int64_t num_shots,
                        int64_t num_results, int64_t in_pitch, const int64_t* det_ptr,
                        const int64_t* det_idx, int64_t num_dets, uint8_t* out_b8,
                        int64_t out_bytes, int64_t out_pitch, void* stream);

/* Roofline denominator for the SMEM-resident frame kernel: measured shared-
 * memory bandwidth (GB/s, loads + stores, CX access mix) over all SMs. */
int pfs_measure_smem_bandwidth(int device, double* gbs);

/* Profiling helpers: per-op clock64 trace (debug_skip bit 6) and the device op
 * list as (kind|code<<8|flags<<16, count) pairs. */
int pfs_program_op_clock(struct pfs_program* prog, long long* out, int64_t n);
int pfs_program_ops(const struct pfs_program* prog, uint32_t* out, int64_t n);

/* Test tooling: the raw tables of a compiled flavour (0 detection events,
 * 1 measurement records) as uint32 words, for the static schedule verifier
 * (tests/test_schedule.py: every pair of ops with no group barrier between
 * them touches disjoint frame rows and ring slots; every application sits in
 * exactly one warp's operand block).  what: 0 device ops (8 words each),
 * 1 targets, 2 det_ptr, 3 det_terms, 4 stream ops (12 words each), 5 operand
 * arena, 6 fused_info (4 words per noise ordinal), 7 row_of.  Copies
 * min(n, words) words into out (may be NULL) and returns the table's length
 * in words, or a negative error. */
int64_t pfs_program_dump(const struct pfs_program* prog, int flavour, int what, uint32_t* out, int64_t n);

void pfs_program_destroy(struct pfs_program* prog);
const char* pfs_last_error(void);
int pfs_version(void);

/* write_table on the GPU (stabsim/io_formats.py:66-201): shot-major b8 rows
 * (host or device, in_pitch bytes apart) -> fmt 0 "01", 2 "hits", 3 "r8",
 * byte-exact with the reference writers.  out == NULL (or too small): only
 * *out_len is set (the bytes needed).  b8 needs no writer (it is the input). */
int pfs_write_format(int device, const uint8_t* b8, int64_t in_pitch, int64_t num_shots,
                     int64_t num_results, int fmt, uint8_t* out, int64_t out_capacity,
                     int64_t* out_len, void* stream);

/* ---- native reference sample (stabsim/tableau_sim.py:326-329) ----------
 * Noiseless inverse-tableau simulation of a circuit lowered to rows
 * (gate code, n_targets, target offset) x int32; noise and annotations are
 * dropped by the caller.  Random measurement / reset collapses consume one
 * coin each from `coins`, in circuit order (the reference draws
 * rng.integers(2) per collapse, tableau_sim.py:177).  Writes one bit per
 * measurement to out_bits and, when non-null, 1/0 to out_determined
 * (SimState.determined_record).  Host-only: needs no GPU. */
enum pfs_tableau_gate {
    PFS_TG_I = 0, PFS_TG_X = 1, PFS_TG_Y = 2, PFS_TG_Z = 3, PFS_TG_H = 4, PFS_TG_S = 5,
    PFS_TG_S_DAG = 6, PFS_TG_SQRT_X = 7, PFS_TG_SQRT_X_DAG = 8, PFS_TG_SQRT_Y = 9,
    PFS_TG_SQRT_Y_DAG = 10, PFS_TG_CX = 11, PFS_TG_CY = 12, PFS_TG_CZ = 13, PFS_TG_SWAP = 14,
    PFS_TG_M = 15, PFS_TG_R = 16, PFS_TG_MR = 17
};
int pfs_reference_sample(const int32_t* ops, int64_t n_ops, const int32_t* targets,
                         int64_t n_targets, int32_t num_qubits, const uint8_t* coins,
                         int64_t n_coins, uint8_t* out_bits, uint8_t* out_determined,
                         int64_t n_out, int64_t* n_written);
const char* pfs_reference_sample_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PFS_H */
