/*
 * pfs_oracle.c — CPU restatement of the reference's bulk Pauli-frame sampler.
 *
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library;
 * the product path (paper_2103_02202_b200/) never links or calls it, and this
 * file uses nothing of the product (its noise schedule is computed here).
 *
 * It restates, over uint32 shot words instead of Python ints:
 *   FrameBatch.__init__            stabsim/frame_sim.py:29-40   (x = 0, z = coins)
 *   _apply_plan per frame rule     stabsim/frame_sim.py:64-72   + gates.py:70-92
 *   measure / reset / measure_reset stabsim/frame_sim.py:74-90
 *   apply_noise                    stabsim/frame_sim.py:92-167  (i.i.d. Bernoulli(p) per
 *                                  (application, frame) trial; entropy.py:65-113;
 *                                  patterns gates.py:98-104, 146-152)
 *   _run_batch opcode loop         stabsim/frame_sim.py:192-205
 *   detector_events                stabsim/io_formats.py:208-227
 *   transposed + write_b8          stabsim/bitvec.py:193-209, io_formats.py:94-96
 *
 * Randomness comes from one of two sources:
 *   - injected rows (coins + noise masks) — bit-exact
 *     against the reference's own FrameBatch (tests/golden/inject_*.npz);
 *   - counter-based Philox4x32-10 driving the chunked Bernoulli sampler of
 *     DESIGN.md §4 (Binomial count by table inversion + distinct uniform
 *     positions — the same i.i.d. Bernoulli(p) trials the reference's geometric
 *     gaps / hybrid sampler produce, drawn in an order a GPU can parallelise).
 *     The layout parameters are the tile size T, the vector size S and the
 *     chunk length L of every noise instruction (they choose the draw order,
 *     not the distribution); the chunk geometry and the Binomial(L, p)
 *     threshold tables are computed here (orc_noise_schedule).  The CUDA
 *     kernels make the same draws, so the GPU's sampled mode is bit-exact
 *     against this file as well as statistically matched to the reference
 *     (tests/golden/stats_*.npz).
 *
 * Parity pinned by: tests/golden/{inject,noiseless,stats,exact}_* generated from
 * the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { K_GATE = 0, K_M = 1, K_R = 2, K_MR = 3, K_NOISE = 4, K_DET = 5, K_OBS = 6 };
enum { R_NONE = 0, R_SWAPXZ = 1, R_ZXORX = 2, R_XXORZ = 3, R_CX = 4, R_CZ = 5, R_CY = 6, R_SWAP = 7 };
enum { CH_XERR = 0, CH_YERR = 1, CH_ZERR = 2, CH_DEP1 = 3, CH_DEP2 = 4 };

typedef struct {
    int32_t kind, code, n_targets, tgt_off, rec_base, coin_base, noise_row_base, aux;
} orc_instr;

/* ---------------- Philox4x32-10 (Salmon et al., SC'11) ---------------- */
static inline void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; r++) {
        philox_round(c, k);
        if (r < 9) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

#define DOMAIN_COIN 0x40000000u
#define DOMAIN_NOISE 0x80000000u
#define NZ_MAX_LIST 16

/* Key of global tile g: counters carry g's low 32 bits, the
 * high bits are folded into key word 1. */
typedef struct { uint32_t k[2]; uint32_t g; } tile_key;
static inline tile_key make_key(uint64_t seed, uint64_t g) {
    tile_key t;
    t.k[0] = (uint32_t)seed;
    t.k[1] = (uint32_t)(seed >> 32) ^ ((uint32_t)(g >> 32) * 0x9E3779B9u);
    t.g = (uint32_t)g;
    return t;
}

/* ---------------- noise schedule ---------------- */
enum { ZONE_TAB = 0, ZONE_NONE = 1, ZONE_ALL = 2 };
typedef struct {
    uint32_t L, cs, ca, nchunks, apps, npat, ch, zone, len;
    uint64_t tab[256];  /* Binomial(L, p) inverse-CDF thresholds, 64-bit fixed point */
} orc_noise;

/* X = min{m : u < t[m]} for u uniform on [0, 2^64); upper-tail thresholds come
 * from the tail sum so their absolute error stays ~2^-64. */
static int binomial_thresholds(uint64_t n, double p, uint64_t* t, int cap) {
    double* pmf = (double*)malloc(sizeof(double) * 4096);
    double* sf = (double*)malloc(sizeof(double) * 4096);
    if (!pmf || !sf) { free(pmf); free(sf); return -1; }
    const double q = 1.0 - p;
    double pm = exp((double)n * log1p(-p));
    const double mean = (double)n * p;
    int M = 0;
    for (uint64_t m = 0;; m++) {
        if (M >= 4096) { free(pmf); free(sf); return -1; }
        pmf[M++] = pm;
        if (m == n) break;
        if ((double)m > mean && pm < 1e-40) break;
        pm = pm * ((double)(n - m) / (double)(m + 1)) * (p / q);
    }
    sf[M - 1] = 0.0;
    for (int m = M - 1; m-- > 0;) sf[m] = sf[m + 1] + pmf[m + 1];
    int len = 0;
    double cdf = 0.0;
    for (int m = 0; m < M; m++) {
        cdf += pmf[m];
        const double tail = ldexp(sf[m], 64);
        if (tail < 1.0) break;
        uint64_t v;
        if (cdf <= 0.5) v = (uint64_t)floor(ldexp(cdf, 64));
        else v = (uint64_t)0 - (uint64_t)ceil(tail);
        if (len >= cap) { free(pmf); free(sf); return -1; }
        t[len++] = v;
    }
    free(pmf);
    free(sf);
    return len;
}

/* Geometry and table of one noise instruction: apps applications, probability
 * p, chunk length L (a power of two), tile T shots, vector S shots. */
static int schedule_one(orc_noise* np, uint32_t apps, int ch, double p, uint32_t L, uint32_t T, uint32_t S) {
    memset(np, 0, sizeof(*np));
    np->apps = apps;
    np->ch = (uint32_t)ch;
    np->npat = ch == CH_DEP1 ? 3u : (ch == CH_DEP2 ? 15u : 1u);
    if ((L & (L - 1)) || L == 0) return -1;
    np->L = L;
    np->cs = L < S ? L : S;
    if (T % np->cs) return -1;
    np->ca = L / np->cs;
    np->nchunks = ((apps + np->ca - 1) / np->ca) * (T / np->cs);
    if (apps == 0 || p <= 0.0) { np->zone = ZONE_NONE; return 0; }
    if (p >= 1.0) { np->zone = ZONE_ALL; return 0; }
    np->zone = ZONE_TAB;
    int len = binomial_thresholds(L, p, np->tab, 256);
    if (len < 0) return -1;
    np->len = (uint32_t)len;
    return 0;
}

/* Exported for the tests: 12 words (L, cs, ca, nchunks, apps, 0, len, zone, npat,
 * ch, 0, 0) and the table of one instruction. */
int orc_noise_schedule(uint32_t apps, int ch, double p, uint32_t L, uint32_t T, uint32_t S, uint32_t* params,
                       uint64_t* tab, int tab_cap) {
    orc_noise* np = (orc_noise*)malloc(sizeof(orc_noise));
    if (!np) return -2;
    int rc = schedule_one(np, apps, ch, p, L, T, S);
    if (rc == 0) {
        uint32_t w[12] = {np->L, np->cs, np->ca, np->nchunks, np->apps, 0, np->len, np->zone, np->npat, np->ch, 0, 0};
        memcpy(params, w, sizeof(w));
        if ((int)np->len > tab_cap) rc = -3;
        else memcpy(tab, np->tab, sizeof(uint64_t) * np->len);
    }
    free(np);
    return rc;
}

typedef struct {
    const orc_instr* ins; int64_t n_ins;
    const int32_t* targets;
    const double* noise_p; const orc_noise* noise;
    int32_t num_qubits; int64_t num_meas;
    const int64_t* det_ptr; const int64_t* det_idx; int64_t num_cols;
    int64_t num_shots; int32_t T; uint64_t seed; uint64_t tile_offset;
    const uint32_t* coins; const uint32_t* masks; int64_t inject_words;
    uint32_t* flips; uint32_t* events; int64_t out_words;
    int64_t n_tiles; int nthreads;
} orc_job;

typedef struct { const orc_job* job; int tid; int rc; } orc_worker;

static inline uint64_t umul64hi(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
}
static inline uint32_t umulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }

/* Philox block j of chunk r. */
static inline void noise_block(const tile_key* tk, uint32_t j, uint32_t r, uint32_t ordinal, uint32_t w[4]) {
    uint32_t ctr[4] = {j, r, tk->g, DOMAIN_NOISE | ordinal};
    orc_philox4x32_10(ctr, tk->k, w);
}

/* Word pair k of chunk r: pair 0 = block 0 (w2, w3); pair k >= 1 = block
 * (k+1)/2, (w0, w1) for odd k, (w2, w3) for even k. */
static inline void noise_pair(const tile_key* tk, uint32_t k, uint32_t r, uint32_t ordinal, uint32_t* a, uint32_t* b) {
    uint32_t w[4];
    noise_block(tk, k == 0 ? 0u : (k + 1) >> 1, r, ordinal, w);
    if (k == 0 || !(k & 1u)) { *a = w[2]; *b = w[3]; }
    else { *a = w[0]; *b = w[1]; }
}

/* hits of chunk r: emit(position within the chunk, pattern pick) for every
 * hit at a position < vlen */
typedef void (*emit_fn)(void* ctx, uint32_t pos, uint32_t pick);
static void noise_chunk(const orc_noise* np, const tile_key* tk, uint32_t ordinal, uint32_t r, uint32_t vlen,
                        emit_fn emit, void* ctx) {
    const uint32_t L = np->L;
    uint32_t lg = 0;
    while ((1u << lg) < L) lg++;
    uint32_t w[4];
    if (np->zone == ZONE_NONE) return;
    if (np->zone == ZONE_ALL) {
        for (uint32_t i = 0; i < vlen; i++) {
            noise_block(tk, 0x80000000u + i, r, ordinal, w);
            emit(ctx, i, np->npat > 1 ? umulhi32(w[2], np->npat) : 0u);
        }
        return;
    }
    noise_block(tk, 0u, r, ordinal, w);
    const uint64_t u = ((uint64_t)w[1] << 32) | w[0];
    uint32_t count = 0;
    while (count < np->len && u >= np->tab[count]) count++;
    if (count == 0) return;
    if (count <= NZ_MAX_LIST) {
        uint32_t pos[NZ_MAX_LIST], pick[NZ_MAX_LIST];
        for (uint32_t attempt = 0;; attempt++) {
            for (uint32_t h = 0; h < count; h++) {
                uint32_t a, b;
                noise_pair(tk, attempt * NZ_MAX_LIST + h, r, ordinal, &a, &b);
                pos[h] = lg ? (a >> (32 - lg)) : 0u;
                pick[h] = np->npat > 1 ? umulhi32(b, np->npat) : 0u;
            }
            int dup = 0;
            for (uint32_t h = 1; h < count; h++)
                for (uint32_t q = 0; q < h; q++) dup |= pos[h] == pos[q];
            if (!dup) break;
        }
        for (uint32_t h = 0; h < count; h++)
            if (pos[h] < vlen) emit(ctx, pos[h], pick[h]);
    } else {
        uint32_t needed = count;
        for (uint32_t i = 0; needed > 0; i++) {
            noise_block(tk, 0x80000000u + i, r, ordinal, w);
            if (umul64hi(((uint64_t)w[1] << 32) | w[0], (uint64_t)(L - i)) < needed) {
                if (i < vlen) emit(ctx, i, np->npat > 1 ? umulhi32(w[2], np->npat) : 0u);
                needed--;
            }
        }
    }
}

typedef struct {
    uint32_t* x; uint32_t* z; const int32_t* tg; int ar; int ch; int nw;
    uint32_t app0, shot0, lgcs;
} hit_ctx;

static const uint8_t DEP1_X[3] = {1, 1, 0}, DEP1_Z[3] = {0, 1, 1};

static inline void pattern_of(int ch, uint32_t pick, uint32_t* xm, uint32_t* zm) {
    switch (ch) {
        case CH_XERR: *xm = 1; *zm = 0; return;
        case CH_YERR: *xm = 1; *zm = 1; return;
        case CH_ZERR: *xm = 0; *zm = 1; return;
        case CH_DEP1: *xm = DEP1_X[pick]; *zm = DEP1_Z[pick]; return;
        default: {  /* DEPOLARIZE2 code = pick + 1, gates.py:98-104 */
            uint32_t code = pick + 1;
            *xm = (code & 1) | (((code >> 2) & 1) << 1);
            *zm = ((code >> 1) & 1) | (((code >> 3) & 1) << 1);
        }
    }
}

/* a hit at chunk position pos: application app0 + pos / cs, shot shot0 + pos % cs */
static void apply_hit(void* vctx, uint32_t pos, uint32_t pick) {
    hit_ctx* c = (hit_ctx*)vctx;
    uint32_t xm, zm;
    pattern_of(c->ch, pick, &xm, &zm);
    const uint32_t app = c->app0 + (pos >> c->lgcs);
    const uint32_t s = c->shot0 + (pos & ((1u << c->lgcs) - 1));
    const uint32_t bit = 1u << (s & 31);
    const uint32_t w = s >> 5;
    for (int sl = 0; sl < c->ar; sl++) {
        int32_t q = c->tg[app * c->ar + sl];
        if ((xm >> sl) & 1) c->x[(size_t)q * c->nw + w] ^= bit;
        if ((zm >> sl) & 1) c->z[(size_t)q * c->nw + w] ^= bit;
    }
}

/* coin words (32 shots each) of coin row e for the tile: word w is word
 * (w & 3) of Philox(e, w >> 2, g, DOMAIN_COIN) */
static inline void coin_words(const orc_job* jb, const tile_key* tk, int64_t e, int64_t local_tile, int nw,
                              uint32_t* dst) {
    if (jb->coins) {
        const uint32_t* src = jb->coins + e * jb->inject_words + local_tile * nw;
        memcpy(dst, src, sizeof(uint32_t) * nw);
        return;
    }
    uint32_t o[4];
    for (int w = 0; w < nw; w++) {
        if ((w & 3) == 0) {
            uint32_t ctr[4] = {(uint32_t)e, (uint32_t)(w >> 2), tk->g, DOMAIN_COIN};
            orc_philox4x32_10(ctr, tk->k, o);
        }
        dst[w] = o[w & 3];
    }
}

static void run_tile(const orc_job* jb, int64_t t, uint32_t* x, uint32_t* z, uint32_t* rec,
                     uint32_t* tmp) {
    const int nw = jb->T / 32;
    const int n = jb->num_qubits;
    const tile_key tk = make_key(jb->seed, jb->tile_offset + (uint64_t)t);
    /* FrameBatch.__init__: x = 0, z = coin rows 0..n-1 (frame_sim.py:36-39) */
    memset(x, 0, sizeof(uint32_t) * (size_t)n * nw);
    for (int q = 0; q < n; q++) coin_words(jb, &tk, q, t, nw, z + (size_t)q * nw);
    for (int64_t i = 0; i < jb->n_ins; i++) {
        const orc_instr* in = &jb->ins[i];
        const int32_t* tg = jb->targets + in->tgt_off;
        switch (in->kind) {
        case K_GATE: {
            int ar = (in->code >= R_CX) ? 2 : 1;
            for (int a = 0; a + ar <= in->n_targets; a += ar) {
                uint32_t* x0 = x + (size_t)tg[a] * nw; uint32_t* z0 = z + (size_t)tg[a] * nw;
                uint32_t* x1 = ar == 2 ? x + (size_t)tg[a + 1] * nw : NULL;
                uint32_t* z1 = ar == 2 ? z + (size_t)tg[a + 1] * nw : NULL;
                switch (in->code) {
                case R_SWAPXZ: for (int w = 0; w < nw; w++) { uint32_t v = x0[w]; x0[w] = z0[w]; z0[w] = v; } break;
                case R_ZXORX: for (int w = 0; w < nw; w++) z0[w] ^= x0[w]; break;
                case R_XXORZ: for (int w = 0; w < nw; w++) x0[w] ^= z0[w]; break;
                case R_CX: for (int w = 0; w < nw; w++) { x1[w] ^= x0[w]; z0[w] ^= z1[w]; } break;
                case R_CZ: for (int w = 0; w < nw; w++) { uint32_t a0 = x0[w], a1 = x1[w]; z0[w] ^= a1; z1[w] ^= a0; } break;
                case R_CY: for (int w = 0; w < nw; w++) {
                        uint32_t ox0 = x0[w], ox1 = x1[w], oz1 = z1[w];
                        z0[w] ^= ox1 ^ oz1; z1[w] = oz1 ^ ox0; x1[w] = ox1 ^ ox0; } break;
                case R_SWAP: for (int w = 0; w < nw; w++) {
                        uint32_t v = x0[w]; x0[w] = x1[w]; x1[w] = v;
                        v = z0[w]; z0[w] = z1[w]; z1[w] = v; } break;
                default: break;
                }
            }
            break;
        }
        case K_M: case K_R: case K_MR: {
            for (int j = 0; j < in->n_targets; j++) {
                uint32_t* xq = x + (size_t)tg[j] * nw; uint32_t* zq = z + (size_t)tg[j] * nw;
                if (in->kind == K_M) {
                    memcpy(rec + (size_t)(in->rec_base + j) * nw, xq, sizeof(uint32_t) * nw);
                    coin_words(jb, &tk, (int64_t)in->coin_base + j, t, nw, tmp);
                    for (int w = 0; w < nw; w++) zq[w] ^= tmp[w];
                } else if (in->kind == K_R) {
                    memset(xq, 0, sizeof(uint32_t) * nw);
                    coin_words(jb, &tk, (int64_t)in->coin_base + j, t, nw, zq);
                } else {
                    memcpy(rec + (size_t)(in->rec_base + j) * nw, xq, sizeof(uint32_t) * nw);
                    /* the measure's coin row (coin_base + 2j) is overwritten by the reset's */
                    memset(xq, 0, sizeof(uint32_t) * nw);
                    coin_words(jb, &tk, (int64_t)in->coin_base + 2 * j + 1, t, nw, zq);
                }
            }
            break;
        }
        case K_NOISE: {
            const int ar = in->code == CH_DEP2 ? 2 : 1;
            const int64_t nid = in->aux;
            if (jb->masks) {
                for (int j = 0; j < in->n_targets; j++) {
                    const uint32_t* mx = jb->masks + ((int64_t)in->noise_row_base + 2 * j) * jb->inject_words + t * nw;
                    const uint32_t* mz = mx + jb->inject_words;
                    uint32_t* xq = x + (size_t)tg[j] * nw; uint32_t* zq = z + (size_t)tg[j] * nw;
                    for (int w = 0; w < nw; w++) { xq[w] ^= mx[w]; zq[w] ^= mz[w]; }
                }
                break;
            }
            const orc_noise* np = &jb->noise[nid];
            if (np->zone == ZONE_NONE) break;
            uint32_t lgcs = 0;
            while ((1u << lgcs) < np->cs) lgcs++;
            const uint32_t nS = (uint32_t)jb->T / np->cs;
            for (uint32_t r = 0; r < np->nchunks; r++) {
                const uint32_t k = r / nS, cc = r % nS;
                const uint32_t left = np->apps - k * np->ca;
                const uint32_t na = left < np->ca ? left : np->ca;
                hit_ctx hc = {x, z, tg, ar, in->code, nw, k * np->ca, cc * np->cs, lgcs};
                noise_chunk(np, &tk, (uint32_t)nid, r, na * np->cs, apply_hit, &hc);
            }
            break;
        }
        default: break;  /* K_DET / K_OBS evaluated below from the full record */
        }
    }

    /* tail mask for shots past num_shots in the last tile */
    int64_t first_shot = t * (int64_t)jb->T;
    for (int w = 0; w < nw; w++) {
        int64_t s0 = first_shot + 32 * (int64_t)w;
        uint32_t m = s0 >= jb->num_shots ? 0u
                   : (jb->num_shots - s0 >= 32 ? 0xFFFFFFFFu : ((1u << (jb->num_shots - s0)) - 1u));
        tmp[w] = m;
    }
    if (jb->flips) {
        for (int64_t m = 0; m < jb->num_meas; m++)
            for (int w = 0; w < nw; w++)
                jb->flips[m * jb->out_words + t * nw + w] = rec[(size_t)m * nw + w] & tmp[w];
    }
    if (jb->events) {
        /* detector_events: XOR of flip bits per detector (io_formats.py:208-227) */
        for (int64_t d = 0; d < jb->num_cols; d++) {
            uint32_t* dst = jb->events + d * jb->out_words + t * nw;
            for (int w = 0; w < nw; w++) dst[w] = 0;
            for (int64_t e = jb->det_ptr[d]; e < jb->det_ptr[d + 1]; e++) {
                const uint32_t* src = rec + (size_t)jb->det_idx[e] * nw;
                for (int w = 0; w < nw; w++) dst[w] ^= src[w];
            }
            for (int w = 0; w < nw; w++) dst[w] &= tmp[w];
        }
    }
}

static void* worker_main(void* arg) {
    orc_worker* wk = (orc_worker*)arg;
    const orc_job* jb = wk->job;
    const int nw = jb->T / 32;
    size_t nq = (size_t)jb->num_qubits * nw;
    uint32_t* x = (uint32_t*)malloc(sizeof(uint32_t) * (nq + 1));
    uint32_t* z = (uint32_t*)malloc(sizeof(uint32_t) * (nq + 1));
    uint32_t* rec = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)jb->num_meas * nw + 1));
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (nw + 4));
    if (!x || !z || !rec || !tmp) { wk->rc = -2; free(x); free(z); free(rec); free(tmp); return NULL; }
    for (int64_t t = wk->tid; t < jb->n_tiles; t += jb->nthreads) run_tile(jb, t, x, z, rec, tmp);
    free(x); free(z); free(rec); free(tmp);
    wk->rc = 0;
    return NULL;
}

/*
 * Sample num_shots shots in tiles of tile_shots (T) shots, noise chunks of
 * chunk_L[ordinal] trials and vectors of vector_shots (S) shots.  Outputs are
 * row-major bit tables [rows][out_words] (shot s = bit s%32 of word s/32) for
 * measurement flips and/or detection events (detector columns then
 * observables).  Returns 0 or a negative error code.
 */
int orc_sample(const orc_instr* ins, int64_t n_ins, const int32_t* targets,
               const double* noise_p, int64_t n_noise, const uint32_t* chunk_L, int32_t vector_shots,
               int32_t num_qubits, int64_t num_meas,
               const int64_t* det_ptr, const int64_t* det_idx, int64_t num_cols,
               int64_t num_shots, int32_t tile_shots, uint64_t seed, uint64_t tile_offset,
               const uint32_t* coins, const uint32_t* masks, int64_t inject_words,
               uint32_t* flips, uint32_t* events, int64_t out_words, int nthreads) {
    if (tile_shots <= 0 || tile_shots % 32) return -1;
    if (num_shots < 1) return -1;
    orc_noise* noise = NULL;
    if (n_noise > 0 && !masks) {
        noise = (orc_noise*)calloc((size_t)n_noise, sizeof(orc_noise));
        if (!noise) return -2;
        for (int64_t i = 0; i < n_ins; i++) {
            if (ins[i].kind != K_NOISE) continue;
            const int ar = ins[i].code == CH_DEP2 ? 2 : 1;
            const int64_t o = ins[i].aux;
            if (o < 0 || o >= n_noise) { free(noise); return -6; }
            if (schedule_one(&noise[o], (uint32_t)(ins[i].n_targets / ar), ins[i].code, noise_p[o], chunk_L[o],
                             (uint32_t)tile_shots, (uint32_t)vector_shots)) {
                free(noise);
                return -7;
            }
        }
    }
    orc_job jb = {ins, n_ins, targets, noise_p, noise, num_qubits, num_meas,
                  det_ptr, det_idx, num_cols, num_shots, tile_shots, seed, tile_offset,
                  coins, masks, inject_words, flips, events, out_words,
                  (num_shots + tile_shots - 1) / tile_shots, nthreads < 1 ? 1 : nthreads};
    if (out_words < jb.n_tiles * (tile_shots / 32)) { free(noise); return -3; }
    if ((coins || masks) && inject_words < jb.n_tiles * (tile_shots / 32)) { free(noise); return -4; }
    int nth = jb.nthreads;
    if (nth > jb.n_tiles) { nth = (int)jb.n_tiles; jb.nthreads = nth; }
    orc_worker* wk = (orc_worker*)calloc((size_t)nth, sizeof(orc_worker));
    pthread_t* th = (pthread_t*)calloc((size_t)nth, sizeof(pthread_t));
    if (!wk || !th) { free(wk); free(th); free(noise); return -2; }
    for (int i = 0; i < nth; i++) {
        wk[i].job = &jb; wk[i].tid = i; wk[i].rc = -5;
        if (nth == 1) worker_main(&wk[i]);
        else pthread_create(&th[i], NULL, worker_main, &wk[i]);
    }
    int rc = 0;
    for (int i = 0; i < nth; i++) {
        if (nth > 1) pthread_join(th[i], NULL);
        if (wk[i].rc) rc = wk[i].rc;
    }
    free(wk); free(th); free(noise);
    return rc;
}

/*
 * Row-major bit table -> shot-major b8 bytes (bitvec.transposed + write_b8):
 * out[s * pitch + r/8] bit r%8 = rows[r][s] ^ xor_bits[r] (xor_bits may be NULL).
 * 8x8 bit-block transposes, shot blocks split over nthreads threads.
 */
typedef struct {
    const uint32_t* rows; int64_t num_rows, num_shots, row_words;
    const uint8_t* xor_bits; uint8_t* out; int64_t pitch;
    int64_t s0, s1;
} b8_job;

static inline uint64_t transpose8x8(uint64_t x) {
    /* byte i = row i (bit j = column j) -> byte j = column j (bit i = row i) */
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull; x ^= t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull; x ^= t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull; x ^= t ^ (t << 28);
    return x;
}

static void* b8_worker(void* arg) {
    const b8_job* j = (const b8_job*)arg;
    const int64_t nb = (j->num_rows + 7) / 8;
    /* 512 shots (one 64-byte line of every row) at a time: the 8 input lines of a
     * row block are used up before the next block is touched, and the 512 output
     * lines stay cached while the row blocks fill them byte by byte -- whatever
     * the row pitch (a power-of-two pitch maps every row to one cache set). */
    for (int64_t c0 = j->s0; c0 < j->s1; c0 += 512) {
        const int64_t c1 = c0 + 512 < j->s1 ? c0 + 512 : j->s1;
        for (int64_t rb = 0; rb < nb; rb++) {              /* 8 rows */
            const int nr = (int)(j->num_rows - rb * 8 < 8 ? j->num_rows - rb * 8 : 8);
            const uint8_t last_mask = (rb == nb - 1 && (j->num_rows & 7)) ? (uint8_t)((1u << (j->num_rows & 7)) - 1) : 0xFFu;
            uint32_t flip[8];
            for (int i = 0; i < nr; i++)
                flip[i] = (j->xor_bits && (j->xor_bits[rb * 8 + i] & 1)) ? 0xFFu : 0u;
            for (int64_t s8 = c0; s8 < c1; s8 += 8) {      /* 8 shots */
                uint64_t blk = 0;
                for (int i = 0; i < nr; i++) {
                    const uint32_t* row = j->rows + (rb * 8 + i) * j->row_words;
                    uint32_t byte = ((row[s8 >> 5] >> (s8 & 31)) & 0xFFu) ^ flip[i];
                    blk |= (uint64_t)byte << (8 * i);
                }
                blk = transpose8x8(blk);
                for (int k = 0; k < 8 && s8 + k < j->num_shots; k++)
                    j->out[(s8 + k) * j->pitch + rb] = (uint8_t)(blk >> (8 * k)) & last_mask;
            }
        }
    }
    return NULL;
}

void orc_rows_to_b8(const uint32_t* rows, int64_t num_rows, int64_t num_shots, int64_t row_words,
                    const uint8_t* xor_bits, uint8_t* out, int64_t pitch, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    const int64_t blocks = (num_shots + 7) / 8;
    if (nthreads > blocks) nthreads = (int)(blocks > 0 ? blocks : 1);
    b8_job* jobs = (b8_job*)calloc((size_t)nthreads, sizeof(b8_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return; }
    for (int i = 0; i < nthreads; i++) {
        b8_job j = {rows, num_rows, num_shots, row_words, xor_bits, out, pitch,
                    8 * (blocks * i / nthreads), 8 * (blocks * (i + 1) / nthreads)};
        jobs[i] = j;
        if (nthreads == 1) b8_worker(&jobs[i]);
        else pthread_create(&th[i], NULL, b8_worker, &jobs[i]);
    }
    if (nthreads > 1)
        for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(jobs);
    free(th);
}
