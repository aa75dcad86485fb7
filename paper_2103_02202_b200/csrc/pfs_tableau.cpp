// Native inverse-tableau reference sampler.
//
// Restates `stabsim/tableau_sim.py` (SimState, reference_sample: lines
// 50-297, 326-329) in C++ with bit-packed columns:
//   * the state is the tableau of the INVERSE of the Clifford applied so far:
//     column X_c / Z_c holds the start-of-time Pauli equivalent to measuring
//     X_c / Z_c now (tableau_sim.py:1-8);
//   * folding a gate G replaces each column P by its image of G^-1 P G
//     (prepend; tableau.py:389-420) — H swaps columns, S and CX multiply
//     columns with phase tracking, Paulis negate signs;
//   * measuring Z_q is deterministic iff column Z_q has no X/Y term; its
//     sign is the result (tableau_sim.py:139-149);
//   * a random measurement collapses (tableau_sim.py:161-199): pivot = lowest
//     X/Y position of column Z_q, append CNOT(pivot, t) for every other such
//     position t, then H (or H_YZ when the pivot term is Y) on the pivot, and
//     an X on the pivot when the coin is 1 — appends act on every column at
//     those start-of-time positions;
//   * R resets the result sign to 0 after collapsing (tableau_sim.py:151-159).
// Gates are folded through H / S / CX / Pauli decompositions that give the
// reference's conjugation tables (stabsim/gates.py:107-140): S_DAG = S^3,
// SQRT_Y = Z then H, SQRT_Y_DAG = H then Z, SQRT_X = H S H,
// SQRT_X_DAG = H S^3 H, CZ = H_t CX H_t, CY = S_t^3 CX S_t, SWAP = 3 CX.
// Coins come from the caller in collapse order (the reference draws
// `rng.integers(2)` once per collapse, tableau_sim.py:177).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "pfs.h"

namespace {

thread_local std::string g_tab_error;

struct Tableau {
    int n = 0;
    size_t nw = 0;  // 64-bit words per column
    // column c of each plane: words [c * nw, (c + 1) * nw)
    std::vector<uint64_t> xx, xz, zx, zz;  // X-/Z-part of the X_c and Z_c columns
    std::vector<uint8_t> xs, zs;            // column signs

    explicit Tableau(int nq) : n(nq), nw(((size_t)nq + 63) / 64) {
        const size_t sz = (size_t)nq * nw;
        xx.assign(sz, 0); xz.assign(sz, 0); zx.assign(sz, 0); zz.assign(sz, 0);
        xs.assign(nq, 0); zs.assign(nq, 0);
        for (int c = 0; c < nq; c++) {
            xx[(size_t)c * nw + (c >> 6)] = 1ull << (c & 63);
            zz[(size_t)c * nw + (c >> 6)] = 1ull << (c & 63);
        }
    }
    uint64_t* X(std::vector<uint64_t>& v, int c) { return v.data() + (size_t)c * nw; }
};

// a <- a * b for Pauli strings (x, z bit vectors, Y = x & z); returns log_i
// of the scalar i^k with a_old * b = i^k * a_new (k mod 4, signs excluded).
uint32_t mul_into(uint64_t* ax, uint64_t* az, const uint64_t* bx, const uint64_t* bz, size_t nw) {
    // (cnt2, cnt1): a mod-4 counter per bit lane; only the total mod 4 matters,
    // so every word accumulates into the same 64 lanes
    uint64_t cnt1 = 0, cnt2 = 0;
    for (size_t w = 0; w < nw; w++) {
        const uint64_t x1 = ax[w], z1 = az[w], x2 = bx[w], z2 = bz[w];
        const uint64_t nx = x1 ^ x2, nz = z1 ^ z2;
        const uint64_t x1z2 = x1 & z2;
        const uint64_t anti = (x2 & z1) ^ x1z2;
        // per position: +i when the factors anticommute in cyclic order, -i otherwise
        cnt2 ^= (cnt1 ^ nx ^ nz ^ x1z2) & anti;
        cnt1 ^= anti;
        ax[w] = nx;
        az[w] = nz;
    }
    return ((uint32_t)__builtin_popcountll(cnt1) + 2u * (uint32_t)__builtin_popcountll(cnt2)) & 3u;
}

// ---- folds (prepend G: column P -> column of G^-1 P G) ----
void fold_h(Tableau& t, int q) {
    std::swap_ranges(t.X(t.xx, q), t.X(t.xx, q) + t.nw, t.X(t.zx, q));
    std::swap_ranges(t.X(t.xz, q), t.X(t.xz, q) + t.nw, t.X(t.zz, q));
    std::swap(t.xs[q], t.zs[q]);
}

// S^-1 X S = -Y = -i X Z: column X_q <- -i (X_q * Z_q); Z_q unchanged
void fold_s(Tableau& t, int q) {
    const uint32_t k = mul_into(t.X(t.xx, q), t.X(t.xz, q), t.X(t.zx, q), t.X(t.zz, q), t.nw);
    const uint32_t ph = (k + 3u) & 3u;  // times -i
    t.xs[q] = (uint8_t)(t.xs[q] ^ t.zs[q] ^ (ph >> 1));
}

// CX^-1 X_c CX = X_c X_t, CX^-1 Z_t CX = Z_c Z_t (commuting: real phase)
void fold_cx(Tableau& t, int c, int tq) {
    uint32_t k = mul_into(t.X(t.xx, c), t.X(t.xz, c), t.X(t.xx, tq), t.X(t.xz, tq), t.nw);
    t.xs[c] = (uint8_t)(t.xs[c] ^ t.xs[tq] ^ (k >> 1));
    // Z_t <- Z_c * Z_t = Z_t * Z_c (the images commute: same phase either order)
    k = mul_into(t.X(t.zx, tq), t.X(t.zz, tq), t.X(t.zx, c), t.X(t.zz, c), t.nw);
    t.zs[tq] = (uint8_t)(t.zs[tq] ^ t.zs[c] ^ (k >> 1));
}

void fold_x(Tableau& t, int q) { t.zs[q] ^= 1; }
void fold_z(Tableau& t, int q) { t.xs[q] ^= 1; }

// ---- collapse (appends at start-of-time positions, every column) ----
inline bool bit(const uint64_t* v, int j) { return (v[j >> 6] >> (j & 63)) & 1ull; }
inline void flip(uint64_t* v, int j) { v[j >> 6] ^= 1ull << (j & 63); }

void collapse(Tableau& t, int q, int coin) {
    const uint64_t* zxq = t.X(t.zx, q);
    int pivot = -1;
    std::vector<int> partners;
    for (size_t w = 0; w < t.nw; w++) {
        uint64_t b = zxq[w];
        while (b) {
            const int j = (int)(w * 64) + __builtin_ctzll(b);
            if (pivot < 0) pivot = j; else partners.push_back(j);
            b &= b - 1;
        }
    }
    if (pivot < 0) return;
    // the pivot term of column Z_q after the CNOT appends decides H vs H_YZ:
    // CNOT(p, t) leaves z_p ^= z_t, so it is the z bit of p xor the z bits of
    // the partners
    bool pivot_is_y = bit(t.X(t.zz, q), pivot);
    for (int tq : partners) pivot_is_y ^= bit(t.X(t.zz, q), tq);
    auto apply = [&](uint64_t* x, uint64_t* z, uint8_t& s) {
        // CNOT(pivot, tq): sign ^= x_p z_t (x_t ^ z_p ^ 1); x_t ^= x_p; z_p ^= z_t
        bool xp = bit(x, pivot), zp = bit(z, pivot);
        for (int tq : partners) {
            const bool xt = bit(x, tq), zt = bit(z, tq);
            if (xp && zt && !(xt ^ zp)) s ^= 1;
            if (xp) flip(x, tq);
            if (zt) zp = !zp;
        }
        if (pivot_is_y) {  // H_YZ: sign flips on pure X; x ^= z
            if (xp && !zp) s ^= 1;
            xp = xp ^ zp;
        } else {           // H: sign flips on Y; swap
            if (xp && zp) s ^= 1;
            const bool tmp = xp; xp = zp; zp = tmp;
        }
        if (coin && zp) s ^= 1;  // X on the pivot negates Z / Y terms there
        if (bit(x, pivot) != xp) flip(x, pivot);
        if (bit(z, pivot) != zp) flip(z, pivot);
    };
    // columns are independent: wide tableaus split them across host threads
#pragma omp parallel for schedule(static) if (t.n >= 4096)
    for (int c = 0; c < t.n; c++) {
        apply(t.X(t.xx, c), t.X(t.xz, c), t.xs[c]);
        apply(t.X(t.zx, c), t.X(t.zz, c), t.zs[c]);
    }
}

bool random_z(Tableau& t, int q) {
    const uint64_t* zxq = t.X(t.zx, q);
    for (size_t w = 0; w < t.nw; w++)
        if (zxq[w]) return true;
    return false;
}

}  // namespace

extern "C" {

const char* pfs_reference_sample_error(void) { return g_tab_error.c_str(); }

int pfs_reference_sample(const int32_t* ops, int64_t n_ops, const int32_t* targets, int64_t n_targets,
                         int32_t num_qubits, const uint8_t* coins, int64_t n_coins, uint8_t* out_bits,
                         uint8_t* out_determined, int64_t n_out, int64_t* n_written) {
    g_tab_error.clear();
    if (num_qubits < 0 || n_ops < 0 || n_targets < 0 || n_coins < 0 || n_out < 0) {
        g_tab_error = "negative size";
        return PFS_E_INVALID;
    }
    if ((n_ops && !ops) || (n_targets && !targets) || (n_coins && !coins) || (n_out && !out_bits)) {
        g_tab_error = "null argument";
        return PFS_E_INVALID;
    }
    try {
        Tableau t(num_qubits);
        int64_t rec = 0, ci = 0;
        auto need_coin = [&]() -> int {
            if (ci >= n_coins) throw std::string("coin stream exhausted");
            return coins[ci++] & 1;
        };
        for (int64_t i = 0; i < n_ops; i++) {
            const int32_t code = ops[3 * i], nt = ops[3 * i + 1], off = ops[3 * i + 2];
            if (nt < 0 || off < 0 || (int64_t)off + nt > n_targets) throw std::string("target range out of bounds");
            const int32_t* tg = targets + off;
            for (int j = 0; j < nt; j++)
                if (tg[j] < 0 || tg[j] >= num_qubits)
                    throw "qubit " + std::to_string(tg[j]) + " out of range [0, " + std::to_string(num_qubits) + ")";
            const int ar = code >= PFS_TG_CX && code <= PFS_TG_SWAP ? 2 : 1;
            if (nt % ar) throw std::string("target count not a multiple of the gate arity");
            for (int j = 0; j < nt; j += ar) {
                const int a = tg[j], b = ar == 2 ? tg[j + 1] : -1;
                if (ar == 2 && a == b) throw std::string("two-qubit gate targets a qubit pair twice");
                switch (code) {
                    case PFS_TG_I: break;
                    case PFS_TG_X: fold_x(t, a); break;
                    case PFS_TG_Y: fold_x(t, a); fold_z(t, a); break;
                    case PFS_TG_Z: fold_z(t, a); break;
                    case PFS_TG_H: fold_h(t, a); break;
                    case PFS_TG_S: fold_s(t, a); break;
                    case PFS_TG_S_DAG: fold_s(t, a); fold_s(t, a); fold_s(t, a); break;
                    case PFS_TG_SQRT_X: fold_h(t, a); fold_s(t, a); fold_h(t, a); break;
                    case PFS_TG_SQRT_X_DAG:
                        fold_h(t, a); fold_s(t, a); fold_s(t, a); fold_s(t, a); fold_h(t, a); break;
                    case PFS_TG_SQRT_Y: fold_z(t, a); fold_h(t, a); break;
                    case PFS_TG_SQRT_Y_DAG: fold_h(t, a); fold_z(t, a); break;
                    case PFS_TG_CX: fold_cx(t, a, b); break;
                    case PFS_TG_CY:
                        fold_s(t, b); fold_s(t, b); fold_s(t, b); fold_cx(t, a, b); fold_s(t, b); break;
                    case PFS_TG_CZ: fold_h(t, b); fold_cx(t, a, b); fold_h(t, b); break;
                    case PFS_TG_SWAP: fold_cx(t, a, b); fold_cx(t, b, a); fold_cx(t, a, b); break;
                    case PFS_TG_M: case PFS_TG_MR: {
                        const bool rnd = random_z(t, a);
                        if (rnd) collapse(t, a, need_coin());
                        if (rec >= n_out) throw std::string("output buffer too small");
                        out_bits[rec] = t.zs[a];
                        if (out_determined) out_determined[rec] = rnd ? 0 : 1;
                        rec++;
                        if (code == PFS_TG_MR) t.zs[a] = 0;
                        break;
                    }
                    case PFS_TG_R:
                        if (random_z(t, a)) collapse(t, a, need_coin());
                        t.zs[a] = 0;
                        break;
                    default: throw "unknown gate code " + std::to_string(code);
                }
            }
        }
        if (n_written) *n_written = rec;
    } catch (const std::string& e) {
        g_tab_error = e;
        return PFS_E_INVALID;
    } catch (const std::bad_alloc&) {
        g_tab_error = "out of host memory";
        return PFS_E_NOMEM;
    }
    return PFS_OK;
}

}  // extern "C"
