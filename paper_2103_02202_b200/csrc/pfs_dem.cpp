// Detector error model: the output signature of every noise component
// ("sparse / error-model detector sampling",
// not implemented by the paper or the reference).
//
// The frame simulation is linear over GF(2): the detection events of a shot are
// the XOR, over everything random that happened in it, of that event's effect
// on the output columns (detectors, then observables; detector_events =
// XOR of record flips, stabsim/io_formats.py:208-227).  Walking the flat
// program backwards with per-qubit sensitivity sets S_x[q], S_z[q] ("the
// columns an X / Z frame flip on q at this point would flip") gives
//   * at M q (record m): S_x[q] ^= cols(m)    (an X before M flips the record,
//     stabsim/frame_sim.py:74-80);
//   * at R / MR: S_x[q] = S_z[q] = {}         (frame_sim.py:82-90);
//   * at a gate: the transpose of its frame rule (gates.py:70-92), e.g. CX:
//     S_x0 ^= S_x1, S_z1 ^= S_z0;
//   * at a noise instruction: the component signatures (x / z on each slot) of
//     every application, read off the current sets.
// The randomness the frame simulation also injects — the z coin rows of
// FrameBatch.__init__, M, R, MR — enters the same way as a Z flip; when every
// such coin has an empty signature (all deterministic-detector circuits: QEC
// memories) the events depend on the noise draws alone, and a shot's events
// are the XOR of the signatures of its noise hits.  Sampling then costs O(hits)
// per shot instead of O(gates), with the identical counter-based noise draws
// — so the output equals the frame sampler's bit for bit.
#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "pfs_internal.h"

namespace pfs {

namespace {

using Set = std::vector<uint32_t>;  // sorted column indices

void xor_into(Set& a, const Set& b) {
    if (b.empty()) return;
    Set out;
    out.reserve(a.size() + b.size());
    size_t i = 0, j = 0;
    while (i < a.size() || j < b.size()) {
        if (j == b.size() || (i < a.size() && a[i] < b[j])) out.push_back(a[i++]);
        else if (i == a.size() || b[j] < a[i]) out.push_back(b[j++]);
        else { i++; j++; }  // in both: cancels
    }
    a.swap(out);
}

}  // namespace

DemModel build_dem(const pfs_instr* ins, int64_t n_ins, const int32_t* targets, const int64_t* det_ptr,
                   const int64_t* det_idx, int64_t n_cols, int32_t num_qubits, int64_t num_meas,
                   int64_t n_noise) {
    DemModel dm;
    // columns of each record (detectors and observables, det CSR)
    std::vector<Set> rec_cols(num_meas);
    for (int64_t c = 0; c < n_cols; c++)
        for (int64_t e = det_ptr[c]; e < det_ptr[c + 1]; e++) {
            const int64_t m = det_idx[e];
            if (m >= 0 && m < num_meas) xor_into(rec_cols[m], Set{(uint32_t)c});
        }
    std::vector<Set> sx(num_qubits), sz(num_qubits);
    // per noise ordinal: apps x 4 component signatures (flat CSR per ordinal),
    // filled backwards
    std::vector<std::vector<uint32_t>> cptr(n_noise), ccols(n_noise);
    auto coin = [&](int32_t q, const char* what) {
        if (!sz[q].empty() && dm.coin_dependent.empty())
            dm.coin_dependent = std::string("the ") + what + " coin of qubit " + std::to_string(q) +
                                " reaches output column " + std::to_string(sz[q][0]) +
                                ": its detectors depend on measurement randomness";
    };
    for (int64_t i = n_ins - 1; i >= 0; i--) {
        const pfs_instr& in = ins[i];
        const int32_t* tg = targets + in.tgt_off;
        switch (in.kind) {
        case K_GATE: {
            const int ar = in.code >= R_CX ? 2 : 1;
            for (int j = in.n_targets - ar; j >= 0; j -= ar) {  // applications in reverse
                const int32_t a = tg[j], b = ar == 2 ? tg[j + 1] : -1;
                switch (in.code) {
                    case R_SWAPXZ: sx[a].swap(sz[a]); break;
                    case R_ZXORX: xor_into(sx[a], sz[a]); break;   // X -> X Z
                    case R_XXORZ: xor_into(sz[a], sx[a]); break;   // Z -> X Z
                    case R_CX: xor_into(sx[a], sx[b]); xor_into(sz[b], sz[a]); break;
                    case R_CZ: xor_into(sx[a], sz[b]); xor_into(sx[b], sz[a]); break;
                    case R_CY: {  // X0 -> X0 X1 Z1, X1 -> X1 Z0, Z1 -> Z1 Z0
                        Set x0 = sx[a];
                        xor_into(x0, sx[b]);
                        xor_into(x0, sz[b]);
                        xor_into(sx[b], sz[a]);
                        xor_into(sz[b], sz[a]);
                        sx[a].swap(x0);
                        break;
                    }
                    default: sx[a].swap(sx[b]); sz[a].swap(sz[b]); break;  // SWAP
                }
            }
            break;
        }
        case K_M:
            for (int j = in.n_targets - 1; j >= 0; j--) {
                const int32_t q = tg[j];
                coin(q, "measurement");
                xor_into(sx[q], rec_cols[in.rec_base + j]);
            }
            break;
        case K_MR:
            for (int j = in.n_targets - 1; j >= 0; j--) {
                const int32_t q = tg[j];
                coin(q, "reset");
                sx[q].clear();
                sz[q].clear();
                xor_into(sx[q], rec_cols[in.rec_base + j]);
            }
            break;
        case K_R:
            for (int j = in.n_targets - 1; j >= 0; j--) {
                const int32_t q = tg[j];
                coin(q, "reset");
                sx[q].clear();
                sz[q].clear();
            }
            break;
        case K_NOISE: {
            const int ar = in.code == CH_DEP2 ? 2 : 1;
            const int apps = in.n_targets / ar;
            std::vector<uint32_t>& pp = cptr[in.aux];
            std::vector<uint32_t>& cc = ccols[in.aux];
            pp.assign(1, 0u);
            cc.clear();
            for (int a2 = 0; a2 < apps; a2++)
                for (int s = 0; s < 2; s++) {
                    const bool has = s < ar;
                    const int32_t q = has ? tg[a2 * ar + s] : 0;
                    if (has) cc.insert(cc.end(), sx[q].begin(), sx[q].end());
                    pp.push_back((uint32_t)cc.size());
                    if (has) cc.insert(cc.end(), sz[q].begin(), sz[q].end());
                    pp.push_back((uint32_t)cc.size());
                }
            break;
        }
        default: break;  // DETECTOR / OBSERVABLE_INCLUDE act through rec_cols
        }
    }
    for (int32_t q = 0; q < num_qubits; q++) coin(q, "initial");
    // flatten: comp_base[o] = first component of ordinal o; comp_ptr CSR
    dm.comp_base.resize(n_noise + 1);
    dm.comp_ptr.push_back(0);
    uint64_t total = 0;
    for (int64_t o = 0; o < n_noise; o++) {
        dm.comp_base[o] = (uint32_t)(dm.comp_ptr.size() - 1);
        const uint64_t base = dm.cols.size();
        if (base + ccols[o].size() > 0xFFFFFFFFull) throw std::invalid_argument("error model too large");
        dm.cols.insert(dm.cols.end(), ccols[o].begin(), ccols[o].end());
        total += ccols[o].size();
        for (size_t k = 1; k < cptr[o].size(); k++) dm.comp_ptr.push_back((uint32_t)(base + cptr[o][k]));
        std::vector<uint32_t>().swap(ccols[o]);
        std::vector<uint32_t>().swap(cptr[o]);
    }
    dm.comp_base[n_noise] = (uint32_t)(dm.comp_ptr.size() - 1);
    // packed component words: a hit's columns in one load (most components of a
    // QEC memory reach 1-2 detectors)
    const bool inline_ok = n_cols < (1ll << 20);
    const size_t ncomp = dm.comp_ptr.size() - 1;
    dm.comp_words.resize(ncomp);
    for (size_t k = 0; k < ncomp; k++) {
        const uint32_t b = dm.comp_ptr[k], n = dm.comp_ptr[k + 1] - b;
        unsigned long long w;
        if (inline_ok && n <= 3) {
            w = (unsigned long long)n << 62;
            for (uint32_t j = 0; j < n; j++) w |= (unsigned long long)dm.cols[b + j] << (20 * j);
        } else {
            if (n >= (1u << 30)) throw std::invalid_argument("error model component too large");
            w = (unsigned long long)b | ((unsigned long long)n << 32);
        }
        dm.comp_words[k] = w;
    }
    dm.mean_cols_per_comp = dm.comp_ptr.size() > 1 ? (double)total / (double)(dm.comp_ptr.size() - 1) : 0.0;
    return dm;
}

}  // namespace pfs
