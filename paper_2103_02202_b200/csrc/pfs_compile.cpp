// Host-side circuit compiler: flat frame program -> device op list.
//
// Replaces the per-call `compile_frame_program` (stabsim/frame_sim.py:170-189)
// with a one-time native pass that prepares the op stream the persistent CUDA
// kernel interprets:
//   * split every instruction at the first repeated qubit, so each device op is
//     a set of independent applications (the reference applies an
//     instruction's applications sequentially, frame_sim.py:61-62, 196-197 —
//     `CX 0 1 1 2` must stay two steps);
//   * merge consecutive instructions of the same frame rule / collapse kind
//     when they touch disjoint qubits (fewer ops, fewer barriers);
//   * allocate measurement-record ring slots by liveness: a record lives from
//     its M until the last DETECTOR / OBSERVABLE_INCLUDE that reads it
//     (detector sets: stabsim/circuit.py:247-256);
//   * schedule __syncthreads: a barrier goes before an op only if it touches a
//     qubit row or record slot already touched since the previous barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "pfs_internal.h"

namespace pfs {

namespace {

int rule_arity(int32_t rule) { return rule >= R_CX ? 2 : 1; }

int64_t rule_bits(int32_t rule) {
    switch (rule) {
        case R_SWAPXZ: return 4;
        case R_ZXORX: case R_XXORZ: return 3;
        case R_CX: case R_CZ: return 6;
        case R_CY: return 7;
        case R_SWAP: return 8;
        default: return 0;
    }
}

[[noreturn]] void bad(const std::string& msg) { throw std::invalid_argument(msg); }

}  // namespace

HostProgram compile_program(const pfs_instr* ins, int64_t n_ins, const int32_t* targets,
                            int64_t n_targets, const double* noise_p, int64_t n_noise,
                            const int64_t* det_ptr, const int64_t* det_idx, int64_t n_cols,
                            int64_t n_obs, int32_t num_qubits, int64_t num_meas,
                            int64_t num_coin_rows, int64_t num_noise_rows) {
    if (num_qubits < 0 || num_meas < 0 || n_cols < 0 || n_obs < 0 || n_obs > n_cols)
        bad("negative sizes");
    if (n_ins > 0 && (!ins || (n_targets > 0 && !targets))) bad("null instruction arrays");
    if (n_cols > 0 && (!det_ptr)) bad("null detector arrays");
    const int64_t n_det = n_cols - n_obs;
    HostProgram hp;
    hp.num_qubits = num_qubits;
    hp.num_meas = num_meas;
    hp.num_cols = n_cols;
    hp.num_obs = n_obs;
    hp.num_noise = n_noise;
    hp.num_coin_rows = num_coin_rows;
    hp.num_noise_rows = num_noise_rows;
    hp.noise_p.assign(noise_p, noise_p + n_noise);
    hp.noise_apps.assign(n_noise, 0);
    hp.noise_arity.assign(n_noise, 1);
    hp.noise_off.assign(n_noise, 0);
    hp.noise_ch.assign(n_noise, 0);
    hp.noise.assign(n_noise, NoiseParam{});
    for (int64_t i = 0; i < n_noise; i++) {
        double p = noise_p[i];
        if (!(p >= 0.0 && p <= 1.0)) bad("noise probability must be in [0, 1], got " + std::to_string(p));
    }

    // ---- pass 1: validate and compute record liveness ----
    std::vector<int64_t> last_use(num_meas, -1);
    {
        int64_t rec = 0, coin = num_qubits, nrow = 0, col = 0;
        for (int64_t i = 0; i < n_ins; i++) {
            const pfs_instr& in = ins[i];
            if (in.n_targets < 0 || in.tgt_off < 0 || (int64_t)in.tgt_off + in.n_targets > n_targets)
                bad("instruction " + std::to_string(i) + ": target range out of bounds");
            const int32_t* tg = targets + in.tgt_off;
            switch (in.kind) {
            case K_GATE:
                if (in.code <= R_NONE || in.code > R_SWAP) bad("unknown frame rule");
                if (in.n_targets % rule_arity(in.code)) bad("gate target count not a multiple of arity");
                for (int j = 0; j < in.n_targets; j++)
                    if (tg[j] < 0 || tg[j] >= num_qubits)
                        bad("qubit " + std::to_string(tg[j]) + " out of range [0, " + std::to_string(num_qubits) + ")");
                for (int j = 0; j + 1 < in.n_targets && rule_arity(in.code) == 2; j += 2)
                    if (tg[j] == tg[j + 1]) bad("two-qubit gate targets a qubit pair twice");
                hp.bframe_bits += rule_bits(in.code) * (in.n_targets / rule_arity(in.code));
                break;
            case K_M: case K_R: case K_MR:
                for (int j = 0; j < in.n_targets; j++)
                    if (tg[j] < 0 || tg[j] >= num_qubits)
                        bad("qubit " + std::to_string(tg[j]) + " out of range [0, " + std::to_string(num_qubits) + ")");
                if (in.kind != K_R && in.rec_base != rec) bad("record numbering is not contiguous");
                if (in.coin_base != coin) bad("coin row numbering is not contiguous");
                if (in.kind != K_R) rec += in.n_targets;
                coin += (int64_t)in.n_targets * (in.kind == K_MR ? 2 : 1);
                hp.bframe_bits += (in.kind == K_R ? 2 : 4) * (int64_t)in.n_targets;
                break;
            case K_NOISE: {
                if (in.code < CH_XERR || in.code > CH_DEP2) bad("unknown noise channel");
                int ar = in.code == CH_DEP2 ? 2 : 1;
                if (in.n_targets % ar) bad("noise target count not a multiple of arity");
                for (int j = 0; j < in.n_targets; j++)
                    if (tg[j] < 0 || tg[j] >= num_qubits)
                        bad("qubit " + std::to_string(tg[j]) + " out of range [0, " + std::to_string(num_qubits) + ")");
                if (in.aux < 0 || in.aux >= n_noise) bad("noise ordinal out of range");
                if (in.noise_row_base != nrow) bad("noise row numbering is not contiguous");
                hp.noise_apps[in.aux] = (uint32_t)(in.n_targets / ar);
                hp.noise_arity[in.aux] = (uint32_t)ar;
                hp.noise[in.aux].npat = in.code == CH_DEP1 ? 3u : (in.code == CH_DEP2 ? 15u : 1u);
                nrow += 2 * (int64_t)in.n_targets;
                break;
            }
            case K_DET: {
                if (in.aux != col || col >= n_det) bad("detector columns out of order");
                for (int64_t e = det_ptr[col]; e < det_ptr[col + 1]; e++) {
                    int64_t m = det_idx[e];
                    if (m < 0 || m >= rec)
                        bad("detector " + std::to_string(col) + " references measurement " +
                            std::to_string(m) + ", have " + std::to_string(rec));
                    last_use[m] = i;
                }
                col++;
                break;
            }
            case K_OBS:
                if (in.aux < n_det || in.aux >= n_cols) bad("observable column out of range");
                for (int j = 0; j < in.n_targets; j++) {
                    int64_t m = tg[j];
                    if (m < 0 || m >= rec) bad("observable references a future measurement");
                    last_use[m] = i;
                }
                break;
            default:
                bad("unknown instruction kind " + std::to_string(in.kind));
            }
        }
        if (rec != num_meas) bad("measurement count mismatch");
        if (col != n_det) bad("detector count mismatch");
        if (coin != num_coin_rows) bad("coin row count mismatch");
        if (nrow != num_noise_rows) bad("noise row count mismatch");
    }

    // ---- pass 2: emit device ops, allocating record slots ----
    std::vector<uint32_t> slot_of(num_meas, NO_SLOT);
    std::vector<uint32_t> free_slots;
    uint32_t next_slot = (uint32_t)n_obs;  // [0, n_obs) = observable accumulators
    std::vector<int64_t> stamp(num_qubits, -1);
    int64_t cur = -1;  // open (mergeable) op index
    auto open_op = [&](uint32_t kind, uint32_t code) {
        // ops read their targets as uint2 pairs (two-qubit rules, (qubit, slot)
        // pairs of M/MR): keep every op's target list 8-byte aligned
        if (hp.targets.size() & 1) hp.targets.push_back(0u);
        DOp op{};
        op.kcf = kind | (code << 8);
        op.off = (uint32_t)hp.targets.size();
        hp.ops.push_back(op);
        cur = (int64_t)hp.ops.size() - 1;
    };
    auto kind_of = [&](int64_t k) { return hp.ops[k].kcf & 0xFF; };
    auto code_of = [&](int64_t k) { return (hp.ops[k].kcf >> 8) & 0xFF; };
    auto alloc = [&]() -> uint32_t {
        if (!free_slots.empty()) { uint32_t s = free_slots.back(); free_slots.pop_back(); return s; }
        return next_slot++;
    };
    hp.det_ptr.assign(1, 0);
    auto release_after = [&](int64_t i, int64_t m) {
        if (last_use[m] == i && slot_of[m] != NO_SLOT) { free_slots.push_back(slot_of[m]); slot_of[m] = NO_SLOT; }
    };

    for (int64_t i = 0; i < n_ins; i++) {
        const pfs_instr& in = ins[i];
        const int32_t* tg = targets + in.tgt_off;
        switch (in.kind) {
        case K_GATE: {
            const int ar = rule_arity(in.code);
            for (int j = 0; j < in.n_targets; j += ar) {
                bool conflict = cur < 0 || kind_of(cur) != K_GATE || code_of(cur) != (uint32_t)in.code;
                for (int s = 0; s < ar && !conflict; s++) conflict = stamp[tg[j + s]] == cur;
                if (conflict) open_op(K_GATE, in.code);
                for (int s = 0; s < ar; s++) { hp.targets.push_back((uint32_t)tg[j + s]); stamp[tg[j + s]] = cur; }
                hp.ops[cur].count++;
            }
            break;
        }
        case K_M: case K_MR: case K_R: {
            const bool records = in.kind != K_R;
            const int coin_per = in.kind == K_MR ? 2 : 1;
            for (int j = 0; j < in.n_targets; j++) {
                const int64_t q = tg[j];
                const uint32_t rec = (uint32_t)(in.rec_base + j);
                const uint32_t coin = (uint32_t)(in.coin_base + (int64_t)coin_per * j);
                bool conflict = cur < 0 || kind_of(cur) != in.kind || stamp[q] == cur;
                if (!conflict) {
                    const DOp& o = hp.ops[cur];
                    if (records && o.a + o.count != rec) conflict = true;
                    if (o.b + (uint32_t)coin_per * o.count != coin) conflict = true;
                }
                if (conflict) {
                    open_op(in.kind, 0);
                    hp.ops[cur].a = records ? rec : 0;
                    hp.ops[cur].b = coin;
                }
                hp.targets.push_back((uint32_t)q);
                if (records) {
                    uint32_t s = NO_SLOT;
                    if (last_use[rec] >= 0) { s = alloc(); slot_of[rec] = s; }
                    hp.targets.push_back(s);
                }
                stamp[q] = cur;
                hp.ops[cur].count++;
            }
            break;
        }
        case K_NOISE: {
            const int ar = in.code == CH_DEP2 ? 2 : 1;
            open_op(K_NOISE, in.code);
            DOp& o = hp.ops[cur];
            o.count = (uint32_t)(in.n_targets / ar);
            o.a = (uint32_t)in.noise_row_base;
            o.b = (uint32_t)in.aux;
            hp.noise_off[in.aux] = o.off;
            hp.noise_ch[in.aux] = (uint32_t)in.code;
            bool dup = false;
            for (int j = 0; j < in.n_targets; j++) {
                if (stamp[tg[j]] == cur) dup = true;
                stamp[tg[j]] = cur;
                hp.targets.push_back((uint32_t)tg[j]);
            }
            if (dup) o.kcf |= F_DUP << 16;
            cur = -1;  // never merge noise ops (one RNG domain per instruction)
            break;
        }
        case K_DET: {
            const int64_t col = in.aux;
            if (cur < 0 || kind_of(cur) != K_DET || hp.ops[cur].a + hp.ops[cur].count != (uint32_t)col) {
                open_op(K_DET, 0);
                hp.ops[cur].a = (uint32_t)col;
            }
            hp.ops[cur].count++;
            for (int64_t e = det_ptr[col]; e < det_ptr[col + 1]; e++) hp.det_terms.push_back(slot_of[det_idx[e]]);
            hp.det_ptr.push_back((uint32_t)hp.det_terms.size());
            for (int64_t e = det_ptr[col]; e < det_ptr[col + 1]; e++) release_after(i, det_idx[e]);
            break;
        }
        case K_OBS: {
            open_op(K_OBS, 0);
            DOp& o = hp.ops[cur];
            o.count = (uint32_t)in.n_targets;
            o.a = (uint32_t)(in.aux - n_det);  // accumulator slot
            for (int j = 0; j < in.n_targets; j++) hp.targets.push_back(slot_of[tg[j]]);
            for (int j = 0; j < in.n_targets; j++) release_after(i, tg[j]);
            cur = -1;
            break;
        }
        }
    }
    // observable columns: one term each, the accumulator slot
    if (n_obs > 0) {
        open_op(K_DET, 0);
        hp.ops[cur].a = (uint32_t)n_det;
        hp.ops[cur].count = (uint32_t)n_obs;
        for (int64_t k = 0; k < n_obs; k++) {
            hp.det_terms.push_back((uint32_t)k);
            hp.det_ptr.push_back((uint32_t)hp.det_terms.size());
        }
    }
    hp.num_slots = next_slot;

    // DET ops whose columns all have the same term count k get direct term
    // addressing: terms of column a+i at det_terms[off + i*k] (off = term base,
    // code = k), one dependent load fewer in the kernel
    for (DOp& o : hp.ops) {
        if ((o.kcf & 0xFF) != K_DET || o.count == 0) continue;
        const uint32_t base = hp.det_ptr[o.a];
        const uint32_t k = hp.det_ptr[o.a + 1] - base;
        bool uniform = k >= 1 && k <= 255;
        for (uint32_t c = o.a; uniform && c < o.a + o.count; c++)
            uniform = hp.det_ptr[c + 1] - hp.det_ptr[c] == k;
        o.off = base;
        if (uniform) o.kcf = (o.kcf & ~0xFF00u) | (k << 8);
    }

    // ---- pass 2b: dead collapse coins ----
    // A coin row sets z_q (FrameBatch.__init__, R, MR: z = coin; M: z ^= coin,
    // frame_sim.py:36-39, 74-90).  If z_q is overwritten by a later R / MR (or
    // the circuit ends) before any gate reads it, that coin can never reach a
    // measurement: the kernels skip its Philox draw.  Gates conservatively count
    // as reads of every operand; noise only XORs into z and DET/OBS touch no
    // frame rows.  Flag = bit 31 of the M/MR/R target word (COIN_DEAD).
    {
        std::vector<std::vector<uint32_t>> pending(num_qubits);  // target-word indices
        std::vector<char> init_pending(num_qubits, 1);
        hp.init_dead.assign(((size_t)num_qubits + 31) / 32, 0u);
        auto kill = [&](uint32_t q) {
            for (uint32_t w : pending[q]) hp.targets[w] |= COIN_DEAD;
            pending[q].clear();
            if (init_pending[q]) { hp.init_dead[q >> 5] |= 1u << (q & 31); init_pending[q] = 0; }
        };
        for (const DOp& o : hp.ops) {
            const uint32_t kind = o.kcf & 0xFF;
            switch (kind) {
            case K_GATE: {
                const int ar = rule_arity((o.kcf >> 8) & 0xFF);
                for (uint32_t j = 0; j < o.count * ar; j++) {
                    const uint32_t q = hp.targets[o.off + j];
                    pending[q].clear();
                    init_pending[q] = 0;
                }
                break;
            }
            case K_M:
                for (uint32_t j = 0; j < o.count; j++) pending[hp.targets[o.off + 2 * j]].push_back(o.off + 2 * j);
                break;
            case K_MR:
                for (uint32_t j = 0; j < o.count; j++) {
                    const uint32_t q = hp.targets[o.off + 2 * j];
                    kill(q);
                    pending[q].push_back(o.off + 2 * j);
                }
                break;
            case K_R:
                for (uint32_t j = 0; j < o.count; j++) {
                    const uint32_t q = hp.targets[o.off + j];
                    kill(q);
                    pending[q].push_back(o.off + j);
                }
                break;
            default: break;
            }
        }
        for (int32_t q = 0; q < num_qubits; q++) kill((uint32_t)q);  // end of circuit
    }

    // ---- pass 3: barrier scheduling over qubit rows + record slots ----
    const int64_t nres = (int64_t)num_qubits + hp.num_slots;
    std::vector<int64_t> rstamp(nres, -1);
    int64_t seg = 0;
    std::vector<int64_t> res;
    for (size_t k = 0; k < hp.ops.size(); k++) {
        DOp& o = hp.ops[k];
        const uint32_t kind = o.kcf & 0xFF;
        res.clear();
        switch (kind) {
        case K_GATE: {
            int ar = rule_arity((o.kcf >> 8) & 0xFF);
            for (uint32_t j = 0; j < o.count * ar; j++) res.push_back(hp.targets[o.off + j]);
            break;
        }
        case K_M: case K_MR:
            for (uint32_t j = 0; j < o.count; j++) {
                res.push_back(hp.targets[o.off + 2 * j] & ~COIN_DEAD);
                uint32_t s = hp.targets[o.off + 2 * j + 1];
                if (s != NO_SLOT) res.push_back(num_qubits + (int64_t)s);
            }
            break;
        case K_R:
            for (uint32_t j = 0; j < o.count; j++) res.push_back(hp.targets[o.off + j] & ~COIN_DEAD);
            break;
        case K_NOISE: {
            int ar = ((o.kcf >> 8) & 0xFF) == CH_DEP2 ? 2 : 1;
            for (uint32_t j = 0; j < o.count * ar; j++) res.push_back(hp.targets[o.off + j]);
            break;
        }
        case K_DET:
            for (uint32_t c = o.a; c < o.a + o.count; c++)
                for (uint32_t e = hp.det_ptr[c]; e < hp.det_ptr[c + 1]; e++)
                    if (hp.det_terms[e] != NO_SLOT) res.push_back(num_qubits + (int64_t)hp.det_terms[e]);
            break;
        case K_OBS:
            res.push_back(num_qubits + (int64_t)o.a);
            for (uint32_t j = 0; j < o.count; j++)
                if (hp.targets[o.off + j] != NO_SLOT) res.push_back(num_qubits + (int64_t)hp.targets[o.off + j]);
            break;
        }
        bool conflict = false;
        for (int64_t r : res) if (rstamp[r] == seg) { conflict = true; break; }
        if (conflict && k > 0) { seg++; o.kcf |= F_BARRIER << 16; }
        for (int64_t r : res) rstamp[r] = seg;
    }
    hp.num_barriers = seg;
    return hp;
}

// Frame-row placement.  Which shared-memory row holds qubit q is free (the
// kernels only ever address rows through the op targets), so rows follow a
// fixed pseudo-random permutation: circuit generators number qubits in
// lattice patterns whose residues mod the bank-group count are badly
// unbalanced (d=25 CX layers: controls mod 4 = {231, 75, 219, 75}), which no
// reordering of one layer can make conflict-free.  row_of[q] = row of qubit q.
void permute_rows(HostProgram& hp) {
    const uint32_t n = (uint32_t)hp.num_qubits;
    hp.row_of.resize(n);
    for (uint32_t q = 0; q < n; q++) hp.row_of[q] = q;
    uint64_t st = 0x9E3779B97F4A7C15ull ^ n;
    for (uint32_t i = n; i > 1; i--) {  // Fisher-Yates with splitmix64
        st += 0x9E3779B97F4A7C15ull;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        std::swap(hp.row_of[i - 1], hp.row_of[z % i]);
    }
    auto map = [&](uint32_t& w) { w = hp.row_of[w & ~COIN_DEAD] | (w & COIN_DEAD); };
    for (const DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF, code = (o.kcf >> 8) & 0xFF;
        uint32_t* t = hp.targets.data() + o.off;
        switch (kind) {
            case K_GATE: for (uint32_t j = 0; j < o.count * rule_arity(code); j++) map(t[j]); break;
            case K_M: case K_MR: for (uint32_t j = 0; j < o.count; j++) map(t[2 * j]); break;
            case K_R: for (uint32_t j = 0; j < o.count; j++) map(t[j]); break;
            case K_NOISE:
                for (uint32_t j = 0; j < o.count * (code == CH_DEP2 ? 2u : 1u); j++) map(t[j]);
                break;
            default: break;
        }
    }
}

// Reorder the applications of every gate op so each aligned group of G
// consecutive applications (the apps one shared-memory wavefront serves: G =
// 128 B / row bytes) touches G distinct bank groups per operand: apps are
// classed by (first, second) operand residue mod G and each group takes one
// app per first residue, choosing among the second residues still unused the
// fullest class.  Apps of one op are independent by construction, so any
// order is the same circuit.
void reorder_for_banks(HostProgram& hp, int W) {
    const int G = W >= 32 ? 1 : 128 / (W * 4);
    if (G <= 1) return;
    std::vector<uint32_t> scratch;
    for (DOp& o : hp.ops) {
        if ((o.kcf & 0xFF) != K_GATE || o.count < 2) continue;
        const int ar = rule_arity((o.kcf >> 8) & 0xFF);
        const uint32_t A = o.count;
        uint32_t* tg = hp.targets.data() + o.off;
        const int G2 = ar == 2 ? G : 1;
        std::vector<std::vector<uint32_t>> cls((size_t)G * G2);
        std::vector<uint32_t> rem0(G, 0);
        for (uint32_t a = 0; a < A; a++) {
            const uint32_t r0 = tg[a * ar] % G, r1 = ar == 2 ? tg[a * ar + 1] % G : 0;
            cls[(size_t)r0 * G2 + r1].push_back(a);
            rem0[r0]++;
        }
        scratch.clear();
        scratch.reserve((size_t)A * ar);
        uint32_t left = A;
        std::vector<char> used1(G2);
        std::vector<int> order(G);
        while (left) {
            std::fill(used1.begin(), used1.end(), 0);
            // fullest first residues first: they are the ones that run out last
            for (int r = 0; r < G; r++) order[r] = r;
            std::sort(order.begin(), order.end(), [&](int x, int y) { return rem0[x] > rem0[y]; });
            for (int r0 : order) {
                if (!rem0[r0] || !left) continue;
                int best = -1;
                for (int r1 = 0; r1 < G2; r1++) {
                    const size_t c = cls[(size_t)r0 * G2 + r1].size();
                    if (!c) continue;
                    if (best < 0 || (!used1[r1] && (used1[best] || c > cls[(size_t)r0 * G2 + best].size()))) best = r1;
                }
                auto& v = cls[(size_t)r0 * G2 + best];
                const uint32_t a = v.back();
                v.pop_back();
                rem0[r0]--;
                used1[best] = 1;
                for (int s2 = 0; s2 < ar; s2++) scratch.push_back(tg[a * ar + s2]);
                left--;
            }
        }
        std::copy(scratch.begin(), scratch.end(), tg);
    }
}

// Operand blocks repeat across the rounds of a REPEAT body (same qubits, and
// with LIFO slot reuse usually the same record slots): point every op at the
// first identical block, so the operand stream a kernel walks (and keeps in
// L1) is one round long.  Blocks stay in place; only offsets move.
void dedup_operands(HostProgram& hp) {
    auto fnv = [](const uint32_t* p, size_t n) {
        uint64_t h = 1469598103934665603ull ^ n;
        for (size_t i = 0; i < n; i++) { h ^= p[i]; h *= 1099511628211ull; }
        return h;
    };
    std::unordered_map<uint64_t, std::vector<uint32_t>> seen_t, seen_d;
    auto canon = [&](std::unordered_map<uint64_t, std::vector<uint32_t>>& seen,
                     const std::vector<uint32_t>& arr, uint32_t off, size_t n) -> uint32_t {
        if (n == 0) return off;
        const uint64_t h = fnv(arr.data() + off, n);
        auto& lst = seen[h];
        for (uint32_t o : lst)
            if (std::equal(arr.begin() + o, arr.begin() + o + n, arr.begin() + off)) return o;
        lst.push_back(off);
        return off;
    };
    for (DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF, code = (o.kcf >> 8) & 0xFF;
        switch (kind) {
            case K_GATE: o.off = canon(seen_t, hp.targets, o.off, (size_t)o.count * rule_arity(code)); break;
            case K_M: case K_MR: o.off = canon(seen_t, hp.targets, o.off, 2 * (size_t)o.count); break;
            case K_R: case K_OBS: o.off = canon(seen_t, hp.targets, o.off, o.count); break;
            case K_NOISE:
                o.off = canon(seen_t, hp.targets, o.off, (size_t)o.count * (code == CH_DEP2 ? 2 : 1));
                hp.noise_off[o.b] = o.off;
                break;
            case K_DET:
                if (code) o.off = canon(seen_d, hp.det_terms, o.off, (size_t)o.count * code);
                break;
            default: break;
        }
    }
}

// Binomial(n, p) inverse-CDF thresholds in 64-bit fixed point:
// X = min{m : u < t[m]} for u uniform on [0, 2^64), X = len(t) if u >= every
// entry.  Upper-tail thresholds are built from the tail sum so their absolute
// error stays ~2^-64.
static std::vector<uint64_t> binomial_thresholds(uint64_t n, double p) {
    std::vector<double> pmf;
    const double q = 1.0 - p;
    double pm = std::exp((double)n * std::log1p(-p));
    const double mean = (double)n * p;
    for (uint64_t m = 0;; m++) {
        pmf.push_back(pm);
        if (m == n) break;
        if ((double)m > mean && pm < 1e-40) break;
        pm = pm * ((double)(n - m) / (double)(m + 1)) * (p / q);
    }
    const size_t M = pmf.size();
    std::vector<double> sf(M, 0.0);  // P(X > m)
    for (size_t m = M - 1; m-- > 0;) sf[m] = sf[m + 1] + pmf[m + 1];
    std::vector<uint64_t> t;
    double cdf = 0.0;
    for (size_t m = 0; m < M; m++) {
        cdf += pmf[m];
        const double tail = std::ldexp(sf[m], 64);
        if (tail < 1.0) break;  // every remaining u lands on X = m
        uint64_t v;
        if (cdf <= 0.5) v = (uint64_t)std::floor(std::ldexp(cdf, 64));
        else v = (uint64_t)0 - (uint64_t)std::ceil(tail);
        t.push_back(v);
    }
    return t;
}

void build_noise_schedule(HostProgram& hp, int tile_shots, double target_hits) {
    hp.noise_tab.clear();
    hp.pregen_ops.clear();
    hp.pregen_chunks = 0;
    hp.hit_capacity = 0;
    for (int64_t j = 0; j < hp.num_noise; j++) {
        NoiseParam& np = hp.noise[j];
        const uint32_t npat = np.npat ? np.npat : 1u;
        np = NoiseParam{};
        np.npat = npat;
        const uint64_t N = (uint64_t)hp.noise_apps[j] * (uint64_t)tile_shots;
        const double p = hp.noise_p[j];
        if (N == 0 || p <= 0.0) { np.flags = NZ_NONE; continue; }
        if (N >= (1ull << 31)) bad("noise instruction too large for one tile");
        uint64_t L;
        if (p >= 1.0) {
            np.flags = NZ_ALL;
            L = 1;
            while (L < N && L < 1024) L *= 2;  // power of two; positions stay below 2^28
        } else {
            // power of two nearest (in ratio) to target_hits / p trials
            double want = target_hits / p;
            L = 1;
            while ((double)(L * 2) <= want * 1.41421356 && L < (1ull << 27)) L *= 2;
            while (L > 1 && L / 2 >= N) L /= 2;  // no chunk longer than needed
        }
        np.L = (uint32_t)L;
        np.nchunks = (uint32_t)((N + L - 1) / L);
        np.last_len = (uint32_t)(N - (uint64_t)(np.nchunks - 1) * L);  // real trials in the last chunk
        if (!(np.flags & NZ_ALL)) {
            // every chunk draws from Binomial(L, p): trials past N are virtual and dropped
            auto tf = binomial_thresholds(L, p);
            np.tab_full = (uint32_t)hp.noise_tab.size();
            np.len_full = (uint32_t)tf.size();
            np.tab_last = np.tab_full;
            np.len_last = np.len_full;
            hp.noise_tab.insert(hp.noise_tab.end(), tf.begin(), tf.end());
        }
        const double E = (double)N * p;
        if (p < 0.25 && E <= 16384.0 && N < (1ull << 28)) {
            np.flags |= NZ_PREGEN;
            // overflow (Poisson tail beyond ~6 sigma + 10, < 1e-9 per list) falls
            // back to inline sampling, so the slack only trades memory for speed
            np.cap = (uint32_t)std::ceil(E + 6.0 * std::sqrt(E) + 10.0);
            np.cap_base = (uint32_t)hp.hit_capacity;
            hp.hit_capacity += np.cap;
            // pre-pass work items are 32-chunk blocks (one warp each)
            np.chunk_base = (uint32_t)hp.pregen_chunks;
            hp.pregen_chunks += (np.nchunks + 31) / 32;
            hp.pregen_ops.push_back((uint32_t)j);
        }
    }
    // noise ops learn their hit-list base and the next pre-generated op, so
    // consumer threads can prefetch the next op's hits while other ops run
    std::vector<uint32_t> next_of(hp.num_noise, NO_SLOT);
    for (size_t k = 0; k + 1 < hp.pregen_ops.size(); k++) next_of[hp.pregen_ops[k]] = hp.pregen_ops[k + 1];
    hp.first_pregen = hp.pregen_ops.empty() ? NO_SLOT : hp.pregen_ops[0];
    hp.first_cap_base = hp.pregen_ops.empty() ? 0 : hp.noise[hp.pregen_ops[0]].cap_base;
    for (DOp& o : hp.ops) {
        if ((o.kcf & 0xFF) != K_NOISE) continue;
        const NoiseParam& np = hp.noise[o.b];
        o.kcf &= ~(F_PREGEN << 16);
        if (np.flags & NZ_PREGEN) o.kcf |= F_PREGEN << 16;
        o.c = np.cap_base;
        o.d = next_of[o.b];
        o.e = o.d != NO_SLOT ? hp.noise[o.d].cap_base : 0u;
    }
}

// Column-kernel op stream: one self-describing block per device op (header,
// the NoiseParam of a noise op, then the op's operands), 16-byte aligned so the
// producer warp can bulk-copy a block into a shared-memory slot in one
// transaction.  Operands larger than slot_cap stay in global memory
// (F_GLOBALP); only their header is staged.
ColStream build_col_stream(const HostProgram& hp, uint32_t slot_cap) {
    ColStream cs;
    std::vector<uint32_t> pay;
    for (const DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF, code = (o.kcf >> 8) & 0xFF;
        pay.clear();
        auto take = [&](const std::vector<uint32_t>& arr, size_t off, size_t n) {
            pay.insert(pay.end(), arr.begin() + off, arr.begin() + off + n);
        };
        switch (kind) {
            case K_GATE: take(hp.targets, o.off, (size_t)o.count * rule_arity(code)); break;
            case K_M: case K_MR: take(hp.targets, o.off, 2 * (size_t)o.count); break;
            case K_R: case K_OBS: take(hp.targets, o.off, o.count); break;
            case K_NOISE: take(hp.targets, o.off, (size_t)o.count * (code == CH_DEP2 ? 2 : 1)); break;
            case K_DET:
                if (code) {
                    take(hp.det_terms, o.off, (size_t)o.count * code);
                } else {
                    const uint32_t base = hp.det_ptr[o.a];
                    for (uint32_t c = 0; c <= o.count; c++) pay.push_back(hp.det_ptr[o.a + c] - base);
                    take(hp.det_terms, base, hp.det_ptr[o.a + o.count] - base);
                }
                break;
            default: break;
        }
        while (cs.words.size() & 3) cs.words.push_back(0u);
        const size_t start = cs.words.size();
        const uint32_t hw = COL_HEAD_WORDS + (kind == K_NOISE ? COL_NP_WORDS : 0u);
        const bool globalp = ((size_t)hw + pay.size()) * 4 > slot_cap;
        CHead h{};
        h.kcf = o.kcf | (globalp ? (F_GLOBALP << 16) : 0u);
        h.count = o.count;
        h.a = o.a;
        h.b = o.b;
        h.pwords = (uint32_t)pay.size();
        h.goff = (uint32_t)(start + hw);
        const uint32_t* hp32 = reinterpret_cast<const uint32_t*>(&h);
        cs.words.insert(cs.words.end(), hp32, hp32 + COL_HEAD_WORDS);
        if (kind == K_NOISE) {
            const uint32_t* np32 = reinterpret_cast<const uint32_t*>(&hp.noise[o.b]);
            cs.words.insert(cs.words.end(), np32, np32 + COL_NP_WORDS);
        }
        cs.words.insert(cs.words.end(), pay.begin(), pay.end());
        const uint32_t staged = (uint32_t)((((globalp ? hw : hw + pay.size()) * 4) + 15) & ~(size_t)15);
        if (start / 4 > 0xFFFFFFFFull) bad("op stream too large");
        cs.binfo.push_back((uint32_t)(start / 4));
        cs.binfo.push_back(staged);
        cs.slot_bytes = std::max(cs.slot_bytes, staged);
    }
    while (cs.words.size() & 3) cs.words.push_back(0u);
    cs.n_blocks = (int64_t)hp.ops.size();
    return cs;
}

}  // namespace pfs
