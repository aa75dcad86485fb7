// Host-side circuit compiler: flat frame program -> device op list.
//
// Replaces the per-call `compile_frame_program` (stabsim/frame_sim.py:170-189)
// with a one-time native pass that prepares the op stream the persistent CUDA
// kernel interprets:
//   * split every instruction at the first repeated qubit, so each device op is
//     a set of independent applications (the reference applies an
//     instruction's applications sequentially, frame_sim.py:61-62, 196-197 —
//     `CX 0 1 1 2` must stay two steps);
//   * fuse a noise instruction into its neighbour when both act on the same
//     target list: gate / reset then noise (DEPOLARIZE2 after CX, DEPOLARIZE1
//     after H or R), noise then measurement (X_ERROR before M) — one kernel
//     item applies both to its rows in registers, no barrier between them;
//   * merge consecutive instructions of the same frame rule / collapse kind
//     when they touch disjoint qubits (fewer ops, fewer barriers);
//   * detection-event programs keep a measurement record in the measured
//     qubit's x row (frame_sim.py:74-80: the record IS x at M) until an op
//     rewrites that row, and only then spill it to a ring slot (fused into the
//     reset that rewrites it); slots live until the last DETECTOR /
//     OBSERVABLE_INCLUDE reading them (stabsim/circuit.py:247-256);
//   * coin relevance: a collapse coin (z row of FrameBatch.__init__, M, R, MR,
//     frame_sim.py:36-39, 74-90) whose effect reaches no output is never
//     drawn (decided by a backward pass over random 128-bit projections of the
//     output columns);
//   * schedule group barriers: one goes before an op only if it touches a
//     qubit row or ring slot already touched since the previous barrier
//     (standalone noise ops commute with each other: their XORs are atomic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>

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

// does the frame rule (stabsim/gates.py:70-92) write the x row of slot s?
bool rule_writes_x(int32_t rule, int s) {
    switch (rule) {
        case R_SWAPXZ: case R_XXORZ: case R_SWAP: return true;
        case R_CX: case R_CY: return s == 1;
        default: return false;  // R_ZXORX, R_CZ write z only
    }
}

int channel_arity(int32_t ch) { return ch == CH_DEP2 ? 2 : 1; }
// noise XORs x rows (injected masks may carry x bits for any channel)
bool channel_writes_x(int32_t) { return true; }

[[noreturn]] void bad(const std::string& msg) { throw std::invalid_argument(msg); }

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// 128-bit random projection of a set of output columns (GF(2) linear)
struct H128 {
    uint64_t a = 0, b = 0;
    void x(const H128& o) { a ^= o.a; b ^= o.b; }
    bool zero() const { return (a | b) == 0; }
};

}  // namespace

HostProgram compile_program(const pfs_instr* ins, int64_t n_ins, const int32_t* targets,
                            int64_t n_targets, const double* noise_p, int64_t n_noise,
                            const int64_t* det_ptr, const int64_t* det_idx, int64_t n_cols,
                            int64_t n_obs, int32_t num_qubits, int64_t num_meas,
                            int64_t num_coin_rows, int64_t num_noise_rows, int mode) {
    if (num_qubits < 0 || num_meas < 0 || n_cols < 0 || n_obs < 0 || n_obs > n_cols)
        bad("negative sizes");
    if (n_ins > 0 && (!ins || (n_targets > 0 && !targets))) bad("null instruction arrays");
    if (n_cols > 0 && (!det_ptr)) bad("null detector arrays");
    if (num_qubits >= (1 << 30)) bad("too many qubits");
    const bool events = mode == PM_EVENTS;
    const int64_t n_det = n_cols - n_obs;
    HostProgram hp;
    hp.mode = mode;
    hp.num_qubits = num_qubits;
    hp.num_meas = num_meas;
    hp.num_cols = n_cols;
    hp.num_obs = n_obs;
    hp.num_noise = n_noise;
    hp.num_coin_rows = num_coin_rows;
    hp.num_noise_rows = num_noise_rows;
    hp.noise_p.assign(noise_p, noise_p + n_noise);
    hp.noise_apps.assign(n_noise, 0);
    hp.noise_ch.assign(n_noise, 0);
    hp.noise_fused.assign(n_noise, 0);
    hp.noise_rowb.assign(n_noise, 0);
    if (num_noise_rows >= (1ll << 32)) bad("too many noise rows");
    for (int64_t i = 0; i < n_noise; i++) {
        double p = noise_p[i];
        if (!(p >= 0.0 && p <= 1.0)) bad("noise probability must be in [0, 1], got " + std::to_string(p));
    }

    // ---- pass 1: validate, record liveness, distinct-target instructions ----
    std::vector<int64_t> last_use(num_meas, -1);
    std::vector<char> distinct(n_ins, 1);
    std::vector<int64_t> qstamp(num_qubits, -1);
    {
        int64_t rec = 0, coin = num_qubits, nrow = 0, col = 0;
        for (int64_t i = 0; i < n_ins; i++) {
            const pfs_instr& in = ins[i];
            if (in.n_targets < 0 || in.tgt_off < 0 || (int64_t)in.tgt_off + in.n_targets > n_targets)
                bad("instruction " + std::to_string(i) + ": target range out of bounds");
            const int32_t* tg = targets + in.tgt_off;
            auto check_qubits = [&]() {
                for (int j = 0; j < in.n_targets; j++) {
                    if (tg[j] < 0 || tg[j] >= num_qubits)
                        bad("qubit " + std::to_string(tg[j]) + " out of range [0, " + std::to_string(num_qubits) + ")");
                    if (qstamp[tg[j]] == i) distinct[i] = 0;
                    qstamp[tg[j]] = i;
                }
            };
            switch (in.kind) {
            case K_GATE:
                if (in.code <= R_NONE || in.code > R_SWAP) bad("unknown frame rule");
                if (in.n_targets % rule_arity(in.code)) bad("gate target count not a multiple of arity");
                check_qubits();
                for (int j = 0; j + 1 < in.n_targets && rule_arity(in.code) == 2; j += 2)
                    if (tg[j] == tg[j + 1]) bad("two-qubit gate targets a qubit pair twice");
                hp.bframe_bits += rule_bits(in.code) * (in.n_targets / rule_arity(in.code));
                break;
            case K_M: case K_R: case K_MR:
                check_qubits();
                if (in.kind != K_R && in.rec_base != rec) bad("record numbering is not contiguous");
                if (in.coin_base != coin) bad("coin row numbering is not contiguous");
                if (in.kind != K_R) rec += in.n_targets;
                coin += (int64_t)in.n_targets * (in.kind == K_MR ? 2 : 1);
                hp.bframe_bits += (in.kind == K_R ? 2 : 4) * (int64_t)in.n_targets;
                break;
            case K_NOISE: {
                if (in.code < CH_XERR || in.code > CH_DEP2) bad("unknown noise channel");
                const int ar = channel_arity(in.code);
                if (in.n_targets % ar) bad("noise target count not a multiple of arity");
                check_qubits();
                if (in.aux < 0 || in.aux >= n_noise) bad("noise ordinal out of range");
                if (in.noise_row_base != nrow) bad("noise row numbering is not contiguous");
                hp.noise_apps[in.aux] = (uint32_t)(in.n_targets / ar);
                hp.noise_ch[in.aux] = (uint32_t)in.code;
                hp.noise_rowb[in.aux] = (uint32_t)in.noise_row_base;
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

    // ---- pass 1b: noise fusion plan ----
    // fuse_post[i]: noise instruction i+1 is applied inside gate / reset i;
    // fuse_pre[i]: noise instruction i is applied inside measurement i+1.
    std::vector<char> fuse_post(n_ins, 0), fuse_pre(n_ins, 0), fused_noise(n_ins, 0);
    auto same_targets = [&](const pfs_instr& a, const pfs_instr& b) {
        return a.n_targets == b.n_targets &&
               std::equal(targets + a.tgt_off, targets + a.tgt_off + a.n_targets, targets + b.tgt_off);
    };
    for (int64_t i = 0; i + 1 < n_ins; i++) {
        const pfs_instr& a = ins[i];
        const pfs_instr& b = ins[i + 1];
        if (!distinct[i] || a.n_targets == 0 || fused_noise[i]) continue;
        if ((a.kind == K_GATE || a.kind == K_R) && b.kind == K_NOISE &&
            (a.kind == K_R ? 1 : rule_arity(a.code)) == channel_arity(b.code) && same_targets(a, b)) {
            fuse_post[i] = 1;
            fused_noise[i + 1] = 1;
        } else if (a.kind == K_NOISE && (b.kind == K_M || b.kind == K_MR) && channel_arity(a.code) == 1 &&
                   same_targets(a, b)) {
            fuse_pre[i] = 1;
            fused_noise[i] = 1;
        }
    }

    // ---- pass 1c: coin relevance ----
    // Backward over the program with a random 128-bit projection h(S) of the
    // output-column set S each frame component would flip (the transposed
    // frame rules; gates.py:70-92): a coin is relevant iff the projection of
    // its z component at the collapse is non-zero (a relevant coin is missed
    // with probability 2^-128).  Outputs: detector / observable columns for
    // event programs, every measurement record for record programs.
    std::vector<char> coin_live(num_coin_rows, 1);
    {
        std::vector<H128> rech(num_meas);
        auto rnd = [](uint64_t salt, uint64_t k) {
            H128 h;
            h.a = splitmix64(k * 2 + 0x51A7 + salt);
            h.b = splitmix64(k * 2 + 1 + 0xC0FFEE00ull + salt);
            return h;
        };
        if (events) {
            for (int64_t c = 0; c < n_cols; c++) {
                const H128 h = rnd(1, (uint64_t)c);
                for (int64_t e = det_ptr[c]; e < det_ptr[c + 1]; e++) rech[det_idx[e]].x(h);
            }
        } else {
            for (int64_t m = 0; m < num_meas; m++) rech[m] = rnd(2, (uint64_t)m);
        }
        std::vector<H128> sx(num_qubits), sz(num_qubits);
        for (int64_t i = n_ins - 1; i >= 0; i--) {
            const pfs_instr& in = ins[i];
            const int32_t* tg = targets + in.tgt_off;
            switch (in.kind) {
            case K_GATE: {
                const int ar = rule_arity(in.code);
                for (int j = in.n_targets - ar; j >= 0; j -= ar) {
                    const int32_t a = tg[j], b = ar == 2 ? tg[j + 1] : -1;
                    switch (in.code) {
                        case R_SWAPXZ: std::swap(sx[a], sz[a]); break;
                        case R_ZXORX: sx[a].x(sz[a]); break;
                        case R_XXORZ: sz[a].x(sx[a]); break;
                        case R_CX: sx[a].x(sx[b]); sz[b].x(sz[a]); break;
                        case R_CZ: sx[a].x(sz[b]); sx[b].x(sz[a]); break;
                        case R_CY: {
                            H128 x0 = sx[a];
                            x0.x(sx[b]);
                            x0.x(sz[b]);
                            sx[b].x(sz[a]);
                            sz[b].x(sz[a]);
                            sx[a] = x0;
                            break;
                        }
                        default: std::swap(sx[a], sx[b]); std::swap(sz[a], sz[b]); break;
                    }
                }
                break;
            }
            case K_M:
                for (int j = in.n_targets - 1; j >= 0; j--) {
                    const int32_t q = tg[j];
                    coin_live[in.coin_base + j] = !sz[q].zero();
                    sx[q].x(rech[in.rec_base + j]);
                }
                break;
            case K_MR:
                for (int j = in.n_targets - 1; j >= 0; j--) {
                    const int32_t q = tg[j];
                    coin_live[in.coin_base + 2 * j + 1] = !sz[q].zero();
                    coin_live[in.coin_base + 2 * j] = 0;  // overwritten by the reset's coin
                    sx[q] = H128{};
                    sz[q] = H128{};
                    sx[q].x(rech[in.rec_base + j]);
                }
                break;
            case K_R:
                for (int j = in.n_targets - 1; j >= 0; j--) {
                    const int32_t q = tg[j];
                    coin_live[in.coin_base + j] = !sz[q].zero();
                    sx[q] = H128{};
                    sz[q] = H128{};
                }
                break;
            default: break;
            }
        }
        for (int32_t q = 0; q < num_qubits; q++) coin_live[q] = !sz[q].zero();
        hp.init_dead.assign(((size_t)num_qubits + 31) / 32, 0u);
        for (int32_t q = 0; q < num_qubits; q++)
            if (!coin_live[q]) hp.init_dead[q >> 5] |= 1u << (q & 31);
        for (char c : coin_live) hp.live_coin_rows += c ? 1 : 0;
    }

    // ---- pass 2: emit device ops ----
    std::vector<uint32_t> slot_of(num_meas, NO_SLOT);
    std::vector<int32_t> home_of(num_meas, -1);            // record homed in this qubit's x row
    std::vector<std::vector<uint32_t>> xrec(num_qubits);    // live records homed in x_q
    std::vector<uint32_t> free_slots;
    uint32_t next_slot = (uint32_t)(events ? n_obs : 0);   // [0, n_obs) = observable accumulators
    std::vector<int64_t> stamp(num_qubits, -1);
    int64_t cur = -1;  // open (mergeable) op index
    auto open_op = [&](uint32_t kind, uint32_t code) {
        // ops read their targets as uint2 pairs (two-qubit rules, (row, slot)
        // pairs): keep every op's target list 8-byte aligned
        if (hp.targets.size() & 1) hp.targets.push_back(0u);
        DOp op{};
        op.kcf = kind | (code << 8);
        op.off = (uint32_t)hp.targets.size();
        op.c = NO_SLOT;
        hp.ops.push_back(op);
        cur = (int64_t)hp.ops.size() - 1;
    };
    auto kind_of = [&](int64_t k) { return hp.ops[k].kcf & 0xFF; };
    auto code_of = [&](int64_t k) { return (hp.ops[k].kcf >> 8) & 0xFF; };
    auto mergeable = [&](int64_t k) { return !((hp.ops[k].kcf >> 16) & F_NOISE); };
    auto alloc = [&]() -> uint32_t {
        if (!free_slots.empty()) { uint32_t s = free_slots.back(); free_slots.pop_back(); return s; }
        return next_slot++;
    };
    // records homed in x_q that are still needed at or after instruction i move
    // to slots: one through `first` (fused into a reset), the rest via a SPILL op
    std::vector<std::pair<uint32_t, uint32_t>> spills;  // (qubit, slot) pairs of the pending SPILL op
    auto take_homes = [&](int32_t q, int64_t i, uint32_t* first) {
        std::vector<uint32_t>& v = xrec[q];
        for (uint32_t m : v) {
            if (last_use[m] < i || home_of[m] != q) continue;
            const uint32_t s = alloc();
            slot_of[m] = s;
            home_of[m] = -1;
            if (first && *first == NO_SLOT) *first = s;
            else spills.emplace_back((uint32_t)q, s);
        }
        v.clear();
    };
    auto flush_spills = [&]() {
        if (spills.empty()) return;
        open_op(K_SPILL, 0);
        for (auto& ps : spills) { hp.targets.push_back(ps.first); hp.targets.push_back(ps.second); }
        hp.ops[cur].count = (uint32_t)spills.size();
        spills.clear();
        cur = -1;
    };
    auto release = [&](int64_t i, int64_t m) {
        if (last_use[m] != i) return;
        if (slot_of[m] != NO_SLOT) { free_slots.push_back(slot_of[m]); slot_of[m] = NO_SLOT; }
        if (home_of[m] >= 0) {
            std::vector<uint32_t>& v = xrec[home_of[m]];
            v.erase(std::remove(v.begin(), v.end(), (uint32_t)m), v.end());
            home_of[m] = -1;
        }
    };
    auto term_of = [&](int64_t m) -> uint32_t {
        if (slot_of[m] != NO_SLOT) return slot_of[m];
        if (home_of[m] >= 0) return XROW | (uint32_t)home_of[m];
        bad("internal: record " + std::to_string(m) + " has no location");
    };
    hp.det_ptr.assign(1, 0);

    for (int64_t i = 0; i < n_ins; i++) {
        const pfs_instr& in = ins[i];
        const int32_t* tg = targets + in.tgt_off;
        switch (in.kind) {
        case K_GATE: {
            const int ar = rule_arity(in.code);
            const bool fz = fuse_post[i] != 0;
            const pfs_instr* nz = fz ? &ins[i + 1] : nullptr;
            if (events) {  // records homed in rows this op rewrites move to slots first
                for (int j = 0; j < in.n_targets; j++)
                    if (rule_writes_x(in.code, j % ar) || (nz && channel_writes_x(nz->code)))
                        if (!xrec[tg[j]].empty()) take_homes(tg[j], i, nullptr);
                flush_spills();
            }
            if (fz) {
                open_op(K_GATE, in.code);
                DOp& o = hp.ops[cur];
                o.kcf |= F_NOISE << 16;
                o.count = (uint32_t)(in.n_targets / ar);
                o.c = (uint32_t)nz->aux;
                hp.noise_fused[nz->aux] = 1;
                for (int j = 0; j < in.n_targets; j++) hp.targets.push_back((uint32_t)tg[j]);
                cur = -1;
                break;
            }
            for (int j = 0; j < in.n_targets; j += ar) {
                bool conflict = cur < 0 || kind_of(cur) != K_GATE || code_of(cur) != (uint32_t)in.code ||
                                !mergeable(cur);
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
            // pre-noise: noise instruction i-1 applied inside this op
            const pfs_instr* pre = (i > 0 && fuse_pre[i - 1]) ? &ins[i - 1] : nullptr;
            const pfs_instr* nz = (in.kind == K_R && fuse_post[i]) ? &ins[i + 1] : pre;
            std::vector<uint32_t> rspill;  // R: slot each target's homed record moves to
            if (events) {
                for (int j = 0; j < in.n_targets; j++) {
                    const int32_t q = tg[j];
                    if (xrec[q].empty()) continue;
                    if (in.kind == K_M && !(pre && channel_writes_x(pre->code))) continue;  // M keeps x
                    if (in.kind == K_R) {
                        if (rspill.empty()) rspill.assign(in.n_targets, NO_SLOT);
                        take_homes(q, i, &rspill[j]);
                    } else {
                        take_homes(q, i, nullptr);
                    }
                }
                flush_spills();
            }
            const bool fused = nz != nullptr;
            for (int j = 0; j < in.n_targets; j++) {
                const int64_t q = tg[j];
                const uint32_t rec = (uint32_t)(in.rec_base + j);
                const uint32_t coin = (uint32_t)(in.coin_base + (int64_t)coin_per * j);
                bool conflict = cur < 0 || kind_of(cur) != in.kind || stamp[q] == cur || !mergeable(cur);
                if (!conflict) {
                    const DOp& o = hp.ops[cur];
                    if (records && o.a + o.count != rec) conflict = true;
                    if (o.b + (uint32_t)coin_per * o.count != coin) conflict = true;
                }
                if (fused) conflict = j == 0;  // one op holds the whole fused instruction
                if (conflict) {
                    open_op(in.kind, 0);
                    hp.ops[cur].a = records ? rec : 0;
                    hp.ops[cur].b = coin;
                    if (fused) {
                        hp.ops[cur].kcf |= F_NOISE << 16;
                        hp.ops[cur].c = (uint32_t)nz->aux;
                        hp.noise_fused[nz->aux] = 1;
                    }
                }
                const bool live = coin_live[coin + (in.kind == K_MR ? 1 : 0)] != 0;
                hp.targets.push_back((uint32_t)q | (live ? 0u : COIN_DEAD));
                uint32_t s = NO_SLOT;
                if (in.kind == K_R) {
                    s = rspill.empty() ? NO_SLOT : rspill[j];
                } else if (events && last_use[rec] >= 0) {
                    if (in.kind == K_MR) { s = alloc(); slot_of[rec] = s; }  // the reset rewrites x
                    else { home_of[rec] = (int32_t)q; xrec[q].push_back(rec); }
                }
                hp.targets.push_back(s);
                stamp[q] = cur;
                hp.ops[cur].count++;
            }
            if (fused) cur = -1;
            break;
        }
        case K_NOISE: {
            if (fused_noise[i]) break;  // emitted inside its gate / collapse op
            const int ar = channel_arity(in.code);
            if (events && channel_writes_x(in.code)) {
                for (int j = 0; j < in.n_targets; j++)
                    if (!xrec[tg[j]].empty()) take_homes(tg[j], i, nullptr);
                flush_spills();
            }
            open_op(K_NOISE, in.code);
            DOp& o = hp.ops[cur];
            o.count = (uint32_t)(in.n_targets / ar);
            o.c = (uint32_t)in.aux;
            if (!distinct[i]) o.kcf |= F_DUP << 16;
            for (int j = 0; j < in.n_targets; j++) hp.targets.push_back((uint32_t)tg[j]);
            cur = -1;  // never merge noise ops (one RNG domain per instruction)
            break;
        }
        case K_DET: {
            if (!events) break;
            const int64_t col = in.aux;
            if (cur < 0 || kind_of(cur) != K_DET || hp.ops[cur].a + hp.ops[cur].count != (uint32_t)col) {
                open_op(K_DET, 0);
                hp.ops[cur].a = (uint32_t)col;
            }
            hp.ops[cur].count++;
            for (int64_t e = det_ptr[col]; e < det_ptr[col + 1]; e++) hp.det_terms.push_back(term_of(det_idx[e]));
            hp.det_ptr.push_back((uint32_t)hp.det_terms.size());
            for (int64_t e = det_ptr[col]; e < det_ptr[col + 1]; e++) release(i, det_idx[e]);
            break;
        }
        case K_OBS: {
            if (!events) break;
            open_op(K_OBS, 0);
            DOp& o = hp.ops[cur];
            o.count = (uint32_t)in.n_targets;
            o.a = (uint32_t)(in.aux - n_det);  // accumulator slot
            for (int j = 0; j < in.n_targets; j++) hp.targets.push_back(term_of(tg[j]));
            for (int j = 0; j < in.n_targets; j++) release(i, tg[j]);
            cur = -1;
            break;
        }
        }
    }
    // observable columns: one term each, the accumulator slot
    if (events && n_obs > 0) {
        open_op(K_DET, 0);
        hp.ops[cur].a = (uint32_t)n_det;
        hp.ops[cur].count = (uint32_t)n_obs;
        for (int64_t k = 0; k < n_obs; k++) {
            hp.det_terms.push_back((uint32_t)k);
            hp.det_ptr.push_back((uint32_t)hp.det_terms.size());
        }
    }
    hp.num_slots = next_slot;

    // event programs: a measurement that keeps its records in x rows, draws no
    // coin and carries no noise does nothing — drop it
    if (events) {
        std::vector<DOp> kept;
        kept.reserve(hp.ops.size());
        for (const DOp& o : hp.ops) {
            bool noop = (o.kcf & 0xFF) == K_M && !((o.kcf >> 16) & F_NOISE);
            for (uint32_t j = 0; noop && j < o.count; j++)
                noop = (hp.targets[o.off + 2 * j] & COIN_DEAD) && hp.targets[o.off + 2 * j + 1] == NO_SLOT;
            if (!noop) kept.push_back(o);
        }
        hp.ops.swap(kept);
    }

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

    // ---- pass 3: barrier scheduling over qubit rows + ring slots ----
    const int64_t nres = (int64_t)num_qubits + hp.num_slots;
    std::vector<int64_t> rstamp(nres, -1);
    std::vector<char> rnoise(nres, 0);  // touched only by standalone noise ops in this segment
    int64_t seg = 0;
    std::vector<int64_t> res;
    for (size_t k = 0; k < hp.ops.size(); k++) {
        DOp& o = hp.ops[k];
        const uint32_t kind = o.kcf & 0xFF;
        res.clear();
        auto row = [&](uint32_t w) { res.push_back((int64_t)(w & ~COIN_DEAD)); };
        auto slot = [&](uint32_t s) { if (s != NO_SLOT) res.push_back(num_qubits + (int64_t)s); };
        auto term = [&](uint32_t t) {
            if (t == NO_SLOT) return;
            if (t & XROW) res.push_back((int64_t)(t & ~XROW));
            else res.push_back(num_qubits + (int64_t)t);
        };
        switch (kind) {
        case K_GATE: {
            const int ar = rule_arity((o.kcf >> 8) & 0xFF);
            for (uint32_t j = 0; j < o.count * ar; j++) row(hp.targets[o.off + j]);
            break;
        }
        case K_M: case K_MR: case K_R: case K_SPILL:
            for (uint32_t j = 0; j < o.count; j++) {
                row(hp.targets[o.off + 2 * j]);
                slot(hp.targets[o.off + 2 * j + 1]);
            }
            break;
        case K_NOISE: {
            const int ar = channel_arity((o.kcf >> 8) & 0xFF);
            for (uint32_t j = 0; j < o.count * ar; j++) row(hp.targets[o.off + j]);
            break;
        }
        case K_DET:
            for (uint32_t c = o.a; c < o.a + o.count; c++)
                for (uint32_t e = hp.det_ptr[c]; e < hp.det_ptr[c + 1]; e++) term(hp.det_terms[e]);
            break;
        case K_OBS:
            slot(o.a);
            for (uint32_t j = 0; j < o.count; j++) term(hp.targets[o.off + j]);
            break;
        }
        const bool nz = kind == K_NOISE;
        bool conflict = false;
        for (int64_t r : res)
            if (rstamp[r] == seg && !(nz && rnoise[r])) { conflict = true; break; }
        if (conflict && k > 0) { seg++; o.kcf |= F_BARRIER << 16; }
        for (int64_t r : res) {
            if (rstamp[r] != seg) rnoise[r] = nz ? 1 : 0;
            else rnoise[r] = rnoise[r] && nz;
            rstamp[r] = seg;
        }
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
static uint32_t warp_share(uint32_t apps, uint32_t nw, uint32_t ca);

// Local search over the bank classes of the qubits.  Cost = for every gate op,
// every warp's share of its applications (the range one warp walks,
// lower_stream) and each operand: the applications in excess of an even split
// over the G classes — with none, the warp's passes can be ordered so that every
// shared-memory wavefront serves G distinct bank groups (bank_reorder).  Moves
// swap the classes of two qubits (class sizes stay what the row pools can hold);
// a move is kept when it does not raise the cost.  Ops with identical target
// lists (the rounds of a REPEAT body) are counted once, weighted.  Measured with
// tools/bank_model.py at d=25 (4 classes): CX row wavefronts 1.45x -> 1.08x the
// conflict-free count.  With 32 classes (one-word tiles, d=100) an even split
// is not enough for the greedy grouping (2.05x vs 1.85x for the first-appearance
// classes, whose order is already regular), so the search runs for G <= 8 only;
// a cost on aligned groups in instruction order converged worse in both cases.
static void refine_classes(const HostProgram& hp, std::vector<int32_t>& cls, uint32_t G, uint32_t nw) {
    struct Occ { uint32_t cell; uint32_t w; };
    const uint32_t n = (uint32_t)hp.num_qubits;
    std::unordered_map<uint64_t, uint32_t> uniq;   // target-list hash -> unique op
    std::vector<uint32_t> weight, first_op;
    for (size_t i = 0; i < hp.ops.size(); i++) {
        const DOp& o = hp.ops[i];
        if ((o.kcf & 0xFF) != K_GATE || o.count == 0) continue;
        const int ar = rule_arity((o.kcf >> 8) & 0xFF);
        uint64_t h = 1469598103934665603ull ^ ((uint64_t)o.count * 2 + ar);
        for (uint32_t j = 0; j < o.count * ar; j++) { h ^= hp.targets[o.off + j]; h *= 1099511628211ull; }
        auto it = uniq.find(h);
        if (it == uniq.end()) { uniq.emplace(h, (uint32_t)weight.size()); weight.push_back(1); first_op.push_back((uint32_t)i); }
        else weight[it->second]++;
    }
    const size_t U = weight.size();
    if (U == 0) return;
    std::vector<std::vector<Occ>> occ(n);
    std::vector<int32_t> cnt(U * nw * 2 * G, 0), cap(U * nw * 2, 0);
    for (size_t u = 0; u < U; u++) {
        const DOp& o = hp.ops[first_op[u]];
        const int ar = rule_arity((o.kcf >> 8) & 0xFF);
        const uint32_t ca = ((o.kcf >> 16) & F_NOISE) && o.c != NO_SLOT && o.c < hp.noise.size() ? hp.noise[o.c].ca : 1u;
        const uint32_t Kc = std::max<uint32_t>(1u, warp_share(o.count, nw, ca));
        for (uint32_t j = 0; j < o.count; j++) {
            const uint32_t r = std::min(nw - 1, j / Kc);
            for (int s2 = 0; s2 < ar; s2++) {
                const uint32_t q = hp.targets[o.off + (size_t)j * ar + s2];
                const uint32_t cell = (uint32_t)((u * nw + r) * 2 + s2);
                occ[q].push_back(Occ{cell, weight[u]});
                if (cls[q] >= 0) cnt[(size_t)cell * G + cls[q]]++;
                cap[cell]++;
            }
        }
    }
    for (int32_t& c : cap) c = (c + (int32_t)G - 1) / (int32_t)G;  // even split
    std::vector<uint32_t> movable;
    for (uint32_t q = 0; q < n; q++)
        if (cls[q] >= 0 && !occ[q].empty()) movable.push_back(q);
    if (movable.size() < 2) return;
    auto over = [&](uint32_t cell, int32_t c) { return std::max(0, cnt[(size_t)cell * G + c] - cap[cell]); };
    auto move = [&](uint32_t q, int32_t from, int32_t to) -> int64_t {  // returns the cost change
        int64_t d = 0;
        for (const Occ& oc : occ[q]) {
            d -= (int64_t)oc.w * (over(oc.cell, from) + over(oc.cell, to));
            cnt[(size_t)oc.cell * G + from]--;
            cnt[(size_t)oc.cell * G + to]++;
            d += (int64_t)oc.w * (over(oc.cell, from) + over(oc.cell, to));
        }
        return d;
    };
    uint64_t st = 0xD1B54A32D192ED03ull ^ n;
    auto rnd = [&]() { st += 0x9E3779B97F4A7C15ull; uint64_t z = st; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                       z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); };
    const uint64_t iters = std::min<uint64_t>(6000000ull, 600ull * movable.size());
    for (uint64_t it = 0; it < iters; it++) {
        const uint32_t a = movable[rnd() % movable.size()], b = movable[rnd() % movable.size()];
        const int32_t ca2 = cls[a], cb2 = cls[b];
        if (ca2 == cb2) continue;
        int64_t d = move(a, ca2, cb2);
        d += move(b, cb2, ca2);
        if (d <= 0) { cls[a] = cb2; cls[b] = ca2; }
        else { move(b, ca2, cb2); move(a, cb2, ca2); }
    }
}

void permute_rows(HostProgram& hp, int bank_classes, int warps_per_group) {
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
    // Bank classes (row mod G, G = 128 B / row bytes): a warp pass serves G
    // consecutive applications per shared-memory wavefront, conflict-free when
    // their rows fall into G distinct classes.  Walk the gate ops in program
    // order and give every qubit, at its first appearance, the class of its
    // application's position (j mod G): in circuits whose layers list their
    // applications in a regular (lattice) order, neighbouring applications then
    // land in distinct classes in every layer.  Rows are dealt per class from
    // the random permutation (a full class takes from the emptiest one).
    const uint32_t G = (uint32_t)std::max(1, bank_classes);
    if (G > 1 && n >= G) {
        std::vector<int32_t> cls(n, -1);
        for (const DOp& o : hp.ops) {
            if ((o.kcf & 0xFF) != K_GATE) continue;
            const int ar = rule_arity((o.kcf >> 8) & 0xFF);
            for (uint32_t j = 0; j < o.count; j++)
                for (int s2 = 0; s2 < ar; s2++) {
                    const uint32_t q = hp.targets[o.off + (size_t)j * ar + s2];
                    if (cls[q] < 0) cls[q] = (int32_t)(j % G);
                }
        }
        // class sizes must fit the row pools: move the overflow to the emptiest classes
        {
            std::vector<uint32_t> size(G, 0), room(G, 0);
            for (uint32_t q = 0; q < n; q++) room[hp.row_of[q] % G]++;
            for (uint32_t q = 0; q < n; q++) if (cls[q] >= 0) size[cls[q]]++;
            for (uint32_t q = n; q-- > 0;) {
                if (cls[q] < 0 || size[cls[q]] <= room[cls[q]]) continue;
                uint32_t best = 0;
                for (uint32_t c = 1; c < G; c++)
                    if ((int64_t)room[c] - size[c] > (int64_t)room[best] - size[best]) best = c;
                size[cls[q]]--;
                cls[q] = (int32_t)best;
                size[best]++;
            }
        }
        if (warps_per_group > 0 && G <= 8) refine_classes(hp, cls, G, (uint32_t)warps_per_group);
        // pools: the rows of each class, in the order of the random permutation
        std::vector<std::vector<uint32_t>> pool(G);
        for (uint32_t q = 0; q < n; q++) pool[hp.row_of[q] % G].push_back(hp.row_of[q]);
        std::vector<uint32_t> rest;
        for (uint32_t q = 0; q < n; q++) {
            if (cls[q] >= 0 && !pool[cls[q]].empty()) {
                hp.row_of[q] = pool[cls[q]].back();
                pool[cls[q]].pop_back();
            } else {
                rest.push_back(q);
            }
        }
        for (uint32_t q : rest) {
            uint32_t best = 0;
            for (uint32_t c = 1; c < G; c++)
                if (pool[c].size() > pool[best].size()) best = c;
            hp.row_of[q] = pool[best].back();
            pool[best].pop_back();
        }
    }
    auto map = [&](uint32_t& w) { w = hp.row_of[w & ~COIN_DEAD] | (w & COIN_DEAD); };
    auto map_term = [&](uint32_t& t) { if (t != NO_SLOT && (t & XROW)) t = XROW | hp.row_of[t & ~XROW]; };
    for (const DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF, code = (o.kcf >> 8) & 0xFF;
        uint32_t* t = hp.targets.data() + o.off;
        switch (kind) {
            case K_GATE: for (uint32_t j = 0; j < o.count * rule_arity(code); j++) map(t[j]); break;
            case K_M: case K_MR: case K_R: case K_SPILL: for (uint32_t j = 0; j < o.count; j++) map(t[2 * j]); break;
            case K_NOISE:
                for (uint32_t j = 0; j < o.count * channel_arity(code); j++) map(t[j]);
                break;
            case K_OBS: for (uint32_t j = 0; j < o.count; j++) map_term(t[j]); break;
            default: break;
        }
    }
    for (uint32_t& t : hp.det_terms) map_term(t);
}

// Bank-aware order of A applications (ar targets each) in place: each
// aligned group of G consecutive applications (the apps one shared-memory
// wavefront serves: G = 128 B / row bytes) touches G distinct bank groups per
// operand: apps are classed by (first, second) operand residue mod G and each
// group takes one app per first residue, choosing among the second residues
// still unused the fullest class.
static void bank_reorder(uint32_t* tg, uint32_t A, int ar, int G, std::vector<uint32_t>& scratch) {
    if (G <= 1 || A < 2) return;
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

static int bank_groups(int W) { return W >= 32 ? 1 : 128 / (W * 4); }

// Applications per warp of a group for an op of `apps` applications: an even
// split rounded up to whole noise chunks (ca applications), so every chunk of
// a fused noise instruction has one owner warp.
static uint32_t warp_share(uint32_t apps, uint32_t nw, uint32_t ca) {
    ca = std::max<uint32_t>(1u, ca);
    return ((apps + nw - 1) / nw + ca - 1) / ca * ca;
}

// Stream form of the device ops for tiles of W words run by groups of
// `warps_per_group` warps (SOp, pfs_internal.h).  Every gate op becomes one
// block of packed operand words per warp: the warp's (chunk-aligned) range of
// applications in bank order, padded to whole warp passes, so the kernel's
// item loop is a coalesced word load, two shifts and the row work.  Collapses,
// detectors and observables get a copy of their operand lists; identical
// blocks (the rounds of a REPEAT body) are stored once.
void lower_stream(HostProgram& hp, int W, int warps_per_group) {
    const int V = W >= 4 ? 4 : W, C = W / V;
    const uint32_t PI = 32u / (uint32_t)C;  // applications per warp pass
    const uint32_t nw = (uint32_t)std::max(1, warps_per_group);
    const int G = bank_groups(W);
    if (hp.num_qubits + DUMMY_ROWS >= 65536) bad("frame rows exceed the 16-bit operand format");
    hp.sops.assign(hp.ops.size(), SOp{});
    hp.arena.clear();
    hp.first_span = NO_SLOT;
    hp.all_presampled = true;
    std::unordered_map<uint64_t, std::vector<std::pair<uint32_t, uint32_t>>> seen;
    auto add_block = [&](const std::vector<uint32_t>& blk) -> uint32_t {
        if (blk.empty()) return 0u;
        uint64_t h = 1469598103934665603ull ^ blk.size();
        for (uint32_t v : blk) { h ^= v; h *= 1099511628211ull; }
        auto& lst = seen[h];
        for (auto& c : lst)
            if (c.second == blk.size() && std::equal(blk.begin(), blk.end(), hp.arena.begin() + c.first)) return c.first;
        while (hp.arena.size() & 31) hp.arena.push_back(STREAM_NOP);  // 128-byte aligned blocks
        const uint32_t where = (uint32_t)hp.arena.size();
        hp.arena.insert(hp.arena.end(), blk.begin(), blk.end());
        lst.emplace_back(where, (uint32_t)blk.size());
        return where;
    };
    std::vector<uint32_t> blk, range, scratch;
    for (size_t i = 0; i < hp.ops.size(); i++) {
        const DOp& o = hp.ops[i];
        SOp& s = hp.sops[i];
        const uint32_t kind = o.kcf & 0xFF, code = (o.kcf >> 8) & 0xFF, flags = o.kcf >> 16;
        s.kcf = o.kcf;
        s.count = o.count;
        s.a = o.a;
        s.b = o.b;
        s.span = s.next_span = NO_SLOT;
        s.ordinal = (kind == K_NOISE || (flags & F_NOISE)) ? o.c : NO_SLOT;
        const bool fz = (flags & F_NOISE) != 0;
        const uint32_t ca = fz ? hp.noise[o.c].ca : 1u;
        if ((fz || kind == K_NOISE) && hp.noise[o.c].zone != NZONE_NONE &&
            (!fz || hp.fused_info.empty() || hp.fused_info[(size_t)o.c * 4 + 1] != 1u))
            hp.all_presampled = false;
        if (fz && hp.noise[o.c].zone == NZONE_NONE) s.kcf &= ~(F_NOISE << 16);  // p == 0: nothing to apply
        if (fz && !hp.fused_info.empty() && hp.fused_info[(size_t)o.c * 4 + 1] == 1u) {
            s.kcf |= F_PRESAMPLED << 16;
            s.span = o.c * (uint32_t)hp.list_warps;
        }
        blk.clear();
        switch (kind) {
        case K_GATE: {
            const int ar = rule_arity(code);
            const uint32_t Kc = warp_share(o.count, nw, ca);
            const uint32_t passes = (Kc + PI - 1) / PI;
            // a warp's block holds at least GATE_AHEAD_PASSES passes (the kernel
            // prefetches that many words per lane without predicates);
            // padding applications act on the group's dummy rows (rows num_qubits ..)
            const uint32_t stride = std::max<uint32_t>(passes, GATE_AHEAD_PASSES) * PI;
            blk.resize((size_t)nw * stride);
            for (size_t j = 0; j < blk.size(); j++) {
                const uint32_t dr = (uint32_t)hp.num_qubits + (uint32_t)(j % DUMMY_ROWS);
                blk[j] = dr | (dr << 16);
            }
            for (uint32_t w = 0; w < nw; w++) {
                const uint32_t A0 = std::min(o.count, w * Kc), A1 = std::min(o.count, A0 + Kc);
                if (A0 >= A1) continue;
                range.assign(hp.targets.begin() + o.off + (size_t)A0 * ar, hp.targets.begin() + o.off + (size_t)A1 * ar);
                bank_reorder(range.data(), A1 - A0, ar, G, scratch);
                for (uint32_t j = 0; j < A1 - A0; j++)
                    blk[(size_t)w * stride + j] = range[(size_t)j * ar] | (ar == 2 ? range[(size_t)j * ar + 1] << 16 : 0u);
            }
            s.K = passes;
            s.r0 = Kc;
            break;
        }
        case K_M: case K_MR: case K_R: case K_SPILL: {
            blk.assign(hp.targets.begin() + o.off, hp.targets.begin() + o.off + 2 * (size_t)o.count);
            s.K = warp_share(o.count, nw, ca);
            // an event-program M whose coins are all dead and whose records all
            // stay in their x rows has no row work (only its fused noise)
            bool norows = kind == K_M && hp.mode == PM_EVENTS;
            for (uint32_t j = 0; norows && j < o.count; j++)
                norows = (blk[2 * j] & COIN_DEAD) && blk[2 * j + 1] == NO_SLOT;
            if (norows) s.kcf |= F_NOROWS << 16;
            break;
        }
        case K_DET:
            if (code) blk.assign(hp.det_terms.begin() + o.off, hp.det_terms.begin() + o.off + (size_t)o.count * code);
            break;
        case K_OBS:
            blk.assign(hp.targets.begin() + o.off, hp.targets.begin() + o.off + o.count);
            break;
        default: break;  // standalone noise reads its DOp
        }
        s.off = blk.empty() ? o.off : add_block(blk);
    }
    uint32_t next = NO_SLOT;
    for (size_t i = hp.sops.size(); i-- > 0;) {
        SOp& s = hp.sops[i];
        if (!((s.kcf >> 16) & F_PRESAMPLED)) continue;
        s.next_span = next == NO_SLOT ? s.span : next;
        next = s.span;
    }
    hp.first_span = next;
    if (hp.arena.size() >= (1ull << 31)) bad("operand arena too large");
}

// Pre-sampled fused noise (noise_kernel): a fused op's consumer warp w owns
// applications [w K, w K + K) (K = ceil(apps / warps) rounded up to whole
// chunks, the kernel's warp_range), and reads its hits from a fixed-capacity
// list filled by noise_kernel (capacity = mean + 6 sigma + 8; a fuller list,
// or a chunk needing the general path, is left to the consumer to draw).
void build_hit_lists(HostProgram& hp, int tile_shots, int warps_per_group) {
    const uint32_t nw = (uint32_t)std::max(1, warps_per_group);
    hp.list_warps = (int32_t)nw;
    hp.fused_info.assign((size_t)hp.num_noise * 4, 0u);
    hp.hit_items.clear();
    double mean_all = 0.0;
    for (const DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF;
        if (!((o.kcf >> 16) & F_NOISE) || o.c == NO_SLOT) continue;
        const NoiseParam& np = hp.noise[o.c];
        if (np.zone != NZONE_TAB) continue;  // p == 0 / p == 1: drawn by the consumer
        const uint32_t K = warp_share(np.apps, nw, np.ca);
        const double p = hp.noise_p[o.c];
        // consumer warps per noise_kernel item: as many as keep the item's hits
        // (mean + 6 sigma + slack) within one warp's staging buffer
        const double per_warp = (double)K * tile_shots * p;
        uint32_t wpi = std::min<uint32_t>(nw, 16u);  // noise_kernel tags a hit's consumer warp in 4 bits
        while (wpi > 0 && per_warp * wpi + 6.0 * std::sqrt(per_warp * wpi) + 16.0 > (double)NK_SCR) wpi--;
        if (wpi == 0) continue;  // heavy noise: drawn by the consumer
        uint32_t* fi = &hp.fused_info[(size_t)o.c * 4];
        fi[0] = K;
        fi[1] = 1u;
        fi[3] = o.off | (kind == K_GATE ? 0u : FUSED_PAIRS);
        for (uint32_t wb = 0; wb < nw; wb += wpi) {
            hp.hit_items.push_back(o.c);
            hp.hit_items.push_back(wb | (std::min(nw, wb + wpi) << 16));
        }
        mean_all += (double)np.apps * tile_shots * p;
    }
    // a tile's entries; an item that finds the block full leaves its warps to
    // draw inline (still exact), so the bound only sets how rare that is
    hp.hit_block = hp.hit_items.empty() ? 0 : (int64_t)std::ceil(mean_all + 8.0 * std::sqrt(mean_all) + 256.0);
    if (hp.hit_block >= (1ll << 31)) bad("noise hit lists too large");
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
            case K_M: case K_MR: case K_R: case K_SPILL:
                o.off = canon(seen_t, hp.targets, o.off, 2 * (size_t)o.count);
                break;
            case K_OBS: o.off = canon(seen_t, hp.targets, o.off, o.count); break;
            case K_NOISE: o.off = canon(seen_t, hp.targets, o.off, (size_t)o.count * channel_arity(code)); break;
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

static uint32_t ilog2(uint64_t v) {
    uint32_t l = 0;
    while ((1ull << l) < v) l++;
    return l;
}

// Chunk geometry and Binomial tables of every noise instruction (DESIGN.md
// §4).  L = the power of two nearest (in ratio) to target / p trials (fused
// instructions use their own, smaller target: one kernel item owns a chunk's
// ca applications), cs = min(L, S) shots, ca = L / cs applications.
void build_noise_schedule(HostProgram& hp, int tile_shots, int vector_shots, double target_hits,
                          double fused_target_hits) {
    hp.noise_tab.clear();
    hp.noise.assign(hp.num_noise, NoiseParam{});
    std::map<std::pair<uint32_t, double>, std::pair<uint32_t, uint32_t>> tabs;  // (L, p) -> (offset, len)
    const uint64_t T = (uint64_t)tile_shots;
    for (int64_t j = 0; j < hp.num_noise; j++) {
        NoiseParam& np = hp.noise[j];
        const uint32_t ch = hp.noise_ch[j];
        np.ch = ch;
        np.npat = ch == CH_DEP1 ? 3u : (ch == CH_DEP2 ? 15u : 1u);
        np.apps = hp.noise_apps[j];
        np.fused = hp.noise_fused[j];
        const uint64_t N = (uint64_t)np.apps * T;
        const double p = hp.noise_p[j];
        uint64_t L = 1;
        if (N == 0 || p <= 0.0) {
            np.zone = NZONE_NONE;
        } else if (p >= 1.0) {
            np.zone = NZONE_ALL;
            while (L < N && L < 1024) L *= 2;  // power of two; positions stay below 2^28
        } else {
            np.zone = NZONE_TAB;
            const double want = (np.fused ? fused_target_hits : target_hits) / p;
            while ((double)(L * 2) <= want * 1.41421356 && L < (1ull << 27)) L *= 2;
            while (L > 1 && L / 2 >= N) L /= 2;  // no chunk longer than needed
        }
        if (N >= (1ull << 31)) bad("noise instruction too large for one tile");
        const uint64_t cs = std::min<uint64_t>(L, (uint64_t)vector_shots);
        np.L = (uint32_t)L;
        np.cs = (uint32_t)cs;
        np.ca = (uint32_t)(L / cs);
        const uint64_t nA = (np.apps + (uint64_t)np.ca - 1) / np.ca;
        const uint64_t nch = nA * (T / cs);
        if (nch >= (1ull << 31)) bad("noise instruction too large for one tile");
        np.nchunks = (uint32_t)nch;
        if (np.zone == NZONE_TAB) {
            // every chunk draws from Binomial(L, p): trials past the end are virtual and dropped
            auto key = std::make_pair((uint32_t)L, p);
            auto it = tabs.find(key);
            if (it == tabs.end()) {
                auto tf = binomial_thresholds(L, p);
                if (tf.size() > 255) bad("noise threshold table too long");
                it = tabs.emplace(key, std::make_pair((uint32_t)hp.noise_tab.size(), (uint32_t)tf.size())).first;
                hp.noise_tab.insert(hp.noise_tab.end(), tf.begin(), tf.end());
            }
            np.tab = it->second.first;
            np.len = it->second.second;
        }
    }
    if (hp.noise_tab.size() >= (1u << 24)) bad("noise threshold tables too large");
    for (DOp& o : hp.ops) {
        const uint32_t kind = o.kcf & 0xFF, flags = o.kcf >> 16;
        if (!(kind == K_NOISE || (flags & F_NOISE))) continue;
        const NoiseParam& np = hp.noise[o.c];
        o.d = ilog2(np.L) | (ilog2(np.cs) << 5) | (np.npat << 10) | (np.ch << 14) | (np.zone << 17);
        o.e = np.tab | (np.len << 24);
    }
}

}  // namespace pfs
