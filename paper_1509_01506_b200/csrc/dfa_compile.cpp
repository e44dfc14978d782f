// Host-side compilation of a reference Dfa into its device form.
//
// Input layout is the reference's (automaton.py:26-51): transitions
// int32[nq][5] (a,c,g,t,OTHER), CSR output multisets.  Output (HostDfa):
//   * renumbering: accepting states first, so the device hit test is
//     `state < n_accept` instead of two out_offsets loads per symbol
//     (the reference's inner CSR loop, _kernels.py:26-28);
//   * K-symbol stride table: one uint16 load advances K bases; bit 15 flags
//     "some state entered on this K-step has outputs";
//   * synchronisation depth D: the smallest k such that every k-symbol word
//     maps all states to one state.  For Aho-Corasick tables with OTHER ->
//     START, D <= longest literal.  With D known, the true state at any
//     position is the state reached by scanning the D preceding symbols from
//     any state -- no speculation, no cross-chunk dependency;
//   * otherwise the transition monoid (closure of the 5 column maps) when it
//     is small: chunk maps become monoid element ids, composed by a
//     product-table lookup in an exclusive device-wide scan.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <unordered_set>

#include "ks_internal.h"

namespace ks {
namespace {

struct VecHash {
    template <class T>
    size_t operator()(const std::vector<T>& v) const noexcept {
        uint64_t h = 1469598103934665603ull ^ v.size();
        for (T x : v) h = (h ^ x) * 1099511628211ull;
        return static_cast<size_t>(h);
    }
};

int stride_for(int nq, size_t budget) {
    const char* force = std::getenv("KS_FORCE_STRIDE");
    if (force && *force) {
        int k = std::atoi(force);
        if (k >= 1 && k <= 4) return k;
    }
    for (int k = 4; k >= 2; --k) {
        size_t bytes = size_t(nq) * (size_t(1) << (2 * k)) * 2 + size_t(nq) * 5 * 2;
        if (bytes <= budget) return k;
    }
    return 1;   // K = 1 scans the 1-base table itself (no stride table)
}

void build_stride_table(CompiledTable* t, size_t budget) {
    const int nq = t->nq;
    const int k = stride_for(nq, budget);
    t->stride = k;
    const int words = 1 << (2 * k);
    t->tk.assign(k == 1 ? 0 : size_t(nq) * words, 0);
    for (int s = 0; s < (k == 1 ? 0 : nq); ++s) {
        for (int w = 0; w < words; ++w) {
            int x = s;
            bool hit = false;
            for (int i = 0; i < k; ++i) {
                x = t->t1[size_t(x) * 5 + ((w >> (2 * i)) & 3)];
                hit |= x < t->n_accept;
            }
            t->tk[size_t(s) * words + w] = uint16_t(x | (hit ? kFlag : 0));
        }
    }
    // fast form
    t->fast_k = 0;
    t->tkc.clear();
    t->t1z.clear();
    if (nq <= 4096 && !(std::getenv("KS_DISABLE_FAST") && *std::getenv("KS_DISABLE_FAST") == '1')) {
        const int fk = nq <= 256 ? 4 : (nq <= 1024 ? 3 : 2);
        const int sb = 16 - 2 * fk;  // state bits
        const int fw = 1 << (2 * fk);
        const int z = nq;
        t->fast_k = fk;
        t->tkc.assign(size_t(1) << 16, uint16_t(z << 1));
        for (int w = 0; w < fw; ++w) {
            for (int s = 0; s < nq; ++s) {
                int x = s;
                bool hit = false;
                bool first_hit = false;
                for (int i = 0; i < fk; ++i) {
                    x = t->t1[size_t(x) * 5 + ((w >> (2 * i)) & 3)];
                    hit |= x < t->n_accept;
                    if (i == 0) first_hit = x < t->n_accept;
                }
                // bit 15: any state on the K-step accepting (ring modes); for
                // K = 2 also bit 13: the intermediate one, bit 14: the final one
                // (direct counting).  Bits >= LC are overwritten by the next
                // lookup's input field, so they never reach an address.
                uint32_t v = uint32_t(x << 1) | (hit ? 0x8000u : 0u);
                if (fk == 2) v |= (first_hit ? 0x2000u : 0u) | (x < t->n_accept ? 0x4000u : 0u);
                // K >= 3: row-swizzled (scan_fast.cu swizzled())
                const int row = fk >= 3 ? (s ^ (w & 31)) : s;
                t->tkc[(size_t(w) << sb) + row] = uint16_t(v);
            }
        }
    }
    {  // hit-rate estimate: 64 Ki uniform random bases from state 0 (xorshift)
        uint64_t z = 0x9E3779B97F4A7C15ull;
        int x = 0;
        int64_t hits = 0;
        const int steps = 1 << 16;
        for (int i = 0; i < steps; ++i) {
            z ^= z << 13;
            z ^= z >> 7;
            z ^= z << 17;
            x = t->t1[size_t(x) * 5 + (z & 3)];
            hits += x < t->n_accept;
        }
        t->hit_rate = double(hits) / steps;
    }
    const uint16_t r = t->t1[4];
    bool resets = true;
    for (int s = 1; s < nq && resets; ++s) resets = t->t1[size_t(s) * 5 + 4] == r;
    t->reset_state = resets ? int(r) : -1;
    // the fast kernel's 1-base table: 4 columns when OTHER resets every state
    // (smaller shared footprint, a deeper hit ring), else all 5
    if (t->fast_k) {
        t->t1z_cols = resets ? 4 : 5;
        t->t1z.assign(size_t(nq + 1) * t->t1z_cols, uint16_t(nq));
        for (int s = 0; s < nq; ++s)
            for (int c = 0; c < t->t1z_cols; ++c) t->t1z[size_t(s) * t->t1z_cols + c] = t->t1[size_t(s) * 5 + c];
    }
}

// Visit-class form of a K = 2 fast table (CompiledTable::cls_*).  A 2-base
// step from s over (b1, b2) passes I = t1[s][b1] and ends in F = t1[I][b2].
// When I accepts, the entry's row/sub names the pair (out(I), F): the row
// carries F's transitions, (row, sub) the histogram slot whose multiset is
// out(I) + out(F).  Each state holds three such pairs in subs 1-3 of its own
// row (sub 0: I does not accept, the slot of out(F) alone); further pairs get
// copies of the row.  One histogram add per accepting K-step, no re-walk of
// the intermediate state.  Returns false (no class form) when the rows do
// not fit 12-bit ids.
bool build_class_table(CompiledTable* t, const std::vector<int32_t>& acc_off, const std::vector<int32_t>& acc_ids) {
    t->cls_rows = t->cls_nhist = 0;
    t->cls_tk.clear();
    t->cls_t1.clear();
    t->cls_prim.clear();
    t->cls_out_off.clear();
    t->cls_out_ids.clear();
    t->cls_used.clear();
    if (t->fast_k != 2 || t->t1z.empty()) return false;
    const int nq = t->nq, A = t->n_accept;
    auto key = [&](int s) { return std::vector<int32_t>(acc_ids.begin() + acc_off[s], acc_ids.begin() + acc_off[s + 1]); };
    // accepting-intermediate multisets entering each state (sorted, distinct)
    std::vector<std::vector<std::vector<int32_t>>> pairs(nq);
    for (int s = 0; s < nq; ++s)
        for (int b1 = 0; b1 < 4; ++b1) {
            const int I = t->t1[size_t(s) * 5 + b1];
            if (I >= A) continue;
            for (int b2 = 0; b2 < 4; ++b2) pairs[t->t1[size_t(I) * 5 + b2]].push_back(key(I));
        }
    struct Slot { int row, sub; };
    std::vector<std::unordered_map<std::vector<int32_t>, Slot, VecHash>> where(nq);
    std::vector<uint16_t> prim(nq + 1);
    std::iota(prim.begin(), prim.end(), uint16_t(0));
    int next_row = nq + 1;   // row nq is the padding row
    for (int F = 0; F < nq; ++F) {
        auto& v = pairs[F];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        for (size_t k = 0; k < v.size(); ++k) {
            Slot sl;
            if (k < 3) {
                sl = {F, int(k) + 1};
            } else {
                if ((k - 3) % 4 == 0) {
                    prim.push_back(uint16_t(F));
                    ++next_row;
                }
                sl = {next_row - 1, int((k - 3) % 4)};
            }
            where[F][v[k]] = sl;
        }
    }
    const int rows = next_row;
    if (rows > 4096) return false;
    t->cls_tk.assign(size_t(1) << 16, uint16_t(nq << 1));
    for (int r = 0; r < rows; ++r) {
        if (r == nq) continue;
        const int s = prim[r];
        for (int w = 0; w < 16; ++w) {
            const int I = t->t1[size_t(s) * 5 + (w & 3)];
            const int F = t->t1[size_t(I) * 5 + (w >> 2)];
            uint32_t v;
            if (I < A) {
                const Slot sl = where[F].at(key(I));
                v = uint32_t(sl.row << 1) | uint32_t(sl.sub << 13) | 0x8000u;
            } else {
                v = uint32_t(F << 1) | (F < A ? 0x8000u : 0u);
            }
            t->cls_tk[(size_t(w) << 12) + r] = uint16_t(v);
        }
    }
    const int cols = t->t1z_cols;
    t->cls_t1.assign(size_t(rows) * cols, 0);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) t->cls_t1[size_t(r) * cols + c] = t->t1z[size_t(std::min<int>(prim[r], nq)) * cols + c];
    // slot multisets: (sub << 12) | row
    std::vector<std::vector<int32_t>> ms(size_t(4) << 12);
    int nhist = 0;
    for (int F = 0; F < A; ++F) {
        ms[F] = key(F);
        nhist = std::max(nhist, F + 1);
    }
    for (int F = 0; F < nq; ++F)
        for (const auto& kv : where[F]) {
            const int idx = (kv.second.sub << 12) | kv.second.row;
            auto m = kv.first;
            if (F < A) {
                const auto o = key(F);
                m.insert(m.end(), o.begin(), o.end());
            }
            ms[idx] = std::move(m);
            nhist = std::max(nhist, idx + 1);
        }
    t->cls_out_off.assign(1, 0);
    t->cls_used.clear();
    for (int i = 0; i < nhist; ++i) {
        t->cls_out_ids.insert(t->cls_out_ids.end(), ms[i].begin(), ms[i].end());
        t->cls_out_off.push_back(int32_t(t->cls_out_ids.size()));
        if (!ms[i].empty()) t->cls_used.push_back(i);
    }
    t->cls_prim = prim;
    t->cls_rows = rows;
    t->cls_nhist = nhist;
    return true;
}

// Smallest D with |delta(Q, w)| == 1 for all |w| == D, or -1.
template <class T>
int synchronisation_depth(const std::vector<T>& t1, int nq) {
    if (nq <= 1) return 0;
    std::vector<std::vector<T>> level(1);
    level[0].resize(nq);
    std::iota(level[0].begin(), level[0].end(), T(0));
    std::vector<uint32_t> stamp(nq, 0);
    uint32_t tick = 0;
    int64_t work = 0;
    const int64_t budget = 200000000;
    std::vector<T> img;
    for (int k = 0; k < kMaxSyncDepth; ++k) {
        std::unordered_set<std::vector<T>, VecHash> next;
        for (const auto& set : level) {
            for (int c = 0; c < 5; ++c) {
                ++tick;
                img.clear();
                for (T q : set) {
                    T x = t1[size_t(q) * 5 + c];
                    if (stamp[x] != tick) {
                        stamp[x] = tick;
                        img.push_back(x);
                    }
                }
                work += int64_t(set.size());
                if (img.size() > 1) {
                    std::sort(img.begin(), img.end());
                    next.insert(img);
                }
            }
            if (work > budget) return -1;
        }
        if (next.empty()) return k + 1;
        // a level that maps onto itself never shrinks (e.g. permutation columns)
        if (next.size() == level.size() &&
            std::all_of(level.begin(), level.end(), [&](const std::vector<T>& v) { return next.count(v); }))
            return -1;
        level.assign(next.begin(), next.end());
    }
    return -1;
}

// Closure of the column maps; false if it exceeds the caps.  With `sub`
// (OTHER resets every state) the OTHER-free submonoid is closed first, so its
// elements take the ids [0, nS), and `mono` is built over it alone.
bool build_monoid(const CompiledTable& t, int start, bool sub, HostDfa* h) {
    const int nq = t.nq;
    const size_t cap_entries = size_t(16) << 20;
    std::vector<uint16_t> maps(nq);
    std::iota(maps.begin(), maps.end(), uint16_t(0));
    std::vector<int32_t> parent{-1}, psym{-1};
    std::unordered_map<std::string, int> ids;
    auto key_of = [&](const uint16_t* m) {
        return std::string(reinterpret_cast<const char*>(m), size_t(nq) * 2);
    };
    ids.emplace(key_of(maps.data()), 0);
    std::vector<int32_t> mt(5, -1);  // nm x 5
    std::vector<uint16_t> next(nq);
    int n_sub = -1;
    for (int phase = sub ? 0 : 1; phase < 2; ++phase) {
        const int nsym = phase == 0 ? 4 : 5;
        for (size_t m = 0; m < parent.size(); ++m) {
            for (int c = 0; c < nsym; ++c) {
                if (mt[m * 5 + c] >= 0) continue;
                const uint16_t* src = &maps[m * nq];
                for (int q = 0; q < nq; ++q) next[q] = t.t1[size_t(src[q]) * 5 + c];
                auto key = key_of(next.data());
                auto it = ids.find(key);
                int id;
                if (it == ids.end()) {
                    id = int(parent.size());
                    if (id >= kMaxMonoid || size_t(id + 1) * nq > cap_entries) return false;
                    ids.emplace(std::move(key), id);
                    maps.insert(maps.end(), next.begin(), next.end());
                    parent.push_back(int32_t(m));
                    psym.push_back(c);
                    mt.resize(mt.size() + 5, -1);
                } else {
                    id = it->second;
                }
                mt[m * 5 + c] = id;
            }
        }
        if (phase == 0) n_sub = int(parent.size());
    }
    const int nm = int(parent.size());
    h->nm = nm;
    h->mono_sub = sub;
    h->mono_other = mt[4];
    const int nrow = sub ? n_sub : nm;
    h->mono.nq = nrow;
    h->mono.n_accept = 0;
    h->mono.t1.resize(size_t(nrow) * 5);
    for (int m = 0; m < nrow; ++m)
        for (int c = 0; c < 5; ++c)   // submonoid: OTHER is tracked by the kernels, the column is the identity
            h->mono.t1[size_t(m) * 5 + c] = uint16_t(sub && c == 4 ? 0 : mt[size_t(m) * 5 + c]);
    h->prod.assign(size_t(nm) * nm, 0);
    for (int a = 0; a < nm; ++a) {
        uint16_t* row = &h->prod[size_t(a) * nm];
        row[0] = uint16_t(a);
        for (int b = 1; b < nm; ++b)  // parents precede children in discovery order
            row[b] = uint16_t(mt[size_t(row[parent[b]]) * 5 + psym[b]]);
    }
    h->act0.resize(nm);
    for (int m = 0; m < nm; ++m) h->act0[m] = maps[size_t(m) * nq + start];
    h->action = std::move(maps);
    return true;
}

}  // namespace

int compile_dfa(const int32_t* trans, int nq, const int32_t* out_off, const int32_t* out_ids,
                int ne, int force_strategy, size_t smem_budget, HostDfa* h) {
    if (!trans || !out_off || nq < 1) return fail(KS_E_INVALID, "dfa: empty transition table");
    if (nq > (1 << 30)) return fail(KS_E_UNSUPPORTED, "dfa: too many states");
    if (ne < 0) return fail(KS_E_INVALID, "dfa: negative expression count");
    if (out_off[0] != 0) return fail(KS_E_INVALID, "dfa: out_offsets[0] must be 0");
    for (int s = 0; s < nq; ++s) {
        if (out_off[s + 1] < out_off[s]) return fail(KS_E_INVALID, "dfa: out_offsets not monotone");
        for (int c = 0; c < 5; ++c) {
            int32_t x = trans[size_t(s) * 5 + c];
            if (x < 0 || x >= nq) return fail(KS_E_INVALID, "dfa: transition target out of range");
        }
    }
    const int32_t n_out = out_off[nq];
    if (n_out > 0 && !out_ids) return fail(KS_E_INVALID, "dfa: missing out_ids");
    for (int32_t i = 0; i < n_out; ++i)
        if (out_ids[i] < 0 || out_ids[i] >= ne) return fail(KS_E_INVALID, "dfa: output id out of range");

    h->nq = nq;
    h->ne = ne;
    h->new_of_old.assign(nq, 0);
    h->old_of_new.clear();
    int hot_lo = 0, hot_n = 0;
    // the wide form (32-bit ids, hot table in shared memory + cold
    // transitions from L2) above the 16-bit range, and for definite automata
    // whose 1-base table does not fit shared memory (~22K-32K states: the
    // 16-bit kernel would read it through L1/L2 on every step)
    bool wide = nq > kMaxStates;
    if (!wide && nq > 16384 && (force_strategy == 0 || force_strategy == KS_STRATEGY_LOOKBACK)) {
        size_t acc_n = 0;
        for (int s = 0; s < nq; ++s) acc_n += out_off[s + 1] > out_off[s];
        if (size_t(nq) * 10 + acc_n * 4 + 4096 > smem_budget) {
            const std::vector<uint32_t> t(trans, trans + size_t(nq) * 5);
            wide = synchronisation_depth(t, nq) >= 0;
        }
    }
    if (wide) {
        // wide automata: accepting states still first ([0, A): the hit test),
        // and the hot set -- the states nearest START (BFS depth, then id:
        // a scan of AC-like automata spends almost every step there) -- one
        // contiguous range: [cold accepting | hot accepting | hot other | cold other]
        std::vector<int32_t> depth(nq, -1), q;
        q.reserve(nq);
        depth[0] = 0;
        q.push_back(0);
        for (size_t i = 0; i < q.size(); ++i)
            for (int c = 0; c < 5; ++c) {
                const int32_t x = trans[size_t(q[i]) * 5 + c];
                if (depth[x] < 0) {
                    depth[x] = depth[q[i]] + 1;
                    q.push_back(x);
                }
            }
        std::vector<int32_t> by(nq);
        std::iota(by.begin(), by.end(), 0);
        auto key = [&](int32_t x) { return depth[x] < 0 ? INT32_MAX : depth[x]; };
        std::stable_sort(by.begin(), by.end(), [&](int32_t x, int32_t y) { return key(x) < key(y); });
        const int A = int(std::count_if(by.begin(), by.end(), [&](int32_t x) { return out_off[x + 1] > out_off[x]; }));
        const size_t hist = std::min<size_t>(size_t(A) * 4, 64 * 1024);
        const size_t room = smem_budget > hist + 4096 ? smem_budget - hist - 4096 : 0;
        hot_n = int(std::min<size_t>({size_t(nq), size_t(32766), room / 8}));
        if (const char* e = std::getenv("KS_WIDE_HOT_STATES"); e && *e)   // test knob: a smaller hot set
            hot_n = std::max(0, std::min(hot_n, std::atoi(e)));
        std::vector<char> hot(nq, 0);
        for (int i = 0; i < hot_n; ++i) hot[by[i]] = 1;
        auto acc = [&](int32_t x) { return out_off[x + 1] > out_off[x]; };
        for (int32_t x = nq - 1; x >= 0; --x)   // cold accepting, deepest first
            if (acc(by[x]) && !hot[by[x]]) h->old_of_new.push_back(by[x]);
        hot_lo = int(h->old_of_new.size());
        for (int32_t x = 0; x < nq; ++x)
            if (acc(by[x]) && hot[by[x]]) h->old_of_new.push_back(by[x]);
        h->n_accept = int(h->old_of_new.size());
        for (int32_t x = 0; x < nq; ++x)
            if (!acc(by[x]) && hot[by[x]]) h->old_of_new.push_back(by[x]);
        for (int32_t x = 0; x < nq; ++x)
            if (!acc(by[x]) && !hot[by[x]]) h->old_of_new.push_back(by[x]);
    } else {
        for (int s = 0; s < nq; ++s)
            if (out_off[s + 1] > out_off[s]) h->old_of_new.push_back(s);
        h->n_accept = int(h->old_of_new.size());
        for (int s = 0; s < nq; ++s)
            if (out_off[s + 1] == out_off[s]) h->old_of_new.push_back(s);
    }
    for (int i = 0; i < nq; ++i) h->new_of_old[h->old_of_new[i]] = i;
    h->start_internal = h->new_of_old[0];

    h->acc_out_off.assign(1, 0);
    h->acc_out_ids.clear();
    h->acc_outcnt.clear();
    h->max_outcnt = 0;
    for (int i = 0; i < h->n_accept; ++i) {
        int old = h->old_of_new[i];
        for (int32_t k = out_off[old]; k < out_off[old + 1]; ++k) h->acc_out_ids.push_back(out_ids[k]);
        h->acc_out_off.push_back(int32_t(h->acc_out_ids.size()));
        int cnt = out_off[old + 1] - out_off[old];
        h->acc_outcnt.push_back(uint16_t(std::min(cnt, 65535)));
        h->max_outcnt = std::max(h->max_outcnt, cnt);
        if (cnt > 65535) return fail(KS_E_UNSUPPORTED, "dfa: more than 65535 outputs on one state");
    }

    CompiledTable& t = h->scan;
    t.nq = nq;
    t.n_accept = h->n_accept;
    if (wide) {
        // wide automata: 32-bit ids, definite only (every build_dfa automaton
        // is), scanned one base at a time from the hot table / L2
        if (force_strategy != 0 && force_strategy != KS_STRATEGY_LOOKBACK)
            return fail(KS_E_UNSUPPORTED, "dfa: automata above 32767 states scan with the LOOKBACK strategy only");
        h->wide = true;
        t.stride = 1;
        t.t1w.resize(size_t(nq) * 5);
        for (int s = 0; s < nq; ++s)
            for (int c = 0; c < 5; ++c)
                t.t1w[size_t(h->new_of_old[s]) * 5 + c] = uint32_t(h->new_of_old[trans[size_t(s) * 5 + c]]);
        const uint32_t r = t.t1w[4];
        bool resets = true;
        for (int s = 1; s < nq && resets; ++s) resets = t.t1w[size_t(s) * 5 + 4] == r;
        t.reset_state = resets ? int(r) : -1;
        if (resets && hot_n > 0) {   // hot table (4 columns: OTHER resets, not stored)
            t.hot_lo = hot_lo;
            t.hot_n = hot_n;
            t.ht.assign(size_t(hot_n) * 4, 0xFFFFu);
            for (int i = 0; i < hot_n; ++i)
                for (int c = 0; c < 4; ++c) {
                    const uint32_t x = t.t1w[size_t(hot_lo + i) * 5 + c];
                    if (x - uint32_t(hot_lo) < uint32_t(hot_n)) t.ht[size_t(i) * 4 + c] = uint16_t(x - hot_lo);
                }
        }
        h->sync_depth = synchronisation_depth(t.t1w, nq);
        if (h->sync_depth < 0)
            return fail(KS_E_UNSUPPORTED, "dfa: automata above 32767 states must be definite "
                                          "(synchronise within 2048 symbols)");
        h->strategy = KS_STRATEGY_LOOKBACK;
        return KS_OK;
    }
    t.t1.resize(size_t(nq) * 5);
    for (int s = 0; s < nq; ++s)
        for (int c = 0; c < 5; ++c)
            t.t1[size_t(h->new_of_old[s]) * 5 + c] = uint16_t(h->new_of_old[trans[size_t(s) * 5 + c]]);
    const size_t hist_bytes = size_t(h->n_accept) * 4;
    const size_t budget = smem_budget > hist_bytes + 4096 ? smem_budget - hist_bytes - 4096 : 0;
    build_stride_table(&t, budget);
    if (!(std::getenv("KS_NO_CLS") && *std::getenv("KS_NO_CLS") == '1'))
        build_class_table(&t, h->acc_out_off, h->acc_out_ids);

    h->sync_depth = synchronisation_depth(t.t1, nq);
    bool want_lookback = h->sync_depth >= 0 && force_strategy != KS_STRATEGY_MAPSCAN &&
                         force_strategy != KS_STRATEGY_SPECULATE;
    if (force_strategy == KS_STRATEGY_LOOKBACK && h->sync_depth < 0)
        return fail(KS_E_INVALID, "dfa: LOOKBACK forced but the automaton is not definite");
    if (want_lookback) {
        h->strategy = KS_STRATEGY_LOOKBACK;
        return KS_OK;
    }
    if (force_strategy != KS_STRATEGY_SPECULATE &&
        build_monoid(t, h->start_internal, t.reset_state >= 0 && !(std::getenv("KS_MONO_FULL") && *std::getenv("KS_MONO_FULL") == '1'), h)) {
        build_stride_table(&h->mono, smem_budget > 4096 ? smem_budget - 4096 : 0);
        h->strategy = KS_STRATEGY_MAPSCAN;
        return KS_OK;
    }
    if (force_strategy == KS_STRATEGY_MAPSCAN)
        return fail(KS_E_INVALID, "dfa: MAPSCAN forced but the transition monoid exceeds 4096 maps");
    // SPECULATE: candidate entry states per preceding symbol (the image of its
    // column, engine.py:80-91) and their inverse index
    h->strategy = KS_STRATEGY_SPECULATE;
    h->pss_off.assign(6, 0);
    h->pss.clear();
    h->pss_inv.assign(size_t(5) * nq, int16_t(-1));
    h->pss_max = 0;
    std::vector<char> seen(nq);
    for (int x = 0; x < 5; ++x) {
        std::fill(seen.begin(), seen.end(), 0);
        for (int q = 0; q < nq; ++q) seen[t.t1[size_t(q) * 5 + x]] = 1;
        int k = 0;
        for (int q = 0; q < nq; ++q)
            if (seen[q]) {
                h->pss_inv[size_t(x) * nq + q] = int16_t(k++);
                h->pss.push_back(uint16_t(q));
            }
        h->pss_off[x + 1] = int32_t(h->pss.size());
        h->pss_max = std::max(h->pss_max, k);
    }
    return KS_OK;
}

}  // namespace ks
