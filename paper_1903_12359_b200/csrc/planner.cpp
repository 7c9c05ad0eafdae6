// planner.cpp -- host-side weld-schedule planner (partition.py:149-324).
//
// Combinatorial, integer-exact: for every step the reference scans all
// component pairs (O(K^3 L) overall, 82.6 s at K=256). Here the best run of
// every *adjacent* pair (components sharing a boundary vertex) is cached and
// only pairs involving the component that just grew are re-scanned, which
// gives the identical choice (the key (-len, ca, cb, chain[0]) is a total
// order over candidates) in O(K * deg * L).
//
// Output (two-call protocol): per step 8 int64 of meta
//   comp_a, comp_b, k, closed, offset, len_a, len_b, len_merged
// and the concatenated a_cycle | b_cycle | merged_cycle parent ids in idx.
#include <algorithm>
#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "common.cuh"

namespace {

using Cycle = std::vector<int64_t>;
using Runs = std::vector<Cycle>;

// flat scratch indexed by parent vertex id (generation-stamped, no resets)
struct Scratch {
    std::vector<int64_t> pos;     // position in the current c2
    std::vector<uint32_t> gen;    // generation of pos[]
    std::vector<uint32_t> mark;   // generation marks for set tests
    uint32_t g = 0, gm = 0;
    void ensure(int64_t n) {
        if ((int64_t)pos.size() < n) {
            pos.assign(n, 0);
            gen.assign(n, 0);
            mark.assign(n, 0);
        }
    }
};
thread_local Scratch g_scr;

// maximal runs of consecutive c1 vertices that are consecutive reversed in
// c2 (partition.py:149-179); *full when the whole cycle matches
bool cyclic_runs(const Cycle& c1, const Cycle& c2, Runs* runs, bool* full, std::string* err) {
    runs->clear();
    *full = false;
    const size_t n1 = c1.size(), n2 = c2.size();
    Scratch& S = g_scr;
    const uint32_t g = ++S.g;
    for (size_t i = 0; i < n2; ++i) {
        S.pos[c2[i]] = (int64_t)i;
        S.gen[c2[i]] = g;
    }
    std::vector<char> ok(n1, 0);
    bool all = n1 > 0, any = false;
    for (size_t i = 0; i < n1; ++i) {
        int64_t u = c1[i], v = c1[(i + 1) % n1];
        if (S.gen[u] == g && S.gen[v] == g && (S.pos[v] + 1) % (int64_t)n2 == S.pos[u]) ok[i] = 1;
        all = all && ok[i];
        any = any || ok[i];
    }
    if (all) {
        if (n1 != n2) {
            *err = "inconsistent full-cycle correspondence";
            return false;
        }
        *full = true;
        return true;
    }
    if (!any) return true;
    size_t start = 0;
    while (ok[start]) ++start;
    size_t i = start;
    for (size_t t = 0; t < n1; ++t) {
        i = (i + 1) % n1;
        size_t im1 = (i + n1 - 1) % n1;
        if (ok[i] && !ok[im1]) {
            size_t j = i;
            Cycle chain{c1[j]};
            while (ok[j % n1]) {
                chain.push_back(c1[(j + 1) % n1]);
                ++j;
            }
            runs->push_back(std::move(chain));
        }
    }
    return true;
}

Cycle rotate_to(const Cycle& c, int64_t v) {
    auto it = std::find(c.begin(), c.end(), v);
    Cycle out(it, c.end());
    out.insert(out.end(), c.begin(), it);
    return out;
}

struct Step {
    int64_t ca, cb, k, closed;
    Cycle a, b, merged;
};

struct Key {
    int64_t neglen, ca, cb, first;
    bool operator<(const Key& o) const {
        if (neglen != o.neglen) return neglen < o.neglen;
        if (ca != o.ca) return ca < o.ca;
        if (cb != o.cb) return cb < o.cb;
        return first < o.first;
    }
};

struct Planner {
    std::map<int64_t, Cycle> cycles;
    std::vector<Step> steps;
    std::string err;

    int glue(int64_t ca, int64_t cb, const Cycle& chain) {
        Scratch& S = g_scr;
        const uint32_t ga = ++S.gm;   // on a's cycle
        for (int64_t v : cycles[ca]) S.mark[v] = ga;
        const uint32_t gc = ++S.gm;   // on the chain (overrides)
        for (int64_t v : chain) S.mark[v] = gc;
        for (int64_t v : cycles[cb])
            if (S.mark[v] == ga) {
                err = "components " + std::to_string(ca) + " and " + std::to_string(cb) +
                      " share vertices beyond one contiguous arc; this cut layout needs multi-arc gluing, which "
                      "is unsupported";
                return PGCP_E_PARTITION;
            }
        Cycle a = rotate_to(cycles[ca], chain[0]);
        Cycle rb(cycles[cb].rbegin(), cycles[cb].rend());
        Cycle b = rotate_to(rb, chain[0]);
        const int64_t k = (int64_t)chain.size() - 1;
        if (!std::equal(chain.begin(), chain.end(), a.begin()) || !std::equal(chain.begin(), chain.end(), b.begin())) {
            err = "arc is not a prefix of both component cycles";
            return PGCP_E_PARTITION;
        }
        Cycle merged{chain.back()};
        merged.insert(merged.end(), a.begin() + k + 1, a.end());
        merged.push_back(chain.front());
        merged.insert(merged.end(), b.rbegin(), b.rend() - (k + 1));
        steps.push_back({ca, cb, k, 0, a, b, merged});
        cycles.erase(cb);
        cycles[ca] = merged;
        return PGCP_OK;
    }

    int sphere_close() {
        auto it = cycles.begin();
        int64_t ca = it->first, cb = std::next(it)->first;
        const Cycle& c1 = cycles[ca];
        const Cycle& c2 = cycles[cb];
        std::set<int64_t> s1(c1.begin(), c1.end()), s2(c2.begin(), c2.end());
        if (s1 != s2 || c1.size() != c2.size()) {
            err = "final two components do not share their full boundary";
            return PGCP_E_PARTITION;
        }
        Runs runs;
        bool full = false;
        if (!cyclic_runs(c1, c2, &runs, &full, &err)) return PGCP_E_PARTITION;
        if (!full) {
            err = "final boundaries are not a reversed cyclic match";
            return PGCP_E_PARTITION;
        }
        int64_t s = *std::min_element(c1.begin(), c1.end());
        Cycle a = rotate_to(c1, s);
        Cycle rb(c2.rbegin(), c2.rend());
        Cycle b = rotate_to(rb, s);
        steps.push_back({ca, cb, (int64_t)a.size() - 1, 1, a, b, {}});
        return PGCP_OK;
    }

    int check_cover(const int64_t* cuts, int64_t ncuts) {
        // sorted edge lists instead of ordered sets: the glued edges must be
        // distinct and equal to the cut set
        std::vector<std::pair<int64_t, int64_t>> glued;
        for (const Step& st : steps) {
            for (int64_t i = 0; i < st.k; ++i)
                glued.push_back({std::min(st.a[i], st.a[i + 1]), std::max(st.a[i], st.a[i + 1])});
            if (st.closed) glued.push_back({std::min(st.a[st.k], st.a[0]), std::max(st.a[st.k], st.a[0])});
        }
        std::vector<std::pair<int64_t, int64_t>> order = glued;
        std::sort(order.begin(), order.end());
        for (size_t i = 1; i < order.size(); ++i)
            if (order[i] == order[i - 1]) {
                // report the first duplicate in schedule order, as the set-based check would
                std::set<std::pair<int64_t, int64_t>> seen;
                for (auto& e : glued)
                    if (!seen.insert(e).second) {
                        err = "edge (" + std::to_string(e.first) + ", " + std::to_string(e.second) +
                              ") glued twice in the schedule";
                        return PGCP_E_PARTITION;
                    }
            }
        std::vector<std::pair<int64_t, int64_t>> want((size_t)ncuts);
        for (int64_t i = 0; i < ncuts; ++i) want[i] = {cuts[2 * i], cuts[2 * i + 1]};
        std::sort(want.begin(), want.end());
        want.erase(std::unique(want.begin(), want.end()), want.end());
        if (order != want) {
            size_t missing = 0;
            for (auto& e : want) missing += std::binary_search(order.begin(), order.end(), e) ? 0 : 1;
            err = "schedule does not cover all cut edges (" + std::to_string(missing) + " missing)";
            return PGCP_E_PARTITION;
        }
        return PGCP_OK;
    }

    // best candidate of one pair (ca < cb); returns false if none
    bool pair_best(int64_t ca, int64_t cb, Key* key, Cycle* chain, int* st) {
        Runs runs;
        bool full = false;
        if (!cyclic_runs(cycles[ca], cycles[cb], &runs, &full, &err)) {
            *st = PGCP_E_PARTITION;
            return false;
        }
        if (full || runs.empty()) return false;
        bool have = false;
        for (auto& ch : runs) {
            Key k{-(int64_t)ch.size(), ca, cb, ch[0]};
            if (!have || k < *key) {
                *key = k;
                *chain = ch;
                have = true;
            }
        }
        return have;
    }

    int greedy(int target) {
        // vertex -> components containing it
        std::unordered_map<int64_t, std::set<int64_t>> owner;
        for (auto& kv : cycles)
            for (int64_t v : kv.second) owner[v].insert(kv.first);
        std::map<std::pair<int64_t, int64_t>, std::pair<Key, Cycle>> cand;
        auto rescan = [&](int64_t c) -> int {
            std::set<int64_t> nb;
            for (int64_t v : cycles[c])
                for (int64_t o : owner[v])
                    if (o != c) nb.insert(o);
            for (int64_t o : nb) {
                int64_t a = std::min(c, o), b = std::max(c, o);
                Key k;
                Cycle ch;
                int st = PGCP_OK;
                if (pair_best(a, b, &k, &ch, &st))
                    cand[{a, b}] = {k, ch};
                else
                    cand.erase({a, b});
                if (st != PGCP_OK) return st;
            }
            return PGCP_OK;
        };
        for (auto& kv : cycles) {
            int st = rescan(kv.first);
            if (st != PGCP_OK) return st;
        }
        while ((int)cycles.size() > target) {
            if (cand.empty()) {
                err = "no contiguous shared arc between any two components; multi-arc gluing in one step is "
                      "unsupported";
                return PGCP_E_PARTITION;
            }
            auto best = cand.begin();
            for (auto it = cand.begin(); it != cand.end(); ++it)
                if (it->second.first < best->second.first) best = it;
            int64_t ca = best->first.first, cb = best->first.second;
            Cycle chain = best->second.second;
            // update ownership: cb's vertices now belong to ca
            for (int64_t v : cycles[cb]) {
                owner[v].erase(cb);
                owner[v].insert(ca);
            }
            int st = glue(ca, cb, chain);
            if (st != PGCP_OK) return st;
            for (auto it = cand.begin(); it != cand.end();) {
                if (it->first.first == cb || it->first.second == cb || it->first.first == ca ||
                    it->first.second == ca)
                    it = cand.erase(it);
                else
                    ++it;
            }
            std::unordered_set<int64_t> onca(cycles[ca].begin(), cycles[ca].end());
            for (int64_t v : chain)
                if (!onca.count(v)) owner[v].erase(ca);
            st = rescan(ca);
            if (st != PGCP_OK) return st;
        }
        return PGCP_OK;
    }
};

}  // namespace

namespace {
// the two-call protocol (sizes, then copy-out) must not plan twice: keep the
// last plan of this thread keyed by a checksum of its inputs
struct PlanCache {
    uint64_t key = 0;
    bool valid = false;
    std::vector<Step> steps;
};
thread_local PlanCache g_cache;

uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}
}  // namespace

extern "C" PGCP_API int pgcp_plan_weld_schedule(const int64_t* cyc, const int64_t* cyc_off, int32_t K,
                                                const int64_t* cuts, int64_t ncuts, int mode_sphere,
                                                const int32_t* pairs, int32_t npairs, int64_t* out_meta,
                                                int64_t* out_idx, int64_t out_cap, int64_t* out_len) {
    if (K < 0 || !cyc_off || !out_len) {
        pgcp::set_error("plan_weld_schedule: invalid arguments");
        return PGCP_E_INVALID;
    }
    uint64_t key = mix(0, (uint64_t)K);
    key = mix(key, (uint64_t)mode_sphere);
    key = mix(key, (uint64_t)ncuts);
    for (int64_t i = 0; i < cyc_off[K]; ++i) key = mix(key, (uint64_t)cyc[i] * 2654435761ull + (uint64_t)i);
    for (int64_t i = 0; i < 2 * ncuts; ++i) key = mix(key, (uint64_t)cuts[i]);
    key = mix(key, (uint64_t)(pairs ? npairs : -1));
    for (int32_t i = 0; pairs && i < 2 * npairs; ++i) key = mix(key, (uint64_t)pairs[i]);

    if (!(g_cache.valid && g_cache.key == key)) {
        int64_t vmax = 0;
        for (int64_t i = 0; i < cyc_off[K]; ++i) vmax = std::max(vmax, cyc[i]);
        for (int64_t i = 0; i < 2 * ncuts; ++i) vmax = std::max(vmax, cuts[i]);
        g_scr.ensure(vmax + 1);
        Planner P;
        for (int32_t i = 0; i < K; ++i) P.cycles[i] = Cycle(cyc + cyc_off[i], cyc + cyc_off[i + 1]);
        int target = mode_sphere ? 2 : 1;
        if (mode_sphere && K < 2) {
            pgcp::set_error("sphere mode needs at least 2 submeshes");
            return PGCP_E_PARTITION;
        }
        int st = PGCP_OK;
        if (pairs && npairs > 0) {
            for (int32_t q = 0; q < npairs && st == PGCP_OK; ++q) {
                int64_t ca = std::min(pairs[2 * q], pairs[2 * q + 1]), cb = std::max(pairs[2 * q], pairs[2 * q + 1]);
                if (!P.cycles.count(ca) || !P.cycles.count(cb)) {
                    P.err = "pair (" + std::to_string(ca) + ", " + std::to_string(cb) + ") is not two live components";
                    st = PGCP_E_PARTITION;
                    break;
                }
                Key k;
                Cycle ch;
                if (!P.pair_best(ca, cb, &k, &ch, &st)) {
                    if (st == PGCP_OK) {
                        P.err = "components " + std::to_string(ca) + " and " + std::to_string(cb) +
                                " share no open arc";
                        st = PGCP_E_PARTITION;
                    }
                    break;
                }
                st = P.glue(ca, cb, ch);
            }
            if (st == PGCP_OK && (int)P.cycles.size() != target) {
                P.err = "merge order leaves more than the target components";
                st = PGCP_E_PARTITION;
            }
        } else {
            st = P.greedy(target);
        }
        if (st == PGCP_OK && mode_sphere) st = P.sphere_close();
        if (st == PGCP_OK) st = P.check_cover(cuts, ncuts);
        if (st != PGCP_OK) {
            g_cache.valid = false;
            pgcp::set_error("%s", P.err.c_str());
            return st;
        }
        g_cache.steps = std::move(P.steps);
        g_cache.key = key;
        g_cache.valid = true;
    }
    const std::vector<Step>& steps = g_cache.steps;
    int64_t need = 0;
    for (auto& s : steps) need += (int64_t)(s.a.size() + s.b.size() + s.merged.size());
    out_len[0] = (int64_t)steps.size();
    out_len[1] = need;
    if (!out_meta || !out_idx || out_cap < need) return PGCP_OK;
    int64_t off = 0;
    for (size_t i = 0; i < steps.size(); ++i) {
        const Step& s = steps[i];
        int64_t* m = out_meta + 8 * i;
        m[0] = s.ca;
        m[1] = s.cb;
        m[2] = s.k;
        m[3] = s.closed;
        m[4] = off;
        m[5] = (int64_t)s.a.size();
        m[6] = (int64_t)s.b.size();
        m[7] = (int64_t)s.merged.size();
        for (int64_t v : s.a) out_idx[off++] = v;
        for (int64_t v : s.b) out_idx[off++] = v;
        for (int64_t v : s.merged) out_idx[off++] = v;
    }
    g_cache.valid = false;  // copy-out done: no memoisation across plans
    return PGCP_OK;
}

// ---------------------------------------------------------------------------
// Weld plan over tracked boundary slots (the bookkeeping of pipeline.py:
// 172-213 on per-component dicts, flattened): slot s = one entry of one
// submesh's boundary loop (submesh order, loop order). For every step the
// slots of a_cycle / b_cycle (phase-1 inputs; a parent vertex present in
// several loops of a component resolves to its last slot) and the
// write-back code of every slot of the two components:
//   bits 0..23 arc position + 1 (0: replay), bit 25 / 26 on a_cycle / b_cycle,
//   bit 31 slot of the b side.
// Inputs: cycles (parent ids, cyc_off[K+1]) and the planner's flat output
// (meta[8*nsteps], idx). Outputs (two-call protocol, lens[0] = total src
// entries, lens[1] = total write-back entries):
//   info[6*nsteps] (k, closed, na, nb, comp_a, comp_b), src, wb_off[nsteps+1],
//   wb[2*total] (slot, code), ext[K] = 1 / 2 for the submeshes on the a / b
//   side of the closing (sphere) step, else 0.
extern "C" PGCP_API int pgcp_weld_plan(const int64_t* cyc, const int64_t* cyc_off, int32_t K, const int64_t* meta,
                                       const int64_t* idx, int32_t nsteps, int64_t n_parent, int32_t* info,
                                       int32_t* src, int64_t* wb_off, int32_t* wb, int32_t* ext, int64_t* lens) {
    if (K < 0 || nsteps < 0 || !cyc_off || !lens || (nsteps > 0 && (!meta || !idx))) {
        pgcp::set_error("weld_plan: invalid arguments");
        return PGCP_E_INVALID;
    }
    // members of every live component (submesh lists, in merge order)
    std::vector<std::vector<int32_t>> members(K);
    for (int32_t i = 0; i < K; ++i) members[i] = {i};
    int64_t nsrc = 0, nwb = 0;
    for (int32_t q = 0; q < nsteps; ++q) {
        const int64_t* m = meta + 8 * (int64_t)q;
        nsrc += m[5] + m[6];
        int64_t ca = m[0], cb = m[1];
        if (ca < 0 || ca >= K || cb < 0 || cb >= K) {
            pgcp::set_error("weld_plan: component id out of range");
            return PGCP_E_INVALID;
        }
        for (int32_t sub : members[ca]) nwb += cyc_off[sub + 1] - cyc_off[sub];
        for (int32_t sub : members[cb]) nwb += cyc_off[sub + 1] - cyc_off[sub];
        members[ca].insert(members[ca].end(), members[cb].begin(), members[cb].end());
        members[cb].clear();
    }
    lens[0] = nsrc;
    lens[1] = nwb;
    if (!info || !src || !wb_off || !wb) return PGCP_OK;
    for (int32_t i = 0; i < K; ++i) members[i] = {i};
    if (ext)
        for (int32_t i = 0; i < K; ++i) ext[i] = 0;
    // persistent per-thread scratch over parent ids (restored after every use)
    thread_local std::vector<int32_t> table, code;
    if ((int64_t)table.size() < std::max<int64_t>(n_parent, 1)) {
        table.assign((size_t)std::max<int64_t>(n_parent, 1), -1);
        code.assign((size_t)std::max<int64_t>(n_parent, 1), 0);
    }
    const int32_t CYC_A = 1 << 25, CYC_B = 1 << 26;
    const uint32_t SIDE_B = 1u << 31;
    int64_t so = 0, wo = 0;
    wb_off[0] = 0;
    for (int32_t q = 0; q < nsteps; ++q) {
        const int64_t* m = meta + 8 * (int64_t)q;
        const int64_t ca = m[0], cb = m[1], k = m[2], closed = m[3], o = m[4], na = m[5], nb = m[6];
        const int64_t* ac = idx + o;
        const int64_t* bc = ac + na;
        auto slots_src = [&](const std::vector<int32_t>& mem, const int64_t* cy, int64_t len) -> int {
            for (int32_t sub : mem)
                for (int64_t t = cyc_off[sub]; t < cyc_off[sub + 1]; ++t) table[cyc[t]] = (int32_t)t;
            int bad = 0;
            for (int64_t i = 0; i < len; ++i) {
                int64_t v = cy[i];
                int32_t sl = (v >= 0 && v < n_parent) ? table[v] : -1;
                if (sl < 0) bad = 1;
                src[so++] = sl;
            }
            for (int32_t sub : mem)
                for (int64_t t = cyc_off[sub]; t < cyc_off[sub + 1]; ++t) table[cyc[t]] = -1;
            return bad;
        };
        if (slots_src(members[ca], ac, na) | slots_src(members[cb], bc, nb)) {
            pgcp::set_error("weld step references a boundary vertex outside its components");
            return PGCP_E_WELD;
        }
        for (int64_t i = 0; i <= k && i < na; ++i) code[ac[i]] = (int32_t)(i + 1);
        for (int64_t i = 0; i < na; ++i) code[ac[i]] |= CYC_A;
        for (int64_t i = 0; i < nb; ++i) code[bc[i]] |= CYC_B;
        for (int32_t sub : members[ca])
            for (int64_t t = cyc_off[sub]; t < cyc_off[sub + 1]; ++t) {
                wb[2 * wo] = (int32_t)t;
                wb[2 * wo + 1] = code[cyc[t]];
                ++wo;
            }
        for (int32_t sub : members[cb])
            for (int64_t t = cyc_off[sub]; t < cyc_off[sub + 1]; ++t) {
                wb[2 * wo] = (int32_t)t;
                wb[2 * wo + 1] = (int32_t)((uint32_t)code[cyc[t]] | SIDE_B);
                ++wo;
            }
        for (int64_t i = 0; i < na; ++i) code[ac[i]] = 0;
        for (int64_t i = 0; i < nb; ++i) code[bc[i]] = 0;
        wb_off[q + 1] = wo;
        int32_t* in = info + 6 * (int64_t)q;
        in[0] = (int32_t)k;
        in[1] = (int32_t)closed;
        in[2] = (int32_t)na;
        in[3] = (int32_t)nb;
        in[4] = (int32_t)ca;
        in[5] = (int32_t)cb;
        if (closed && ext) {
            for (int32_t sub : members[ca]) ext[sub] = 1;
            for (int32_t sub : members[cb]) ext[sub] = 2;
        }
        members[ca].insert(members[ca].end(), members[cb].begin(), members[cb].end());
        members[cb].clear();
    }
    return PGCP_OK;
}
