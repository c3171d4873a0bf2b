// Drop-in replacement of the reference's hot-path translation units.
//
// The reference library (/root/reference/proj) is built from src/{domain,model,parser,state,
// generators,report,propagation,search}.cpp. This file replaces the last two: it implements
// every function declared in proj/include/fd/search.hpp and proj/include/fd/propagation.hpp on
// top of the C ABI of libcubics.so (include/cubics.h), so existing callers (fdsolve,
// bench_propagation, the reference tests) link unchanged and run on the B200 engine.
// It is compiled against the reference's own headers where they lie; see INTEGRATION.md.
//
// Reference interfaces implemented here (paths relative to proj/):
//   fd::solve_satisfy / enumerate_solutions / solve_optimize      include/fd/search.hpp:62-77
//   fd::select_variable / select_value                              include/fd/search.hpp:46-51
//   fd::lns_optimize (host orchestration over GPU B&B searches)     include/fd/search.hpp:92
//   fd::propagate_fixpoint / propagate_round / run_batch            include/fd/propagation.hpp:88-118
//   fd::prop_* / propagate_one / group_batches / RemovalSet         include/fd/propagation.hpp:28-83
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cubics.h"
#include "fd/propagation.hpp"
#include "fd/rng.hpp"
#include "fd/search.hpp"

namespace {

[[noreturn]] void raise(int rc) {
    const char* msg = cubics_last_error();
    std::string m = msg ? msg : "";
    if (rc == CUBICS_E_OVERFLOW) throw fd::ArithmeticOverflowError(m.empty() ? "overflow in linear propagation" : m);
    if (rc == CUBICS_E_NO_OBJECTIVE) throw std::logic_error(m);
    throw std::runtime_error("cubics engine error " + std::to_string(rc) + ": " + m);
}

void check(int rc) {
    if (rc != CUBICS_OK) raise(rc);
}

// Flat copy of an fd::Model (or of a domain vector + constraint list) for cubics_model_create.
struct Flat {
    std::vector<int64_t> off;
    std::vector<int32_t> width;
    std::vector<uint64_t> words;
    std::vector<int32_t> kind, op, start{0}, tvar;
    std::vector<int64_t> value, tcoeff;
    int32_t goal = CUBICS_SATISFY, goal_var = 0;

    void add_domains(const std::vector<fd::Domain>& ds) {
        for (const fd::Domain& d : ds) {
            off.push_back(d.offset());
            width.push_back(d.width());
            auto w = d.words();
            words.insert(words.end(), w.begin(), w.end());
        }
    }

    void add_constraints(const std::vector<fd::Constraint>& cs) {
        for (const fd::Constraint& c : cs) {
            if (const auto* rb = std::get_if<fd::RelBin>(&c)) {
                kind.push_back(CUBICS_RELBIN);
                op.push_back(static_cast<int32_t>(rb->op));
                value.push_back(rb->rhs_value);
                tvar.push_back(rb->lhs);
                tcoeff.push_back(1);
                if (rb->rhs_is_var) {
                    tvar.push_back(rb->rhs_var);
                    tcoeff.push_back(1);
                }
            } else if (const auto* lin = std::get_if<fd::Linear>(&c)) {
                kind.push_back(CUBICS_LINEAR);
                op.push_back(static_cast<int32_t>(lin->op));
                value.push_back(lin->bound);
                for (const fd::LinTerm& t : lin->terms) {
                    tvar.push_back(t.var);
                    tcoeff.push_back(t.coeff);
                }
            } else {
                kind.push_back(CUBICS_ALLDIFF);
                op.push_back(0);
                value.push_back(0);
                for (fd::VarId v : std::get<fd::AllDifferent>(c).vars) {
                    tvar.push_back(v);
                    tcoeff.push_back(1);
                }
            }
            start.push_back(static_cast<int32_t>(tvar.size()));
        }
    }

    cubics_model* build() const {
        cubics_model_desc d{};
        d.n_vars = static_cast<int32_t>(off.size());
        d.var_offset = off.data();
        d.var_width = width.data();
        d.var_words = words.data();
        d.n_cons = static_cast<int32_t>(kind.size());
        d.con_kind = kind.data();
        d.con_op = op.data();
        d.con_value = value.data();
        d.con_start = start.data();
        d.term_var = tvar.data();
        d.term_coeff = tcoeff.data();
        d.goal = goal;
        d.goal_var = goal_var;
        cubics_model* m = nullptr;
        check(cubics_model_create(&d, &m));
        return m;
    }
};

struct ModelHandle {
    cubics_model* m;
    explicit ModelHandle(cubics_model* p) : m(p) {}
    ~ModelHandle() { cubics_model_free(m); }
    ModelHandle(const ModelHandle&) = delete;
    ModelHandle& operator=(const ModelHandle&) = delete;
};

struct GoalInfo {
    bool optimizing = false, minimizing = false;
    fd::VarId var = 0;
};

GoalInfo goal_of(const fd::Model& m) {
    if (const auto* mn = std::get_if<fd::Minimize>(&m.goal)) return {true, true, mn->var};
    if (const auto* mx = std::get_if<fd::Maximize>(&m.goal)) return {true, false, mx->var};
    return {};
}

cubics_model* model_of(const fd::Model& m) {
    Flat f;
    f.add_domains(m.domains);
    f.add_constraints(m.constraints);
    GoalInfo g = goal_of(m);
    if (g.optimizing) {
        f.goal = g.minimizing ? CUBICS_MINIMIZE : CUBICS_MAXIMIZE;
        f.goal_var = g.var;
    }
    return f.build();
}

cubics_search_config config_of(const fd::SearchConfig& c) {
    cubics_search_config k;
    cubics_search_config_init(&k);
    k.var_heuristic = c.var_heuristic == fd::VarHeuristic::FirstFail ? CUBICS_FIRST_FAIL : CUBICS_INPUT_ORDER;
    k.max_solutions = c.max_solutions;
    k.thread_count = c.thread_count;
    k.seed = c.seed;
    k.alldiff = c.alldiff == fd::AlldiffLevel::ArcConsistent ? CUBICS_ARC_CONSISTENT : CUBICS_FORWARD_CHECKING;
    k.node_limit = c.node_limit;
    return k;
}

fd::SearchStats stats_of(const cubics_result& r) {
    fd::SearchStats s;
    s.nodes = r.stats.nodes;
    s.failures = r.stats.failures;
    s.rounds = r.stats.rounds;
    s.solutions = r.stats.solutions;
    return s;
}

struct CbCtx {
    const fd::SolutionCallback* cb;
    GoalInfo goal;
};

int32_t trampoline(void* user, const int64_t* values, int32_t n) {
    auto* c = static_cast<CbCtx*>(user);
    fd::Solution sol;
    sol.values.assign(values, values + n);
    if (c->goal.optimizing) sol.objective = sol.values[static_cast<size_t>(c->goal.var)];
    return (*c->cb)(sol) ? 1 : 0;
}

// domain vector <-> u64 words in the desc packing
std::vector<uint64_t> words_of(const std::vector<fd::Domain>& ds) {
    std::vector<uint64_t> w;
    for (const fd::Domain& d : ds) {
        auto x = d.words();
        w.insert(w.end(), x.begin(), x.end());
    }
    if (w.empty()) w.push_back(0);
    return w;
}

// Create the CUDA context and load the kernels when the program starts, as the reference's
// library has no first-call latency to speak of (acceptance.cpp:70-81 bounds the first
// fixpoint at 1 s, context creation included).
struct Warmup {
    Warmup() {
        if (cubics_device_count() > 0) cubics_warmup(-1);
    }
} g_warmup;

} // namespace

namespace fd {

// ---------------------------------------------------------------- search.hpp
VarId select_variable(const std::vector<Domain>& domains, VarHeuristic h) {
    VarId pick = -1;
    for (VarId v = 0; v < static_cast<VarId>(domains.size()); ++v) {
        int sz = domains[static_cast<size_t>(v)].size();
        if (sz < 2) continue;
        if (h == VarHeuristic::InputOrder) return v;
        if (pick < 0 || sz < domains[static_cast<size_t>(pick)].size()) pick = v;
    }
    return pick;
}

std::int64_t select_value(const Domain& d) { return d.min(); }

namespace {
// CUBICS_DEVICES="0,1,..." (two or more): complete enumerations, first solutions and optimizations
// run on all of those GPUs from this process (cubics_solve_multi). With several GPUs a callback
// still sees every solution in the reference's DFS order, but a callback that stops early gets the
// complete search's stats.
std::vector<int32_t> multi_devices() {
    std::vector<int32_t> d;
    const char* e = std::getenv("CUBICS_DEVICES");
    for (const char* p = e; p && *p;) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) break;
        d.push_back(static_cast<int32_t>(v));
        p = *end ? end + 1 : end;
    }
    return d.size() > 1 ? d : std::vector<int32_t>{};
}

bool multi_ok(const cubics_search_config& k, bool optimizing) {
    return k.node_limit == 0 && (optimizing || k.max_solutions == 1 || k.max_solutions == UINT64_MAX);
}
} // namespace

SatisfyResult solve_satisfy(const Model& m, const SearchConfig& cfg, const SolutionCallback& cb) {
    ModelHandle h(model_of(m));
    cubics_search_config k = config_of(cfg);
    CbCtx ctx{&cb, goal_of(m)};
    cubics_result r{};
    const std::vector<int32_t> devs = multi_devices();
    if (!devs.empty() && !goal_of(m).optimizing && multi_ok(k, false))
        check(cubics_solve_multi(h.m, &k, static_cast<int32_t>(devs.size()), devs.data(), cb ? trampoline : nullptr, &ctx,
                                 nullptr, &r));
    else
        check(cubics_solve_satisfy(h.m, &k, cb ? trampoline : nullptr, &ctx, &r));
    SatisfyResult out;
    out.stats = stats_of(r);
    out.complete = r.complete != 0;
    return out;
}

std::vector<Solution> enumerate_solutions(const Model& m, const SearchConfig& cfg, SearchStats* stats) {
    if (!multi_devices().empty() && !goal_of(m).optimizing && multi_ok(config_of(cfg), false)) {
        std::vector<Solution> out; // several GPUs: the merged stream of cubics_solve_multi
        const SatisfyResult r = solve_satisfy(m, cfg, [&](const Solution& s) {
            out.push_back(s);
            return true;
        });
        if (stats) *stats = r.stats;
        return out;
    }
    ModelHandle h(model_of(m));
    cubics_search_config k = config_of(cfg);
    cubics_solutions* sols = nullptr;
    cubics_result r{};
    check(cubics_enumerate(h.m, &k, &sols, &r));
    std::vector<Solution> out(sols->count);
    const GoalInfo g = goal_of(m);
    for (uint64_t i = 0; i < sols->count; ++i) {
        out[i].values.assign(sols->values + i * sols->n_vars, sols->values + (i + 1) * sols->n_vars);
        if (g.optimizing) out[i].objective = out[i].values[static_cast<size_t>(g.var)];
    }
    cubics_solutions_free(sols);
    if (stats) *stats = stats_of(r);
    return out;
}

namespace {
OptimizeResult optimize_with(const Model& m, cubics_search_config k) {
    ModelHandle h(model_of(m));
    std::vector<int64_t> best(static_cast<size_t>(std::max(1, m.num_vars())));
    cubics_result r{};
    const std::vector<int32_t> devs = multi_devices();
    if (!devs.empty() && multi_ok(k, true) && k.max_solutions == UINT64_MAX)
        check(cubics_solve_multi(h.m, &k, static_cast<int32_t>(devs.size()), devs.data(), nullptr, nullptr, best.data(), &r));
    else
        check(cubics_solve_optimize(h.m, &k, best.data(), &r));
    OptimizeResult out;
    out.complete = r.complete != 0;
    out.stats = stats_of(r);
    if (r.has_solution) {
        Solution s;
        s.values.assign(best.begin(), best.begin() + m.num_vars());
        s.objective = r.objective;
        out.best = s;
    }
    return out;
}
} // namespace

OptimizeResult solve_optimize(const Model& m, const SearchConfig& cfg) {
    return optimize_with(m, config_of(cfg)); // no objective -> std::logic_error via the ABI
}

// Large neighbourhood search (search.cpp:225-314): the host orchestrates; the first-solution
// search runs on the device and all neighbourhoods of an iteration run as ONE batched launch
// (cubics_solve_optimize_batch, one thread block per neighbourhood, each in reference order). Semantics follow the reference: Rng::derive per
// (seed, neighbourhood, iteration), partial Fisher-Yates destroy set, incumbent frozen for the
// iteration, deterministic lowest-index merge.
LnsResult lns_optimize(const Model& m, const LnsConfig& cfg) {
    const GoalInfo goal = goal_of(m);
    if (!goal.optimizing) throw std::logic_error("lns_optimize requires a minimize or maximize goal");
    LnsResult res;
    SearchConfig first_cfg;
    first_cfg.max_solutions = 1;
    first_cfg.thread_count = cfg.thread_count;
    first_cfg.alldiff = cfg.alldiff;
    std::optional<Solution> best;
    SatisfyResult first = solve_satisfy(m, first_cfg, [&](const Solution& s) {
        best = s;
        return false;
    });
    res.stats = first.stats;
    res.initial_complete = first.complete || best.has_value();
    if (!best) return res;
    const int n = m.num_vars();
    const int destroy = std::min(n, std::max(1, static_cast<int>(std::ceil(cfg.destroy_rate * n))));
    auto better = [&](std::int64_t a, std::int64_t b) { return goal.minimizing ? a < b : a > b; };
    // every neighbourhood of an iteration is one problem of ONE batched device launch
    ModelHandle h(model_of(m));
    size_t nw = 0;
    std::vector<size_t> wstart(static_cast<size_t>(n) + 1, 0);
    for (int v = 0; v < n; ++v) wstart[v + 1] = wstart[v] + static_cast<size_t>(m.domains[v].word_count());
    nw = wstart[n];
    std::vector<std::uint64_t> base(nw);
    for (int v = 0; v < n; ++v) {
        const auto& w = m.domains[v].words();
        std::copy(w.begin(), w.end(), base.begin() + wstart[v]);
    }
    cubics_search_config k;
    cubics_search_config_init(&k);
    k.alldiff = cfg.alldiff == AlldiffLevel::ArcConsistent ? CUBICS_ARC_CONSISTENT : CUBICS_FORWARD_CHECKING;
    k.node_limit = cfg.per_iteration_node_limit;
    k.engine = CUBICS_ENGINE_PARITY;
    const int nbs = std::max(0, cfg.neighborhoods);
    for (int iter = 0; iter < cfg.iterations; ++iter) {
        const Solution incumbent = *best;
        std::vector<std::optional<Solution>> found(static_cast<size_t>(nbs));
        std::vector<std::uint64_t> words(nw * nbs);
        for (int nb = 0; nb < nbs; ++nb) {
            Rng rng = Rng::derive(cfg.seed, static_cast<std::uint64_t>(nb), static_cast<std::uint64_t>(iter));
            std::vector<char> destroyed(static_cast<size_t>(n), 0);
            std::vector<int> ids(static_cast<size_t>(n));
            for (int i = 0; i < n; ++i) ids[static_cast<size_t>(i)] = i;
            for (int i = 0; i < destroy && n > 0; ++i) {
                int j = i + static_cast<int>(rng.below(static_cast<std::uint64_t>(n - i)));
                std::swap(ids[static_cast<size_t>(i)], ids[static_cast<size_t>(j)]);
                destroyed[static_cast<size_t>(ids[static_cast<size_t>(i)])] = 1;
            }
            std::uint64_t* wd = words.data() + nw * nb;
            std::copy(base.begin(), base.end(), wd);
            for (int v = 0; v < n; ++v)
                if (!destroyed[static_cast<size_t>(v)]) { // neighborhood_model: Domain(val, val)
                    const std::int64_t bit = incumbent.values[static_cast<size_t>(v)] - m.domains[v].offset();
                    std::fill(wd + wstart[v], wd + wstart[v + 1], 0);
                    wd[wstart[v] + bit / 64] = std::uint64_t{1} << (bit % 64);
                }
        }
        std::vector<std::int64_t> bounds(static_cast<size_t>(nbs), *incumbent.objective);
        std::vector<std::int64_t> vals(static_cast<size_t>(nbs) * std::max(1, n));
        std::vector<cubics_result> rs(static_cast<size_t>(nbs));
        if (nbs)
            check(cubics_solve_optimize_batch(h.m, &k, nbs, words.data(), bounds.data(), nullptr, vals.data(), rs.data()));
        for (int nb = 0; nb < nbs; ++nb) {
            const cubics_result& r = rs[static_cast<size_t>(nb)];
            if (r.has_solution) {
                Solution s;
                s.values.assign(vals.begin() + static_cast<size_t>(nb) * n, vals.begin() + static_cast<size_t>(nb + 1) * n);
                s.objective = r.objective;
                found[static_cast<size_t>(nb)] = s;
            }
            res.stats.nodes += r.stats.nodes;
            res.stats.failures += r.stats.failures;
            res.stats.rounds += r.stats.rounds;
        }
        for (int nb = 0; nb < nbs; ++nb) {
            const auto& cand = found[static_cast<size_t>(nb)];
            if (cand && better(*cand->objective, *best->objective)) best = cand;
        }
        res.trajectory.push_back(*best->objective);
    }
    res.best = best;
    return res;
}

// ---------------------------------------------------------------- propagation.hpp
bool RemovalSet::empty() const {
    return std::all_of(entries_.begin(), entries_.end(),
                       [](const Entry& e) { return std::all_of(e.mask.begin(), e.mask.end(), [](std::uint64_t w) { return w == 0; }); });
}

std::vector<std::uint64_t>& RemovalSet::mask_for(VarId var, const Domain& dom) {
    auto it = std::find_if(entries_.begin(), entries_.end(), [&](const Entry& e) { return e.var == var; });
    if (it != entries_.end()) return it->mask;
    entries_.push_back(Entry{var, std::vector<std::uint64_t>(static_cast<size_t>(dom.word_count()), 0)});
    return entries_.back().mask;
}

void RemovalSet::add_value(VarId var, const Domain& dom, std::int64_t v) {
    if (!dom.contains(v)) return;
    const std::int64_t bit = v - dom.offset();
    mask_for(var, dom)[static_cast<size_t>(bit / 64)] |= std::uint64_t{1} << (bit % 64);
}

void RemovalSet::add_range(VarId var, const Domain& dom, std::int64_t lo, std::int64_t hi) {
    if (dom.empty()) return;
    for (std::int64_t v = std::max(lo, dom.min()), e = std::min(hi, dom.max()); v <= e; ++v) add_value(var, dom, v);
}

void RemovalSet::add_all(VarId var, const Domain& dom) {
    if (!dom.empty()) add_range(var, dom, dom.min(), dom.max());
}

void RemovalSet::merge_from(const RemovalSet& other) {
    for (const Entry& oe : other.entries_) {
        auto it = std::find_if(entries_.begin(), entries_.end(), [&](const Entry& e) { return e.var == oe.var; });
        if (it == entries_.end()) {
            entries_.push_back(oe);
            continue;
        }
        if (it->mask.size() < oe.mask.size()) it->mask.resize(oe.mask.size(), 0);
        for (size_t i = 0; i < oe.mask.size(); ++i) it->mask[i] |= oe.mask[i];
    }
}

std::vector<std::int64_t> RemovalSet::removed_values(VarId var, const Domain& dom) const {
    std::vector<std::int64_t> out;
    for (const Entry& e : entries_) {
        if (e.var != var) continue;
        for (size_t w = 0; w < e.mask.size(); ++w)
            for (int b = 0; b < 64; ++b)
                if ((e.mask[w] >> b) & 1) {
                    std::int64_t v = dom.offset() + static_cast<std::int64_t>(w) * 64 + b;
                    if (dom.contains(v)) out.push_back(v);
                }
    }
    std::sort(out.begin(), out.end());
    return out;
}

std::vector<PropagatorBatch> group_batches(const std::vector<Constraint>& constraints) {
    std::vector<PropagatorBatch> out;
    for (int i = 0; i < static_cast<int>(constraints.size()); ++i) {
        ConstraintKind k = constraint_kind(constraints[static_cast<size_t>(i)]);
        auto it = std::find_if(out.begin(), out.end(), [&](const PropagatorBatch& b) { return b.kind == k; });
        if (it == out.end()) {
            out.push_back(PropagatorBatch{k, {}});
            it = out.end() - 1;
        }
        it->members.push_back(i);
    }
    return out;
}

namespace {
// Device removals of constraints `members` of `cs` against the domains of the snapshot.
RemovalSet device_removals(const std::vector<Constraint>& cs, const std::vector<int>& members, const DomainSnapshot& s,
                           AlldiffLevel level) {
    std::vector<Domain> doms;
    doms.reserve(static_cast<size_t>(s.num_vars()));
    for (VarId v = 0; v < s.num_vars(); ++v) doms.push_back(s[v]);
    Flat f;
    f.add_domains(doms);
    f.add_constraints(cs);
    ModelHandle h(f.build());
    std::vector<uint64_t> w = words_of(doms), removed(w.size(), 0);
    check(cubics_removals(h.m, w.data(), level == AlldiffLevel::ArcConsistent ? CUBICS_ARC_CONSISTENT : CUBICS_FORWARD_CHECKING,
                          members.data(), static_cast<int32_t>(members.size()), removed.data()));
    RemovalSet out;
    size_t at = 0;
    for (VarId v = 0; v < s.num_vars(); ++v) {
        const Domain& d = s[v];
        for (int i = 0; i < d.word_count(); ++i, ++at)
            for (int b = 0; b < 64; ++b)
                if ((removed[at] >> b) & 1) out.add_value(v, d, d.offset() + static_cast<std::int64_t>(i) * 64 + b);
    }
    return out;
}

RemovalSet one(const Constraint& c, const DomainSnapshot& s, AlldiffLevel level) {
    return device_removals(std::vector<Constraint>{c}, std::vector<int>{0}, s, level);
}
} // namespace

RemovalSet prop_rel_bin(const RelBin& c, const DomainSnapshot& s) { return one(c, s, AlldiffLevel::ArcConsistent); }
RemovalSet prop_linear(const Linear& c, const DomainSnapshot& s) { return one(c, s, AlldiffLevel::ArcConsistent); }
RemovalSet prop_alldiff_fc(const AllDifferent& c, const DomainSnapshot& s) {
    return one(c, s, AlldiffLevel::ForwardChecking);
}
RemovalSet prop_alldiff_gac(const AllDifferent& c, const DomainSnapshot& s) {
    return one(c, s, AlldiffLevel::ArcConsistent);
}
RemovalSet propagate_one(const Constraint& c, const DomainSnapshot& s, AlldiffLevel level) { return one(c, s, level); }

RemovalSet run_batch(const std::vector<Constraint>& constraints, const PropagatorBatch& batch, const DomainSnapshot& s,
                     const PropagationConfig& cfg) {
    return device_removals(constraints, batch.members, s, cfg.alldiff);
}

namespace {
// Device rounds over `domains`; the hook (which cannot cross the ABI) is replayed per round on
// the host before the round's changes are written back, as the reference fires it (:501-503).
FixpointResult device_rounds(std::vector<Domain>& domains, const std::vector<Constraint>& constraints,
                             const PropagationConfig& cfg, const ModifyHook& hook, int max_rounds) {
    Flat f;
    f.add_domains(domains);
    f.add_constraints(constraints);
    ModelHandle h(f.build());
    const int32_t level = cfg.alldiff == AlldiffLevel::ArcConsistent ? CUBICS_ARC_CONSISTENT : CUBICS_FORWARD_CHECKING;
    FixpointResult res;
    const int step = hook ? 1 : max_rounds;
    for (;;) {
        std::vector<uint64_t> w = words_of(domains);
        cubics_fixpoint_result fr{};
        check(cubics_propagate(h.m, w.data(), level, step, &fr));
        size_t at = 0;
        for (size_t v = 0; v < domains.size(); ++v) {
            Domain& d = domains[v];
            auto old = d.words();
            std::vector<std::uint64_t> gone(old.size());
            bool changed = false;
            for (size_t i = 0; i < old.size(); ++i) {
                gone[i] = old[i] & ~w[at + i];
                changed |= gone[i] != 0;
            }
            at += old.size();
            if (!changed) continue;
            if (hook) hook(static_cast<VarId>(v));
            d.remove_mask(gone);
        }
        res.rounds += fr.rounds;
        if (fr.failed) {
            res.failed = true;
            res.failed_var = fr.failed_var;
            return res;
        }
        if (fr.last_status == 1 || (max_rounds > 0 && res.rounds >= max_rounds)) return res;
    }
}
} // namespace

RoundResult propagate_round(std::vector<Domain>& domains, const std::vector<Constraint>& constraints,
                            const std::vector<PropagatorBatch>& batches, const PropagationConfig& cfg,
                            const ModifyHook& on_before_modify) {
    (void)batches; // the union of all batches is order-free (propagation.hpp:85-87)
    std::vector<uint64_t> before = words_of(domains);
    FixpointResult fx = device_rounds(domains, constraints, cfg, on_before_modify, 1);
    RoundResult r;
    if (fx.failed) {
        r.status = RoundResult::Status::Failed;
        r.failed_var = fx.failed_var;
    } else {
        r.status = words_of(domains) == before ? RoundResult::Status::Stable : RoundResult::Status::Changed;
    }
    return r;
}

FixpointResult propagate_fixpoint(std::vector<Domain>& domains, const std::vector<Constraint>& constraints,
                                  const std::vector<PropagatorBatch>& batches, const PropagationConfig& cfg,
                                  const ModifyHook& on_before_modify) {
    (void)batches;
    return device_rounds(domains, constraints, cfg, on_before_modify, 0);
}

} // namespace fd
