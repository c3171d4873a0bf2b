// Test infrastructure (oracle side): a tiny command-line driver over the UNMODIFIED
// reference library (/root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/). It replaces the reference's own `fdsolve` (tools/fdsolve.cpp:42-143),
// which cannot be built here because CLI11 is absent, and prints one JSON object.
//
// It is never part of the product path: only tests/, bench.py's cpu_baseline /
// --impl reference legs and golden-fixture generation run it.
//
//   fdref_driver solve <model.fd> [--max N|--all] [--input] [--fc] [--node-limit N]
//                [--threads T] [--solutions] [--repeat R] [--solutions-bin PATH]
//     --solutions-bin: every solution's values, in callback (DFS) order, as little-endian int64
//     rows into PATH (the golden sha256 of the full solution stream is taken over this file)
//   fdref_driver fixpoint <model.fd> [--fc]
//   fdref_driver gen-nqueens N
//   fdref_driver gen-random VARS WIDTH CONS SEED
//   fdref_driver corpus SEED          (acceptance.cpp:47-54 corpus_instance text)
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>

#include "fd/generators.hpp"
#include "fd/parser.hpp"
#include "fd/propagation.hpp"
#include "fd/rng.hpp"
#include "fd/search.hpp"

namespace {

std::string slurp(const char* path) {
    std::ifstream in(path);
    if (!in) {
        std::fprintf(stderr, "cannot open %s\n", path);
        std::exit(2);
    }
    std::stringstream b;
    b << in.rdbuf();
    return b.str();
}

fd::Model must_parse(const std::string& text) {
    fd::ParseResult r = fd::parse_model(text);
    if (const auto* e = std::get_if<fd::ParseError>(&r)) {
        std::fprintf(stderr, "parse error: %s\n", e->message().c_str());
        std::exit(2);
    }
    return std::get<fd::Model>(std::move(r));
}

void print_values(std::ostream& os, const std::vector<std::int64_t>& v) {
    os << "[";
    for (std::size_t i = 0; i < v.size(); ++i)
        os << (i ? "," : "") << v[i];
    os << "]";
}

int cmd_solve(int argc, char** argv) {
    fd::Model m = must_parse(slurp(argv[2]));
    fd::SearchConfig cfg;
    bool print_all = false;
    int repeat = 1;
    const char* bin_path = nullptr;
    for (int i = 3; i < argc; ++i) {
        std::string a = argv[i];
        if (a == "--max") cfg.max_solutions = std::stoull(argv[++i]);
        else if (a == "--all") cfg.max_solutions = std::numeric_limits<std::uint64_t>::max();
        else if (a == "--input") cfg.var_heuristic = fd::VarHeuristic::InputOrder;
        else if (a == "--fc") cfg.alldiff = fd::AlldiffLevel::ForwardChecking;
        else if (a == "--node-limit") cfg.node_limit = std::stoull(argv[++i]);
        else if (a == "--threads") cfg.thread_count = std::stoi(argv[++i]);
        else if (a == "--solutions") print_all = true;
        else if (a == "--repeat") repeat = std::stoi(argv[++i]);
        else if (a == "--solutions-bin") bin_path = argv[++i];
        else { std::fprintf(stderr, "unknown flag %s\n", a.c_str()); return 2; }
    }
    bool optimizing = !std::holds_alternative<fd::Satisfy>(m.goal);
    std::ostringstream os;
    double best_ms = 1e300;
    for (int r = 0; r < repeat; ++r) {
        os.str("");
        auto t0 = std::chrono::steady_clock::now();
        try {
            if (optimizing) {
                fd::OptimizeResult res = fd::solve_optimize(m, cfg);
                auto t1 = std::chrono::steady_clock::now();
                best_ms = std::min(best_ms, std::chrono::duration<double, std::milli>(t1 - t0).count());
                os << "{\"status\":\"" << (res.best ? (res.complete ? "OPTIMAL" : "SAT")
                                                     : (res.complete ? "UNSAT" : "UNKNOWN"))
                   << "\",\"nodes\":" << res.stats.nodes << ",\"failures\":" << res.stats.failures
                   << ",\"rounds\":" << res.stats.rounds << ",\"solutions\":" << res.stats.solutions
                   << ",\"complete\":" << (res.complete ? "true" : "false");
                if (res.best) {
                    os << ",\"objective\":" << *res.best->objective << ",\"best\":";
                    print_values(os, res.best->values);
                }
            } else {
                std::vector<std::vector<std::int64_t>> sols;
                std::uint64_t count = 0;
                std::vector<std::int64_t> first;
                std::FILE* bin = bin_path ? std::fopen(bin_path, "wb") : nullptr;
                if (bin_path && !bin) { std::fprintf(stderr, "cannot write %s\n", bin_path); std::exit(2); }
                fd::SatisfyResult res = fd::solve_satisfy(m, cfg, [&](const fd::Solution& s) {
                    if (count == 0) first = s.values;
                    ++count;
                    if (print_all) sols.push_back(s.values);
                    if (bin) std::fwrite(s.values.data(), sizeof(std::int64_t), s.values.size(), bin);
                    return true;
                });
                if (bin) std::fclose(bin);
                auto t1 = std::chrono::steady_clock::now();
                best_ms = std::min(best_ms, std::chrono::duration<double, std::milli>(t1 - t0).count());
                os << "{\"status\":\"" << (count ? "SAT" : (res.complete ? "UNSAT" : "UNKNOWN"))
                   << "\",\"nodes\":" << res.stats.nodes << ",\"failures\":" << res.stats.failures
                   << ",\"rounds\":" << res.stats.rounds << ",\"solutions\":" << res.stats.solutions
                   << ",\"complete\":" << (res.complete ? "true" : "false");
                if (count) {
                    os << ",\"first\":";
                    print_values(os, first);
                }
                if (print_all) {
                    os << ",\"all\":[";
                    for (std::size_t i = 0; i < sols.size(); ++i) {
                        if (i) os << ",";
                        print_values(os, sols[i]);
                    }
                    os << "]";
                }
            }
        } catch (const fd::ArithmeticOverflowError& e) {
            os.str("");
            os << "{\"status\":\"ERROR\",\"error\":\"overflow\"";
        }
    }
    os << ",\"time_ms\":" << best_ms << "}";
    std::cout << os.str() << "\n";
    return 0;
}

int cmd_fixpoint(int argc, char** argv) {
    fd::Model m = must_parse(slurp(argv[2]));
    fd::PropagationConfig pc;
    for (int i = 3; i < argc; ++i)
        if (std::string(argv[i]) == "--fc") pc.alldiff = fd::AlldiffLevel::ForwardChecking;
    std::vector<fd::Domain> doms = m.domains;
    auto batches = fd::group_batches(m.constraints);
    std::ostringstream os;
    try {
        fd::FixpointResult fx = fd::propagate_fixpoint(doms, m.constraints, batches, pc);
        os << "{\"failed\":" << (fx.failed ? "true" : "false") << ",\"failed_var\":" << fx.failed_var
           << ",\"rounds\":" << fx.rounds << ",\"domains\":[";
        for (std::size_t v = 0; v < doms.size(); ++v) {
            if (v) os << ",";
            print_values(os, doms[v].values());
        }
        os << "]}";
    } catch (const fd::ArithmeticOverflowError&) {
        os.str("");
        os << "{\"error\":\"overflow\"}";
    }
    std::cout << os.str() << "\n";
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: fdref_driver solve|fixpoint|gen-nqueens|gen-random|corpus ...\n");
        return 2;
    }
    std::string cmd = argv[1];
    if (cmd == "solve") return cmd_solve(argc, argv);
    if (cmd == "fixpoint") return cmd_fixpoint(argc, argv);
    if (cmd == "gen-nqueens") { std::cout << fd::gen_nqueens(std::atoi(argv[2])); return 0; }
    if (cmd == "gen-random" && argc >= 6) {
        std::cout << fd::gen_random(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]),
                                    std::stoull(argv[5]));
        return 0;
    }
    if (cmd == "corpus") {
        // acceptance.cpp:47-54 (corpus_instance) restated to emit the text.
        std::uint64_t seed = std::stoull(argv[2]);
        fd::Rng rng(seed * 7919 + 13);
        int vars = static_cast<int>(rng.below(5)) + 2;
        int width = static_cast<int>(rng.below(9)) + 2;
        int constraints = static_cast<int>(rng.below(8)) + 1;
        std::cout << fd::gen_random(vars, width, constraints, seed);
        return 0;
    }
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
}
