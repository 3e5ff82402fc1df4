// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference headers, compiled in place
// from /root/reference/proj/include (recipe: oracle/Makefile, output only into
// oracle/_ref/).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load the resulting library.
//
// Entry points mirror the reference call stack CS-1..CS-4:
//   build_entry (gallery.hpp:499) -> assemble (assemble.hpp:405)
//   exact_peak (memory.hpp:63), simulate (simulate.hpp:22)
//   document_from_grid + emit (document.hpp:188,403)
// plus the analysis side through one JSON request/response call:
//   growth_rate (growth.hpp:141), search/frontier (search.hpp:235,240),
//   render_svg/render_ascii (render.hpp:83,177) of grid and simulated-time documents
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>

#include "pipeblock/assemble.hpp"
#include "pipeblock/document.hpp"
#include "pipeblock/gallery.hpp"
#include "pipeblock/growth.hpp"
#include "pipeblock/render.hpp"
#include "pipeblock/search.hpp"
#include "pipeblock/memory.hpp"
#include "pipeblock/simulate.hpp"

using namespace pipeblock;

namespace {
thread_local std::string g_err;
struct RefPass {
    int32_t device, stage, kind, microbatch;
    int64_t start, duration;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// assemble(build_entry(entry, d), n, {sq, re}); writes canonical passes.
int ref_assemble(const char* entry, int d, int n, int sq, int re, RefPass* out, size_t cap, size_t* count) {
    try {
        auto g = assemble(build_entry(entry, d), n, AssembleOptions{sq != 0, re != 0});
        *count = g.passes.size();
        if (!out) return 0;
        if (cap < g.passes.size()) return -4;
        for (size_t i = 0; i < g.passes.size(); ++i) {
            const auto& p = g.passes[i];
            out[i] = {p.device, p.stage, int32_t(p.kind), p.microbatch, p.start, p.duration};
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// exact_peak + simulate(profile) on the assembled schedule.
int ref_analyze(const char* entry, int d, int n, double f, double b, double w, double comm, double* peaks,
                double* makespan, double* bubble) {
    try {
        auto g = assemble(build_entry(entry, d), n);
        auto pk = exact_peak(g);
        for (size_t i = 0; i < pk.per_device.size(); ++i) peaks[i] = pk.per_device[i];
        auto sim = simulate(g, RunTimeProfile{f, b, w, comm});
        *makespan = sim.makespan;
        *bubble = sim.bubble_rate;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The document the reference CLI `assemble` subcommand writes (cli.hpp:146-156).
int ref_emit(const char* entry, int d, int n, char* buf, size_t cap, size_t* len) {
    try {
        auto build = build_entry(entry, d);
        auto g = assemble(build, n);
        ScheduleDocument doc = document_from_grid(g);
        doc.metadata.source_block = build.entry;
        doc.metadata.steps = {"repeat", "squeeze", "reorder"};
        doc.metadata.replicated_weights = build.replicated_weights;
        doc.block = build.block;
        std::string t = emit(doc);
        *len = t.size();
        if (!buf) return 0;
        if (cap < t.size() + 1) return -4;
        std::memcpy(buf, t.c_str(), t.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Reference parse() round trip: returns emit(parse(text)) or the DocumentError text.
int ref_reemit(const char* text, int strict, char* buf, size_t cap, size_t* len) {
    std::string t;
    int rc = 0;
    try {
        t = emit(parse(text, strict != 0));
    } catch (const std::exception& e) {
        t = e.what();
        rc = -2;
    }
    *len = t.size();
    if (buf && cap >= t.size() + 1) std::memcpy(buf, t.c_str(), t.size() + 1);
    return rc;
}

// Reference CPU path timed: build_entry + repeat + squeeze +
// reorder + simulate + exact_peak, `iters` times; returns seconds per pass of
// the whole chain (steady_clock, single thread).
double ref_time_pipeline(const char* entry, int d, int n, int iters, double f, double b, double w) {
    auto t0 = std::chrono::steady_clock::now();
    double sink = 0;
    for (int i = 0; i < iters; ++i) {
        auto g = assemble(build_entry(entry, d), n);
        auto sim = simulate(g, RunTimeProfile{f, b, w, 0.0});
        sink += sim.makespan + exact_peak(g).max;
    }
    auto t1 = std::chrono::steady_clock::now();
    if (sink < 0) return -1;
    return std::chrono::duration<double>(t1 - t0).count() / iters;
}


// ref_analysis(request JSON) -> response JSON (or {"error": what}).
int ref_analysis(const char* request, char* buf, size_t cap, size_t* len) {
    using nlohmann::ordered_json;
    ordered_json out;
    try {
        auto rq = ordered_json::parse(request);
        std::string op = rq.at("op");
        auto prof = [&] {
            auto p = rq.value("profile", std::vector<double>{1, 1, 1, 0});
            return RunTimeProfile{p[0], p[1], p[2], p[3]};
        };
        if (op == "growth") {
            auto blk = build_entry(rq.at("entry").get<std::string>(), rq.at("d").get<int>()).block;
            auto g = growth_rate(blk, prof());
            out = {{"cycle_length", g.cycle_length}, {"growth", g.growth}, {"work", g.work_per_period},
                   {"max_work", g.max_work}, {"repeating_bubble", g.repeating_bubble},
                   {"linear_bubble", g.linear_bubble}, {"tie", g.tie}, {"witness", g.witness},
                   {"unrolled3", growth_rate_unrolled(blk, prof(), 3)}};
        } else if (op == "search" || op == "frontier") {
            SearchSpec sp;
            sp.d = rq.at("d");
            sp.n = rq.value("n", 0);
            sp.profile = prof();
            sp.memory_limit = rq.value("limit", 0.0);
            sp.delta_max = rq.value("delta_max", 6LL);
            sp.tau_max = rq.value("tau_max", 6LL);
            auto P = [](const SearchParams& b) {
                return std::vector<long long>{b.K, b.d0_lo, b.d1_lo, b.d0_hi, b.d1_hi, b.tau1, b.tau2, b.tau3};
            };
            if (op == "search") {
                auto r = search(sp);
                out = {{"feasible", r.feasible}, {"message", r.message}, {"best", P(r.best)}, {"best_str", r.best.str()},
                       {"bubble_rate", r.bubble_rate}, {"exact_peak", r.exact_peak},
                       {"enumerated", r.candidates_enumerated}, {"evaluated", r.candidates_evaluated},
                       {"family_min_peak", r.family_min_peak}, {"turn", r.turn_devices_exercised}};
                if (r.feasible) {
                    std::vector<std::vector<long long>> ps;
                    for (const auto& q : r.schedule.passes)
                        ps.push_back({q.device, q.stage, int(q.kind), q.microbatch, q.start, q.duration});
                    out["passes"] = ps;
                }
            } else {
                auto pts = frontier(sp, rq.at("limits").get<std::vector<double>>());
                out = ordered_json::array();
                for (const auto& q : pts)
                    out.push_back({{"limit", q.limit}, {"feasible", q.feasible}, {"bubble_rate", q.bubble_rate},
                                   {"exact_peak", q.exact_peak}, {"best", P(q.best)}});
            }
        } else if (op == "render") {
            auto build = build_entry(rq.at("entry").get<std::string>(), rq.at("d").get<int>());
            auto g = assemble(build, rq.at("n").get<int>());
            RenderOptions ro;
            ro.ascii_max_width = rq.value("max_width", 200);
            ro.ascii_color = rq.value("color", false);
            ro.title = rq.value("title", std::string());
            ScheduleDocument doc;
            if (rq.value("timed", false)) {
                doc = document_from_timed(simulate(g, prof()).schedule);
                out["emit"] = emit(doc);
            } else {
                doc = document_from_grid(g);
                doc.metadata.source_block = build.entry;
            }
            out["svg"] = render_svg(doc, ro);
            out["ascii"] = render_ascii(doc, ro);
        } else {
            throw std::invalid_argument("unknown op " + op);
        }
    } catch (const std::exception& e) {
        out = {{"error", e.what()}};
    }
    std::string t = out.dump();
    *len = t.size();
    if (buf && cap >= t.size() + 1) std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
}

}  // extern "C"
