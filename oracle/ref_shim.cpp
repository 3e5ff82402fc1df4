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
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>

#include "pipeblock/assemble.hpp"
#include "pipeblock/document.hpp"
#include "pipeblock/gallery.hpp"
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

}  // extern "C"
