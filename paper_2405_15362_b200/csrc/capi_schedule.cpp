// C-ABI for the schedule front end (include/pipeblock_b200.h, "schedules").
#include <cstring>
#include <string>

#include "capi_common.hpp"
#include "schedule/vsched.hpp"

using namespace vsched;

struct pb_schedule {
    Grid grid;
    Document doc;  // what emit() writes (carries source block / steps when built here)
};

namespace pbx {
thread_local std::string g_err;
}

extern "C" const char* pb_last_error(void) { return pbx::g_err.c_str(); }
extern "C" int pb_abi_version(void) { return PB_ABI_VERSION; }

namespace {

Topology topo_from_c(const pb_topology* t) {
    if (!t || t->devices < 1 || t->num_stages < 1 || !t->placement) throw std::invalid_argument("bad topology");
    Topology o;
    o.devices = t->devices;
    o.num_stages = t->num_stages;
    for (int s = 0; s < t->num_stages; ++s) {
        if (t->placement[s] < 1 || t->placement[s] > t->devices)
            throw std::invalid_argument("placement device out of range");
        o.placement.push_back(t->placement[s]);
        o.stage_mem.push_back(t->stage_mem ? t->stage_mem[s] : 1.0);
    }
    o.routes = {Topology::iota(1, o.num_stages)};
    return o;
}

pb_schedule* finish(Grid g, Document d) {
    auto probs = validate_schedule(g);
    if (!probs.empty()) throw std::invalid_argument(probs.front());
    auto* s = new pb_schedule;
    s->grid = std::move(g);
    s->doc = std::move(d);
    return s;
}

}  // namespace

extern "C" int pb_build_info(const char* entry, int32_t devices, int32_t* mpb, int32_t* replicated) {
    return pbx::guard([&] {
        if (!entry) throw std::invalid_argument("null argument");
        Build b = build_entry(entry, devices);
        if (mpb) *mpb = b.block.mb_per_block;
        if (replicated) *replicated = b.replicated_weights ? 1 : 0;
    });
}

extern "C" int pb_schedule_build(const char* entry, int32_t devices, int32_t microbatches, int32_t sq, int32_t re,
                                 pb_schedule** out) {
    return pbx::guard([&] {
        if (!entry || !out) throw std::invalid_argument("null argument");
        Build b = build_entry(entry, devices);
        Grid g = assemble(b, microbatches, sq != 0, re != 0);
        Document d = document_for_assembly(b, g, sq != 0, re != 0);
        *out = finish(std::move(g), std::move(d));
    });
}

extern "C" int pb_schedule_create(const pb_topology* topo, const pb_pass* passes, size_t n, int32_t microbatches,
                                  pb_schedule** out) {
    return pbx::guard([&] {
        if (!out || (n && !passes)) throw std::invalid_argument("null argument");
        Grid g;
        g.topo = topo_from_c(topo);
        g.microbatches = microbatches;
        for (size_t i = 0; i < n; ++i) {
            const pb_pass& p = passes[i];
            if (p.kind < 0 || p.kind > 3) throw std::invalid_argument("kind must be 0..3");
            if (p.stage < 1 || p.stage > g.topo.num_stages) throw std::invalid_argument("stage out of range");
            if (p.microbatch < 0 || p.microbatch >= microbatches) throw std::invalid_argument("microbatch out of range");
            g.ops.push_back({p.device, p.stage, Kind(p.kind), p.microbatch, p.start, p.duration});
        }
        sort_canonical(g);
        Document d;
        d.topo = g.topo;
        d.microbatches = microbatches;
        d.grid = g;
        *out = finish(std::move(g), std::move(d));
    });
}

extern "C" int pb_schedule_parse(const char* text, int32_t strict, pb_schedule** out) {
    return pbx::guard([&] {
        if (!text || !out) throw std::invalid_argument("null argument");
        Document d = parse_document(text, strict != 0);
        if (!d.is_grid()) throw std::invalid_argument("executor needs a 'cells' document, got units 'time'");
        Grid g = d.grid;
        sort_canonical(g);
        *out = finish(std::move(g), std::move(d));
    });
}

extern "C" int pb_schedule_emit(const pb_schedule* s, char* buf, size_t cap, size_t* len) {
    return pbx::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        std::string t = emit_document(s->doc);
        if (len) *len = t.size();
        if (!buf) return;
        if (cap < t.size() + 1) throw pbx::Space("emit buffer too small");
        std::memcpy(buf, t.c_str(), t.size() + 1);
    });
}

extern "C" int pb_schedule_info(const pb_schedule* s, int32_t* devices, int32_t* stages, int32_t* mbs, size_t* n) {
    return pbx::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        if (devices) *devices = s->grid.topo.devices;
        if (stages) *stages = s->grid.topo.num_stages;
        if (mbs) *mbs = s->grid.microbatches;
        if (n) *n = s->grid.ops.size();
    });
}

extern "C" int pb_schedule_topology(const pb_schedule* s, int32_t* placement, double* stage_mem) {
    return pbx::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        for (int i = 0; i < s->grid.topo.num_stages; ++i) {
            if (placement) placement[i] = s->grid.topo.placement[i];
            if (stage_mem) stage_mem[i] = s->grid.topo.stage_mem[i];
        }
    });
}

extern "C" int pb_schedule_passes(const pb_schedule* s, pb_pass* out, size_t n) {
    return pbx::guard([&] {
        if (!s || !out) throw std::invalid_argument("null argument");
        if (n < s->grid.ops.size()) throw pbx::Space("pass buffer too small");
        for (size_t i = 0; i < s->grid.ops.size(); ++i) {
            const auto& o = s->grid.ops[i];
            out[i] = {o.device, o.stage, int32_t(o.kind), o.mb, o.start, o.dur};
        }
    });
}

extern "C" int pb_schedule_exact_peak(const pb_schedule* s, double* per_device) {
    return pbx::guard([&] {
        if (!s || !per_device) throw std::invalid_argument("null argument");
        auto p = exact_peak(s->grid);
        std::memcpy(per_device, p.data(), p.size() * sizeof(double));
    });
}

static void fill_stats(const SimResult& r, pb_timed_pass* out, size_t n, pb_sim_stats* st, double* busy, double* idle_t,
                       double* idle_s, double* peak) {
    if (out) {
        if (n < r.schedule.ops.size()) throw pbx::Space("timed buffer too small");
        for (size_t i = 0; i < r.schedule.ops.size(); ++i) {
            const auto& o = r.schedule.ops[i];
            out[i] = {o.device, o.stage, int32_t(o.kind), o.mb, o.start, o.dur};
        }
    }
    if (st) *st = {r.makespan, r.bubble_rate};
    for (size_t k = 0; k < r.busy.size(); ++k) {
        if (busy) busy[k] = r.busy[k];
        if (idle_t) idle_t[k] = r.idle_total[k];
        if (idle_s) idle_s[k] = r.idle_span[k];
        if (peak) peak[k] = r.peak[k];
    }
}

extern "C" int pb_simulate(const pb_schedule* s, const pb_profile* prof, pb_timed_pass* out, size_t n,
                           pb_sim_stats* st, double* busy, double* idle_t, double* idle_s, double* peak) {
    return pbx::guard([&] {
        if (!s || !prof) throw std::invalid_argument("null argument");
        SimResult r = simulate(s->grid, Profile{prof->f, prof->b, prof->w, prof->comm});
        fill_stats(r, out, n, st, busy, idle_t, idle_s, peak);
    });
}

extern "C" int pb_replay(const pb_schedule* s, const double* durations, size_t n, double comm, pb_timed_pass* out,
                         pb_sim_stats* st, double* busy, double* idle_t, double* idle_s, double* peak) {
    return pbx::guard([&] {
        if (!s || (n && !durations)) throw std::invalid_argument("null argument");
        SimResult r = replay(s->grid, std::vector<double>(durations, durations + n), comm);
        fill_stats(r, out, out ? n : 0, st, busy, idle_t, idle_s, peak);
    });
}

extern "C" int pb_account(const pb_topology* topo, const pb_timed_pass* passes, size_t n, pb_sim_stats* st,
                          double* busy, double* peak) {
    return pbx::guard([&] {
        Timed t;
        t.topo = topo_from_c(topo);
        for (size_t i = 0; i < n; ++i) {
            const auto& p = passes[i];
            if (p.device < 1 || p.device > t.topo.devices) throw std::invalid_argument("device out of range");
            t.ops.push_back({p.device, p.stage, Kind(p.kind & 3), p.microbatch, p.start, p.duration});
        }
        SimResult r = account(t);
        fill_stats(r, nullptr, 0, st, busy, nullptr, nullptr, peak);
    });
}

extern "C" void pb_schedule_destroy(pb_schedule* s) { delete s; }

// schedule access for the executor (same library)
namespace pbx {
const Grid& schedule_grid(const pb_schedule* s) { return s->grid; }
}  // namespace pbx

// ============================================================ analysis
namespace {

void put_text(const std::string& t, char* buf, size_t cap, size_t* len) {
    if (len) *len = t.size();
    if (!buf) return;
    if (cap < t.size() + 1) throw pbx::Space("text buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
}

Profile profile_from_c(const pb_profile* p) {
    if (!p) throw std::invalid_argument("null profile");
    return Profile{p->f, p->b, p->w, p->comm};
}

const Block& block_of(const pb_schedule* s) {
    if (!s) throw std::invalid_argument("null schedule");
    if (!s->doc.block) throw std::invalid_argument("schedule carries no building block (made from passes)");
    return *s->doc.block;
}

SearchSpec spec_from_c(const pb_search_spec* c) {
    if (!c) throw std::invalid_argument("null search spec");
    SearchSpec s;
    s.d = c->devices;
    s.n = c->microbatches;
    s.profile = profile_from_c(&c->profile);
    s.memory_limit = c->memory_limit;
    s.delta_max = c->delta_max;
    s.tau_max = c->tau_max;
    return s;
}

pb_search_params params_to_c(const SearchParams& p) {
    return {p.K, p.d0_lo, p.d1_lo, p.d0_hi, p.d1_hi, p.tau1, p.tau2, p.tau3};
}

Timed timed_from_c(const pb_topology* topo, const pb_timed_pass* passes, size_t n, int32_t microbatches) {
    if (n && !passes) throw std::invalid_argument("null passes");
    Timed t;
    t.topo = topo_from_c(topo);
    t.microbatches = microbatches;
    for (size_t i = 0; i < n; ++i) {
        const auto& p = passes[i];
        if (p.device < 1 || p.device > t.topo.devices) throw std::invalid_argument("device out of range");
        if (p.kind < 0 || p.kind > 3) throw std::invalid_argument("kind must be 0..3");
        t.ops.push_back({p.device, p.stage, Kind(p.kind), p.microbatch, p.start, p.duration});
    }
    return t;
}

}  // namespace

extern "C" int pb_growth_rate(const pb_schedule* s, const pb_profile* prof, pb_growth_report* out, double* work,
                              char* witness, size_t cap, size_t* len) {
    return pbx::guard([&] {
        Growth g = growth_rate(block_of(s), profile_from_c(prof));
        if (out) *out = {g.cycle_length, g.growth, g.max_work, g.repeating_bubble, int32_t(g.linear_bubble), int32_t(g.tie)};
        if (work) std::memcpy(work, g.work_per_period.data(), g.work_per_period.size() * sizeof(double));
        std::string w;
        for (const auto& x : g.witness) w += x + "\n";
        put_text(w, witness, cap, len);
    });
}

extern "C" int pb_growth_rate_unrolled(const pb_schedule* s, const pb_profile* prof, int32_t periods, double* out) {
    return pbx::guard([&] {
        if (!out || periods < 1) throw std::invalid_argument("bad argument");
        *out = growth_rate_unrolled(block_of(s), profile_from_c(prof), periods);
    });
}

extern "C" int pb_vhalf_condition(const pb_profile* prof, int32_t* out) {
    return pbx::guard([&] {
        if (!out) throw std::invalid_argument("null argument");
        *out = vhalf_condition(profile_from_c(prof));
    });
}

extern "C" int pb_lower_bound(int64_t n, int64_t d, int64_t k, int64_t* out) {
    return pbx::guard([&] {
        if (!out) throw std::invalid_argument("null argument");
        *out = makespan_lower_bound(n, d, k);
    });
}

extern "C" int pb_min_memory_for_od_bubble(int32_t d, double* out) {
    return pbx::guard([&] {
        if (!out) throw std::invalid_argument("null argument");
        *out = min_memory_for_od_bubble(d);
    });
}

extern "C" int pb_search_assemble(int32_t devices, const pb_search_params* p, int32_t microbatches, pb_schedule** out) {
    return pbx::guard([&] {
        if (!p || !out) throw std::invalid_argument("null argument");
        SearchParams sp;
        sp.K = p->K;
        sp.d0_lo = p->d0_lo;
        sp.d1_lo = p->d1_lo;
        sp.d0_hi = p->d0_hi;
        sp.d1_hi = p->d1_hi;
        sp.tau1 = p->tau1;
        sp.tau2 = p->tau2;
        sp.tau3 = p->tau3;
        Build b;
        b.name = "search";
        b.block = search_block(devices, sp);
        if (auto v = first_block_violation(b.block)) throw std::invalid_argument("search block: " + *v);
        if (auto c = residue_clash(b.block))
            throw std::invalid_argument("search block: repeat clash on device " + std::to_string(c->first));
        Grid g = assemble(b, microbatches, true, true);
        Document d = document_for_assembly(b, g, true, true);
        *out = finish(std::move(g), std::move(d));
    });
}

extern "C" int pb_search(const pb_search_spec* spec, pb_search_result* out, char* message, size_t cap, size_t* len,
                         pb_schedule** schedule) {
    return pbx::guard([&] {
        if (!out) throw std::invalid_argument("null argument");
        SearchSpec sp = spec_from_c(spec);
        SearchResult r = search(sp);
        *out = {int32_t(r.feasible), params_to_c(r.best), r.bubble_rate, r.exact_peak, r.enumerated, r.evaluated,
                r.family_min_peak, int32_t(r.turn_devices_exercised)};
        put_text(r.message, message, cap, len);
        if (schedule) {
            *schedule = nullptr;
            if (r.feasible) {
                Document d = document_for_assembly(r.build, r.schedule, true, true);
                *schedule = finish(std::move(r.schedule), std::move(d));
            }
        }
    });
}

extern "C" int pb_frontier(const pb_search_spec* spec, const double* limits, size_t n, pb_frontier_point* out) {
    return pbx::guard([&] {
        if (n && (!limits || !out)) throw std::invalid_argument("null argument");
        auto pts = frontier(spec_from_c(spec), std::vector<double>(limits, limits + n));
        for (size_t i = 0; i < pts.size(); ++i)
            out[i] = {pts[i].limit, int32_t(pts[i].feasible), pts[i].bubble_rate, pts[i].exact_peak,
                      params_to_c(pts[i].best)};
    });
}

extern "C" int pb_render(const pb_schedule* s, int32_t format, const char* title, int32_t ascii_max_width,
                         int32_t ascii_color, char* buf, size_t cap, size_t* len) {
    return pbx::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        RenderOptions o;
        if (title) o.title = title;
        if (ascii_max_width > 0) o.ascii_max_width = ascii_max_width;
        o.ascii_color = ascii_color != 0;
        put_text(format == PB_RENDER_ASCII ? render_ascii(s->doc, o) : render_svg(s->doc, o), buf, cap, len);
    });
}

extern "C" int pb_timed_emit(const pb_topology* topo, const pb_timed_pass* passes, size_t n, int32_t microbatches,
                             char* buf, size_t cap, size_t* len) {
    return pbx::guard([&] { put_text(emit_document(document_for_timed(timed_from_c(topo, passes, n, microbatches))), buf, cap, len); });
}

extern "C" int pb_timed_render(const pb_topology* topo, const pb_timed_pass* passes, size_t n, int32_t microbatches,
                               int32_t format, const char* title, int32_t ascii_max_width, char* buf, size_t cap,
                               size_t* len) {
    return pbx::guard([&] {
        Document d = document_for_timed(timed_from_c(topo, passes, n, microbatches));
        RenderOptions o;
        if (title) o.title = title;
        if (ascii_max_width > 0) o.ascii_max_width = ascii_max_width;
        put_text(format == PB_RENDER_ASCII ? render_ascii(d, o) : render_svg(d, o), buf, cap, len);
    });
}
