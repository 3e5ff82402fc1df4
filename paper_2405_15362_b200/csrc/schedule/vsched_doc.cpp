// ScheduleDocument (format_version 1) reader/writer — the on-disk boundary of
// the reference (/root/reference/proj/include/pipeblock/document.hpp:21-421).
// Emission is byte-identical to the reference (same nlohmann ordered_json
// dump(2) + "\n"), so schedule files produced by the reference CLI run here
// unchanged and files written here load in the reference.
#include <algorithm>

#include "json.hpp"
#include "vsched.hpp"

namespace vsched {

using ojson = nlohmann::ordered_json;

namespace {

const char* type_of(const ojson& j) {
    switch (j.type()) {
        case ojson::value_t::array: return "array";
        case ojson::value_t::object: return "object";
        case ojson::value_t::string: return "string";
        case ojson::value_t::boolean: return "boolean";
        case ojson::value_t::null: return "null";
        default: return j.is_number() ? "number" : "value";
    }
}

// JSON-pointer-ish cursor so errors name the offending path (document.hpp:79-118)
struct At {
    const ojson* j;
    std::string path;
    [[noreturn]] void fail(const std::string& msg) const {
        throw DocumentError(path.empty() ? msg : path + ": " + msg);
    }
    At key(const std::string& k) const {
        auto it = j->find(k);
        if (it == j->end()) fail("missing field '" + k + "'");
        return {&*it, path + "/" + k};
    }
    std::optional<At> opt(const std::string& k) const {
        auto it = j->find(k);
        if (it == j->end()) return std::nullopt;
        return At{&*it, path + "/" + k};
    }
    At idx(size_t i) const { return {&(*j)[i], path + "/" + std::to_string(i)}; }
    const At& object() const {
        if (!j->is_object()) fail(std::string("expected object, got ") + type_of(*j));
        return *this;
    }
    const At& array() const {
        if (!j->is_array()) fail(std::string("expected array, got ") + type_of(*j));
        return *this;
    }
    int64_t integer(const char* what = "integer") const {
        if (j->is_number_integer()) return j->get<int64_t>();
        if (j->is_number_float()) {
            double v = j->get<double>();
            if (v == static_cast<double>(static_cast<int64_t>(v))) return static_cast<int64_t>(v);
        }
        fail(std::string("expected ") + what + ", got " + type_of(*j));
    }
    double number() const {
        if (!j->is_number()) fail(std::string("expected number, got ") + type_of(*j));
        return j->get<double>();
    }
    std::string str() const {
        if (!j->is_string()) fail(std::string("expected string, got ") + type_of(*j));
        return j->get<std::string>();
    }
    size_t size() const { return j->size(); }
};

void known_fields(const At& c, std::initializer_list<const char*> known, bool strict, ojson* extras) {
    for (auto it = c.j->begin(); it != c.j->end(); ++it) {
        bool ok = std::any_of(known.begin(), known.end(), [&](const char* k) { return it.key() == k; });
        if (ok) continue;
        if (strict) c.fail("unknown field '" + it.key() + "'");
        if (extras) (*extras)[it.key()] = it.value();
    }
}

template <typename T>
ojson ops_json(const std::vector<Op<T>>& ops) {
    ojson a = ojson::array();
    for (const auto& o : ops) {
        ojson p;
        p["device"] = o.device;
        p["stage"] = o.stage;
        p["kind"] = kind_name(o.kind);
        p["microbatch"] = o.mb;
        p["start"] = o.start;
        p["duration"] = o.dur;
        a.push_back(std::move(p));
    }
    return a;
}

template <typename T>
void overlap_and_closure(const Plan<T>& p) {  // document.hpp:378-395
    std::vector<std::vector<std::pair<double, double>>> spans(size_t(p.topo.devices) + 1);
    for (const auto& o : p.ops) spans[o.device].push_back({double(o.start), double(o.start) + double(o.dur)});
    for (int d = 1; d <= p.topo.devices; ++d) {
        auto& v = spans[d];
        std::sort(v.begin(), v.end());
        for (size_t i = 1; i < v.size(); ++i)
            if (v[i].first < v[i - 1].second - 1e-9)
                throw DocumentError("/passes: collision on device " + std::to_string(d) + " at cell " +
                                    std::to_string(v[i].first));
    }
    auto probs = validate_schedule(p);
    if (!probs.empty()) throw DocumentError("/passes: " + probs.front());
}

}  // namespace

Document parse_document(const std::string& text, bool strict) {
    ojson j;
    try {
        j = ojson::parse(text);
    } catch (const nlohmann::json::parse_error& e) {
        throw DocumentError(std::string("malformed JSON: ") + e.what());
    }
    At root{&j, ""};
    root.object();
    Document d;
    int64_t ver = root.key("format_version").integer();
    if (ver != 1) root.key("format_version").fail("unsupported format_version " + std::to_string(ver));
    d.units = root.key("units").str();
    if (d.units != "cells" && d.units != "time") root.key("units").fail("units must be 'cells' or 'time'");

    At tc = root.key("topology");
    tc.object();
    known_fields(tc, {"devices", "num_stages", "placement", "stage_mem", "routes"}, strict, nullptr);
    Topology& t = d.topo;
    t.devices = int(tc.key("devices").integer());
    t.num_stages = int(tc.key("num_stages").integer());
    if (t.devices < 1) tc.key("devices").fail("must be positive");
    if (t.num_stages < 1) tc.key("num_stages").fail("must be positive");
    At pc = tc.key("placement");
    pc.array();
    if (int(pc.size()) != t.num_stages) pc.fail("placement must list one device per stage");
    for (size_t i = 0; i < pc.size(); ++i) {
        int dev = int(pc.idx(i).integer());
        if (dev < 1 || dev > t.devices) pc.idx(i).fail("device out of range");
        t.placement.push_back(dev);
    }
    At mc = tc.key("stage_mem");
    mc.array();
    if (int(mc.size()) != t.num_stages) mc.fail("stage_mem must list one value per stage");
    for (size_t i = 0; i < mc.size(); ++i) {
        double m = mc.idx(i).number();
        if (m < 0) mc.idx(i).fail("must be non-negative");
        t.stage_mem.push_back(m);
    }
    if (auto rc = tc.opt("routes")) {
        rc->array();
        for (size_t r = 0; r < rc->size(); ++r) {
            At one = rc->idx(r);
            one.array();
            std::vector<int> route;
            for (size_t i = 0; i < one.size(); ++i) {
                int s = int(one.idx(i).integer());
                if (s < 1 || s > t.num_stages) one.idx(i).fail("stage out of range");
                route.push_back(s);
            }
            if (route.empty()) one.fail("route must not be empty");
            t.routes.push_back(std::move(route));
        }
        if (t.routes.empty()) rc->fail("routes must not be empty");
    } else {
        t.routes = {Topology::iota(1, t.num_stages)};
    }

    d.microbatches = int(root.key("microbatches").integer());
    if (d.microbatches < 0) root.key("microbatches").fail("must be non-negative");

    At ps = root.key("passes");
    ps.array();
    auto common = [&](const At& c, auto& o) {
        c.object();
        known_fields(c, {"device", "stage", "kind", "microbatch", "start", "duration"}, strict, nullptr);
        o.device = int(c.key("device").integer());
        o.stage = int(c.key("stage").integer());
        auto k = kind_from_name(c.key("kind").str());
        if (!k) c.key("kind").fail("kind must be one of F, B, W, BW");
        o.kind = *k;
        o.mb = int(c.key("microbatch").integer());
        if (o.stage < 1 || o.stage > t.num_stages) c.key("stage").fail("stage out of range");
        if (o.device < 1 || o.device > t.devices) c.key("device").fail("device out of range");
        if (o.mb < 0 || o.mb >= d.microbatches) c.key("microbatch").fail("microbatch out of range");
    };
    if (d.is_grid()) {
        d.grid.topo = t;
        d.grid.microbatches = d.microbatches;
        for (size_t i = 0; i < ps.size(); ++i) {
            At c = ps.idx(i);
            GridOp o;
            common(c, o);
            o.start = c.key("start").integer("integer cell (cells units)");
            o.dur = c.key("duration").integer("integer cell count (cells units)");
            if (o.dur < 1) c.key("duration").fail("must be at least one cell");
            d.grid.ops.push_back(o);
        }
    } else {
        d.timed.topo = t;
        d.timed.microbatches = d.microbatches;
        for (size_t i = 0; i < ps.size(); ++i) {
            At c = ps.idx(i);
            TimedOp o;
            common(c, o);
            o.start = c.key("start").number();
            o.dur = c.key("duration").number();
            if (o.dur <= 0) c.key("duration").fail("must be positive");
            d.timed.ops.push_back(o);
        }
    }

    ojson meta_extras = ojson::object();
    if (auto mt = root.opt("metadata")) {
        mt->object();
        known_fields(*mt, {"source_block", "steps", "profile", "replicated_weights"}, strict, &meta_extras);
        if (auto sb = mt->opt("source_block")) d.source_block = sb->str();
        if (auto st = mt->opt("steps")) {
            st->array();
            for (size_t i = 0; i < st->size(); ++i) d.steps.push_back(st->idx(i).str());
        }
        if (auto pr = mt->opt("profile")) {
            pr->object();
            Profile p;
            p.f = pr->key("f").number();
            p.b = pr->key("b").number();
            p.w = pr->key("w").number();
            if (auto c = pr->opt("comm")) p.comm = c->number();
            d.profile = p;
        }
        if (auto rw = mt->opt("replicated_weights")) d.replicated_weights = rw->j->is_boolean() && rw->j->get<bool>();
    }
    d.meta_extras_json = meta_extras.dump();

    if (auto bc = root.opt("block")) {
        bc->object();
        known_fields(*bc, {"interval", "microbatches_per_block", "passes", "pattern"}, strict, nullptr);
        Block b;
        b.topo = t;
        b.interval = bc->key("interval").integer();
        if (b.interval < 1) bc->key("interval").fail("must be positive");
        b.mb_per_block = int(bc->key("microbatches_per_block").integer());
        At bp = bc->key("passes");
        bp.array();
        for (size_t i = 0; i < bp.size(); ++i) {
            At c = bp.idx(i);
            c.object();
            BlockOp o;
            o.stage = int(c.key("stage").integer());
            auto k = kind_from_name(c.key("kind").str());
            if (!k) c.key("kind").fail("kind must be one of F, B, W, BW");
            o.kind = *k;
            o.slot = int(c.key("microbatch").integer());
            o.offset = c.key("offset").integer();
            b.ops.push_back(o);
        }
        d.block = std::move(b);
        if (auto pt = bc->opt("pattern")) {
            pt->object();
            std::string kind = pt->key("kind").str();
            if (kind == "explicit") {
                At st = pt->key("starts");
                st.array();
                for (size_t i = 0; i < st.size(); ++i) d.pattern_starts.push_back(st.idx(i).integer());
                d.pattern_explicit = true;
            } else if (kind != "uniform") {
                pt->key("kind").fail("pattern kind must be 'uniform' or 'explicit'");
            }
            d.has_pattern = true;
        }
    }
    ojson extras = ojson::object();
    known_fields(root, {"format_version", "units", "topology", "microbatches", "passes", "metadata", "block"}, strict,
                 &extras);
    d.extras_json = extras.dump();

    if (d.is_grid())
        overlap_and_closure(d.grid);
    else
        overlap_and_closure(d.timed);
    return d;
}

std::string emit_document(const Document& d) {  // document.hpp:131-188
    ojson j;
    j["format_version"] = 1;
    j["units"] = d.units;
    ojson t;
    t["devices"] = d.topo.devices;
    t["num_stages"] = d.topo.num_stages;
    t["placement"] = d.topo.placement;
    t["stage_mem"] = d.topo.stage_mem;
    if (!d.topo.default_routes()) t["routes"] = d.topo.routes;
    j["topology"] = std::move(t);
    j["microbatches"] = d.microbatches;
    j["passes"] = d.is_grid() ? ops_json(d.grid.ops) : ops_json(d.timed.ops);
    ojson meta = ojson::object();
    if (d.source_block) meta["source_block"] = *d.source_block;
    if (!d.steps.empty()) meta["steps"] = d.steps;
    if (d.profile) {
        ojson p;
        p["f"] = d.profile->f;
        p["b"] = d.profile->b;
        p["w"] = d.profile->w;
        p["comm"] = d.profile->comm;
        meta["profile"] = std::move(p);
    }
    if (d.replicated_weights) meta["replicated_weights"] = true;
    ojson mx = ojson::parse(d.meta_extras_json);
    for (auto it = mx.begin(); it != mx.end(); ++it) meta[it.key()] = it.value();
    if (!meta.empty()) j["metadata"] = std::move(meta);
    if (d.block) {
        ojson b;
        b["interval"] = d.block->interval;
        b["microbatches_per_block"] = d.block->mb_per_block;
        ojson ps = ojson::array();
        for (const auto& o : d.block->ops) {
            ojson p;
            p["stage"] = o.stage;
            p["kind"] = kind_name(o.kind);
            p["microbatch"] = o.slot;
            p["offset"] = o.offset;
            ps.push_back(std::move(p));
        }
        b["passes"] = std::move(ps);
        if (d.has_pattern) {
            ojson pat;
            pat["kind"] = d.pattern_explicit ? "explicit" : "uniform";
            if (d.pattern_explicit) pat["starts"] = d.pattern_starts;
            b["pattern"] = std::move(pat);
        }
        j["block"] = std::move(b);
    }
    ojson ex = ojson::parse(d.extras_json);
    for (auto it = ex.begin(); it != ex.end(); ++it) j[it.key()] = it.value();
    return j.dump(2) + "\n";
}

// cli.hpp:146-156 (assembled_document)
Document document_for_assembly(const Build& b, const Grid& g, bool sq, bool re) {
    Document d;
    d.units = "cells";
    d.topo = g.topo;
    d.microbatches = g.microbatches;
    d.grid = g;
    sort_canonical(d.grid);
    d.source_block = b.name;
    d.steps = {"repeat"};
    if (sq) d.steps.push_back("squeeze");
    if (re) d.steps.push_back("reorder");
    d.replicated_weights = b.replicated_weights;
    d.block = b.block;
    return d;
}

Document document_for_timed(const Timed& t) {  // document.hpp:413-421
    Document d;
    d.units = "time";
    d.topo = t.topo;
    d.microbatches = t.microbatches;
    d.timed = t;
    sort_canonical(d.timed);
    return d;
}

}  // namespace vsched
