// vsched — the schedule front end of the B200 V-shape pipeline executor.
//
// A restatement of the reference "pipeblock" building-block API
// (/root/reference/proj/include/pipeblock/*.hpp) with the same results bit for
// bit (pinned by tests/golden against the reference compiled from its own
// headers).  The data model differs (one value-type model, free functions, no
// templates beyond the cell/time duration type), but the greedy passes —
// repeat, validate_schedule, squeeze, reorder (assemble.hpp:85-397) — follow
// the reference statement by statement: their tie-breaks ARE the op order the
// executor must reproduce and their error strings are part of the interface,
// so they are a close transliteration by necessity (CPU front end, not the
// B200 hot path).
//
//   reference symbol                         here
//   model.hpp:15  PassKind                   vsched::Kind
//   model.hpp:50  Topology                   vsched::Topology
//   model.hpp:129 BlockPass/BuildingBlock    vsched::BlockOp / vsched::Block
//   model.hpp:162 ScheduledPassT/ScheduleT   vsched::Op<T> / vsched::Plan<T>
//   model.hpp:189 RunTimeProfile             vsched::Profile
//   model.hpp:220 dependencies_of            vsched::prerequisites
//   gallery.hpp:499 build_entry              vsched::build_entry
//   assemble.hpp:85/188/269/405              vsched::repeat/squeeze/reorder/assemble
//   assemble.hpp:138 validate_schedule       vsched::validate_schedule
//   memory.hpp:63 exact_peak                 vsched::exact_peak
//   simulate.hpp:22 simulate                 vsched::simulate
//   document.hpp:188/192 emit/parse          vsched::emit_document/parse_document
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <tuple>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace vsched {

enum class Kind : uint8_t { F = 0, B = 1, W = 2, BW = 3 };

inline int width(Kind k) { return k == Kind::BW ? 2 : 1; }
const char* kind_name(Kind k);   // "F" "B" "W" "BW"
char kind_letter(Kind k);        // 'F' 'B' 'W' 'D'
std::optional<Kind> kind_from_name(const std::string& s);

// Stage -> device placement, 1-based on both sides (model.hpp:47-56).
struct Topology {
    int devices = 0;
    int num_stages = 0;
    std::vector<int> placement;        // placement[s-1]
    std::vector<double> stage_mem;     // activation units per stage
    std::vector<std::vector<int>> routes;

    int device_of(int stage) const { return placement.at(stage - 1); }
    double mem_of(int stage) const { return stage_mem.at(stage - 1); }
    const std::vector<int>& route_for(int mb) const { return routes[size_t(mb) % routes.size()]; }
    bool default_routes() const;
    bool operator==(const Topology&) const = default;

    static Topology straight(int d);
    static Topology v_shape(int d);
    static Topology twin(int d);
    static Topology looped(int d, int v);
    static std::vector<int> iota(int lo, int hi);
};

struct BlockOp {
    int stage = 0;
    Kind kind = Kind::F;
    int slot = 0;
    int64_t offset = 0;
    bool operator==(const BlockOp&) const = default;
};

struct Block {
    Topology topo;
    int64_t interval = 0;
    int mb_per_block = 1;
    std::vector<BlockOp> ops;
};

// A gallery build: block + optional non-uniform instance starts.
struct Build {
    std::string name;
    Block block;
    bool replicated_weights = false;
    std::function<std::vector<int64_t>(int)> explicit_starts;  // empty -> uniform
};

template <typename T>
struct Op {
    int device = 0;
    int stage = 0;
    Kind kind = Kind::F;
    int mb = 0;
    T start{};
    T dur{};
    T end() const { return start + dur; }
    bool operator==(const Op&) const = default;
};

template <typename T>
struct Plan {
    Topology topo;
    int microbatches = 0;
    std::vector<Op<T>> ops;
};

using GridOp = Op<int64_t>;
using TimedOp = Op<double>;
using Grid = Plan<int64_t>;
using Timed = Plan<double>;

struct Profile {
    double f = 1, b = 1, w = 1, comm = 0;
    double of(Kind k) const {
        switch (k) {
            case Kind::F: return f;
            case Kind::B: return b;
            case Kind::W: return w;
            case Kind::BW: return b + w;
        }
        return 0;
    }
};

struct Ref {
    int stage;
    Kind kind;  // B here means "B or BW"
    int mb;
};

// model.hpp:220-240
std::vector<Ref> prerequisites(const Topology& t, int stage, Kind kind, int mb);

// ---- blocks (gallery.hpp) ----
struct VChain {  // gallery.hpp:88-96
    int64_t df0 = 1, df1 = 1, db1 = 1, db0 = 1, t1 = 1, t2 = 1, t3 = 1;
};
struct VEdges {  // gallery.hpp:102-106
    std::vector<int64_t> down, up;
    int64_t t1 = 1, t2 = 1, t3 = 1;
};
Block v_block_edges(int d, const VEdges& e, int64_t interval = 6);
Block v_block(int d, const VChain& c, int64_t interval = 6);
bool place_greedy_w(Block& blk);
std::optional<std::string> first_block_violation(const Block& blk);
std::optional<std::pair<int, int64_t>> residue_clash(const Block& blk);  // (device, residue)

Build build_entry(const std::string& name, int d, const std::map<std::string, int64_t>& params = {});
std::vector<std::string> gallery_names();

// ---- assembly (assemble.hpp) ----
struct Collision {
    int device = 0;
    int64_t cell = 0;
    GridOp first, second;
    std::string str() const;
};
Grid repeat(const Block& blk, const std::vector<int64_t>* starts, int instances,
            std::optional<Collision>* collision);
Grid squeeze(const Grid& g);
Grid reorder(const Grid& g);
Grid assemble(const Build& b, int n, bool do_squeeze = true, bool do_reorder = true);

template <typename T>
std::vector<std::string> validate_schedule(const Plan<T>& p);
template <typename T>
void sort_canonical(Plan<T>& p);

// ---- memory (memory.hpp) ----
template <typename T>
std::vector<double> exact_peak(const Plan<T>& p);
std::vector<double> peak_bound(const Block& blk);
std::vector<double> steady_peak(const Block& blk);
struct TraceRow {
    double time;
    int device;
    double units;
};
template <typename T>
std::vector<TraceRow> memory_trace(const Plan<T>& p);

// ---- replay (simulate.hpp) ----
struct SimResult {
    Timed schedule;
    double makespan = 0;
    std::vector<double> busy, idle_total, idle_span;
    double bubble_rate = 0;
    std::vector<double> peak;
};
SimResult simulate(const Grid& g, const Profile& prof);
// simulate() with one duration per pass (canonical order) — replays measured
// per-pass times (e.g. from an isolated-pass executor run) in grid order.
SimResult replay(const Grid& g, const std::vector<double>& dur, double comm);
// Same accounting as simulate() over already-timed passes (used for measured
// timelines): makespan, busy, idle, bubble = 1 - sum busy / (d * makespan).
SimResult account(const Timed& t);

// ---- documents (document.hpp) ----
struct Document {
    std::string units = "cells";
    Topology topo;
    int microbatches = 0;
    Grid grid;
    Timed timed;
    std::optional<std::string> source_block;
    std::vector<std::string> steps;
    std::optional<Profile> profile;
    bool replicated_weights = false;
    std::optional<Block> block;
    bool has_pattern = false;
    bool pattern_explicit = false;
    std::vector<int64_t> pattern_starts;
    std::string extras_json = "{}";       // unknown top-level fields (kept verbatim)
    std::string meta_extras_json = "{}";  // unknown metadata fields
    bool is_grid() const { return units == "cells"; }
};
struct DocumentError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
Document parse_document(const std::string& text, bool strict = false);
std::string emit_document(const Document& d);
Document document_for_assembly(const Build& b, const Grid& g, bool sq, bool re);
Document document_for_timed(const Timed& t);

// ---- growth (growth.hpp) — vanalysis.cpp ----
struct Growth {  // growth.hpp:13-22
    int cycle_length = 0;
    double growth = 0.0;
    std::vector<double> work_per_period;
    double max_work = 0.0;
    double repeating_bubble = 0.0;
    bool linear_bubble = false;
    bool tie = false;
    std::vector<std::string> witness;
};
Growth growth_rate(const Block& blk, const Profile& prof);
double growth_rate_unrolled(const Block& blk, const Profile& prof, int periods);
bool vhalf_condition(const Profile& p);
int64_t makespan_lower_bound(int64_t n, int64_t d, int64_t k);  // growth.hpp:195 lower_bound
double min_memory_for_od_bubble(int d);

// ---- adaptive search (search.hpp) — vanalysis.cpp ----
struct SearchSpec {  // search.hpp:15-25
    int d = 0;
    int n = 0;  // 0 -> 3d
    Profile profile;
    double memory_limit = 0.0;  // units of m
    int64_t delta_max = 6, tau_max = 6;
    int eval_n() const { return n > 0 ? n : 3 * d; }
};
struct SearchParams {  // search.hpp:27-42
    int K = 1;
    int64_t d0_lo = 1, d1_lo = 1, d0_hi = 1, d1_hi = 1;
    int64_t tau1 = 1, tau2 = 1, tau3 = 1;
    auto key() const { return std::tie(K, d0_lo, d1_lo, d0_hi, d1_hi, tau1, tau2, tau3); }
    std::string str() const;
    VEdges edges(int d) const;
};
struct SearchResult {  // search.hpp:44-56
    bool feasible = false;
    std::string message;
    SearchParams best;
    Build build;
    Grid schedule;
    double bubble_rate = 1.0, exact_peak = 0.0;
    int64_t enumerated = 0, evaluated = 0;
    double family_min_peak = 0.0;
    bool turn_devices_exercised = false;
};
struct FrontierPoint {
    double limit = 0.0;
    bool feasible = false;
    double bubble_rate = 1.0, exact_peak = 0.0;
    SearchParams best;
};
Block search_block(int d, const SearchParams& p);  // one family member's block (search.hpp:208-216)

class Family {  // search.hpp:121-206 FamilyEvaluation
  public:
    struct Eval {
        SearchParams params;
        double peak = 0.0, bubble = 1.0;
    };
    explicit Family(const SearchSpec& spec);
    int64_t enumerated() const { return enumerated_; }
    int64_t evaluated() const { return int64_t(evals_.size()); }
    double family_min_peak() const { return min_peak_; }
    std::optional<Eval> best_under(double limit) const;
    Block rebuild(const SearchParams& p) const;
    Build build_of(const SearchParams& p) const;

  private:
    static constexpr int64_t kInterval = 6;
    SearchSpec spec_;
    int64_t enumerated_ = 0;
    double min_peak_ = std::numeric_limits<double>::infinity();
    std::vector<Eval> evals_;
};
SearchResult search_with(const Family& fam, const SearchSpec& spec);
SearchResult search(const SearchSpec& spec);
std::vector<FrontierPoint> frontier(const SearchSpec& spec, const std::vector<double>& limits);

// ---- render (render.hpp) — vanalysis.cpp ----
struct RenderOptions {
    bool stamp = false;
    std::string title;
    int ascii_max_width = 200;
    bool ascii_color = false;
    std::vector<char> highlight;
};
std::string render_svg(const Document& doc, const RenderOptions& opt = {});
std::string render_ascii(const Document& doc, const RenderOptions& opt = {});

}  // namespace vsched
