// vanalysis — the analysis side of the schedule front end:
// stable-phase growth of a repeated block (growth.hpp), the adaptive V-family
// search and its memory/bubble frontier (search.hpp), and the SVG / ASCII
// Gantt views of grid or measured timelines (render.hpp).  Restated from the
// reference's published semantics; outputs are pinned bit for bit (numbers,
// witnesses, SVG/ASCII bytes) by tests/test_analysis_golden.py against the
// reference compiled from its own headers.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <iomanip>
#include <limits>
#include <map>
#include <sstream>
#include <tuple>

#include "schedule/vsched.hpp"

namespace vsched {

// ============================================================ growth (growth.hpp)
//
// One building-block period as a cyclic graph: node = block op; arcs are the
// device succession in residue order (the last op of a device wraps into the
// next period) and the dependency arcs (period shift = floor(offset / T)
// difference).  Arc weight = duration of the source op (+ comm across
// devices).  The growth per period is the heaviest (node, p0) -> (node, p1)
// path on the two-period unrolling (growth.hpp:98-187).
namespace {

struct Arc {
    int to;
    int shift;
    double w;
};

struct PeriodGraph {
    int n = 0;
    std::vector<std::vector<Arc>> arcs;
    std::vector<int64_t> residue;
    std::vector<std::string> label;
    std::vector<int> topo_order;  // ids of the unrolled DAG in (period, residue) order
    int periods = 0;

    PeriodGraph(const Block& blk, const Profile& prof) {  // growth.hpp:39-94
        if (blk.interval <= 0) throw std::invalid_argument("growth: interval must be positive");
        n = int(blk.ops.size());
        arcs.resize(n);
        residue.resize(n);
        label.resize(n);
        std::map<std::tuple<int, int, int>, int> at;  // (stage, kind, slot) -> node
        for (int i = 0; i < n; ++i) {
            const auto& o = blk.ops[i];
            residue[i] = ((o.offset % blk.interval) + blk.interval) % blk.interval;
            label[i] = std::string(kind_name(o.kind)) + "(stage " + std::to_string(o.stage) + ", slot " +
                       std::to_string(o.slot) + ")";
            at[{o.stage, int(o.kind), o.slot}] = i;
        }
        auto lookup = [&](const Ref& r) -> int {
            auto it = at.find({r.stage, int(r.kind), r.mb});
            if (it == at.end() && (r.kind == Kind::B || r.kind == Kind::BW))
                it = at.find({r.stage, int(r.kind == Kind::B ? Kind::BW : Kind::B), r.mb});
            return it == at.end() ? -1 : it->second;
        };
        std::map<int, std::vector<int>> per_dev;
        for (int i = 0; i < n; ++i) per_dev[blk.topo.device_of(blk.ops[i].stage)].push_back(i);
        for (auto& [dev, ids] : per_dev) {
            std::sort(ids.begin(), ids.end(), [&](int a, int b) { return residue[a] < residue[b]; });
            for (size_t k = 0; k < ids.size(); ++k) {
                bool wrap = k + 1 == ids.size();
                arcs[ids[k]].push_back({ids[wrap ? 0 : k + 1], wrap ? 1 : 0, prof.of(blk.ops[ids[k]].kind)});
            }
        }
        for (int v = 0; v < n; ++v) {
            const auto& o = blk.ops[v];
            for (const auto& r : prerequisites(blk.topo, o.stage, o.kind, o.slot)) {
                int u = lookup(r);
                if (u < 0) continue;
                const auto& src = blk.ops[u];
                double w = prof.of(src.kind);
                if (blk.topo.device_of(src.stage) != blk.topo.device_of(o.stage)) w += prof.comm;
                arcs[u].push_back({v, int(o.offset / blk.interval - src.offset / blk.interval), w});
            }
        }
    }

    void unroll(int p) {
        if (periods == p) return;
        periods = p;
        topo_order.resize(size_t(n) * p);
        for (int i = 0; i < n * p; ++i) topo_order[i] = i;
        std::sort(topo_order.begin(), topo_order.end(), [&](int a, int b) {
            return std::make_pair(a / n, residue[a % n]) < std::make_pair(b / n, residue[b % n]);
        });
    }

    // heaviest path (src, period 0) -> (src, period p-1)
    double heaviest_cycle(int src, int p, std::vector<int>* parent_out) {
        unroll(p);
        const double ninf = -std::numeric_limits<double>::infinity();
        std::vector<double> dist(size_t(n) * p, ninf);
        std::vector<int> parent(size_t(n) * p, -1);
        dist[src] = 0.0;
        for (int id : topo_order) {
            if (dist[id] == ninf) continue;
            int u = id % n, period = id / n;
            for (const auto& a : arcs[u]) {
                int np = period + a.shift;
                if (np >= p) continue;
                int nid = np * n + a.to;
                if (dist[id] + a.w > dist[nid]) {
                    dist[nid] = dist[id] + a.w;
                    parent[nid] = id;
                }
            }
        }
        if (parent_out) *parent_out = std::move(parent);
        return dist[size_t(p - 1) * n + src];
    }
};

}  // namespace

double growth_rate_unrolled(const Block& blk, const Profile& prof, int periods) {  // growth.hpp:132-139
    PeriodGraph g(blk, prof);
    double best = 0.0;
    for (int s = 0; s < g.n; ++s) best = std::max(best, g.heaviest_cycle(s, periods, nullptr));
    return best;
}

Growth growth_rate(const Block& blk, const Profile& prof) {  // growth.hpp:141-187
    PeriodGraph g(blk, prof);
    Growth r;
    r.work_per_period.assign(blk.topo.devices, 0.0);
    std::vector<int> count(blk.topo.devices, 0);
    for (const auto& o : blk.ops) {
        int dev = blk.topo.device_of(o.stage);
        r.work_per_period[dev - 1] += prof.of(o.kind);
        count[dev - 1] += 1;
    }
    for (int d = 0; d < blk.topo.devices; ++d) {
        if (!count[d]) continue;
        r.max_work = std::max(r.max_work, r.work_per_period[d]);
        r.cycle_length = std::max(r.cycle_length, count[d]);
    }
    int best_src = -1;
    std::vector<int> best_parent;
    for (int s = 0; s < g.n; ++s) {
        std::vector<int> parent;
        double v = g.heaviest_cycle(s, 2, &parent);
        if (v > r.growth) {
            r.growth = v;
            best_src = s;
            best_parent = std::move(parent);
        }
    }
    const double eps = 1e-9 * std::max(1.0, r.max_work);
    r.repeating_bubble = std::max(0.0, r.growth - r.max_work);
    r.linear_bubble = r.repeating_bubble > eps;
    r.tie = std::abs(r.growth - r.max_work) <= eps;
    if (best_src >= 0) {
        for (int id = g.n + best_src; id >= 0; id = best_parent[id])
            r.witness.push_back(g.label[id % g.n] + "@period" + std::to_string(id / g.n));
        std::reverse(r.witness.begin(), r.witness.end());
    }
    return r;
}

bool vhalf_condition(const Profile& p) {  // growth.hpp:190-192
    return p.w + 2 * p.b >= 2 * p.f && p.w + 2 * p.f >= 2 * p.b;
}

int64_t makespan_lower_bound(int64_t n, int64_t d, int64_t k) {  // growth.hpp:195-198
    if (k < 1 || k > 2 * d) throw std::invalid_argument("lower_bound: k must be in [1, 2d]");
    return std::max(6 * n, 6 * n + 6 * d - 3 * k - 1);
}

double min_memory_for_od_bubble(int d) {  // growth.hpp:202-205
    if (d < 1) throw std::invalid_argument("min_memory_for_od_bubble: d must be positive");
    return 2.0 * d;
}

// ============================================================ search (search.hpp)
//
// The V family with two spacing values per chain direction, switching at the
// split device K, plus the three turn gaps.  Every canonical, residue-clean
// candidate is assembled at n = eval_n, replayed under the profile and its
// exact peak recorded once; search/frontier then pick the lowest bubble under
// a memory limit (ties: lexicographic parameters).
std::string SearchParams::str() const {
    std::ostringstream s;
    s << "K=" << K << " d0=(" << d0_lo << ',' << d0_hi << ") d1=(" << d1_lo << ',' << d1_hi << ") tau=(" << tau1
      << ',' << tau2 << ',' << tau3 << ')';
    return s.str();
}

VEdges SearchParams::edges(int d) const {  // search.hpp:67-82
    VEdges e;
    e.down.resize(std::max(0, d - 1));
    e.up.resize(std::max(0, d - 1));
    for (int x = 0; x + 1 < d; ++x) {
        e.down[x] = (x + 1) < K ? d0_lo : d0_hi;      // device pair (x+1, x+2)
        e.up[x] = (d - x - 1) <= K ? d1_lo : d1_hi;   // device pair (d-x-1, d-x)
    }
    e.t1 = tau1;
    e.t2 = tau2;
    e.t3 = tau3;
    return e;
}

namespace {

// The four chain cells of every device (F down, F up, B up, B down) must
// occupy distinct residues mod the interval (search.hpp:84-108).
bool chain_cells_distinct(int d, const VEdges& e, int64_t T) {
    std::vector<int64_t> f(2 * d), b(2 * d);
    f[0] = 0;
    for (int i = 1; i < d; ++i) f[i] = f[i - 1] + e.down[i - 1];
    f[d] = f[d - 1] + e.t1;
    for (int i = d + 1; i < 2 * d; ++i) f[i] = f[i - 1] + e.up[i - d - 1];
    b[2 * d - 1] = f[2 * d - 1] + e.t2;
    for (int k = 1; k < d; ++k) b[2 * d - 1 - k] = b[2 * d - k] + e.down[k - 1];
    b[d - 1] = b[d] + e.t3;
    for (int l = 1; l < d; ++l) b[d - 1 - l] = b[d - l] + e.up[l - 1];
    for (int dev = 1; dev <= d; ++dev) {
        unsigned seen = 0;
        for (int64_t c : {f[dev - 1], f[2 * d - dev], b[2 * d - dev], b[dev - 1]}) {
            unsigned bit = 1u << (c % T);
            if (seen & bit) return false;
            seen |= bit;
        }
    }
    return true;
}

}  // namespace

Block Family::rebuild(const SearchParams& p) const { return search_block(spec_.d, p); }

// search.hpp:208-216 (FamilyEvaluation::rebuild) without the family: the block of one parameter
// tuple, e.g. to assemble a searched winner at the step's own microbatch count
Block search_block(int d, const SearchParams& p) {
    if (d < 2) throw std::invalid_argument("search: d must be at least 2");
    Block blk = v_block_edges(d, p.edges(d), 6);
    if (!place_greedy_w(blk)) throw std::invalid_argument("search: W fill failed on rebuild");
    return blk;
}

Build Family::build_of(const SearchParams& p) const {
    Build b;
    b.name = "search";
    b.block = rebuild(p);
    return b;
}

Family::Family(const SearchSpec& spec) : spec_(spec) {  // search.hpp:121-206
    const int d = spec.d;
    if (d < 2) throw std::invalid_argument("search: d must be at least 2");
    if (spec.delta_max < 1 || spec.tau_max < 1) throw std::invalid_argument("search: ranges must be positive");
    const int64_t D = spec.delta_max, U = spec.tau_max;
    SearchParams c;
    for (c.K = 1; c.K <= d; ++c.K)
        for (c.d0_lo = 1; c.d0_lo <= D; ++c.d0_lo)
            for (c.d1_lo = 1; c.d1_lo <= D; ++c.d1_lo)
                for (c.d0_hi = 1; c.d0_hi <= D; ++c.d0_hi)
                    for (c.d1_hi = 1; c.d1_hi <= D; ++c.d1_hi)
                        for (c.tau1 = 1; c.tau1 <= U; ++c.tau1)
                            for (c.tau2 = 1; c.tau2 <= U; ++c.tau2)
                                for (c.tau3 = 1; c.tau3 <= U; ++c.tau3) {
                                    ++enumerated_;
                                    // spacings that touch no edge are pinned to 1
                                    if ((c.K == 1 && c.d0_lo != 1) || (c.K == d && c.d0_hi != 1) ||
                                        (c.K >= d - 1 && c.d1_hi != 1))
                                        continue;
                                    if (!chain_cells_distinct(d, c.edges(d), kInterval)) continue;
                                    Grid g = assemble(build_of(c), spec.eval_n());
                                    auto pk = exact_peak(g);
                                    evals_.push_back({c, *std::max_element(pk.begin(), pk.end()),
                                                      simulate(g, spec.profile).bubble_rate});
                                }
    for (const auto& e : evals_) min_peak_ = std::min(min_peak_, e.peak);
}

std::optional<Family::Eval> Family::best_under(double limit) const {
    std::optional<Eval> best;
    for (const auto& e : evals_) {
        if (e.peak > limit + 1e-9) continue;
        if (!best || e.bubble < best->bubble - 1e-12 ||
            (std::abs(e.bubble - best->bubble) <= 1e-12 && e.params.key() < best->params.key()))
            best = e;
    }
    return best;
}

SearchResult search_with(const Family& fam, const SearchSpec& spec) {  // search.hpp:208-233
    SearchResult r;
    r.enumerated = fam.enumerated();
    r.evaluated = fam.evaluated();
    r.family_min_peak = fam.family_min_peak();
    auto best = fam.best_under(spec.memory_limit);
    if (!best) {
        std::ostringstream m;
        m << "infeasible: memory limit " << spec.memory_limit << "m is below the family minimum "
          << fam.family_min_peak() << "m";
        r.message = m.str();
        return r;
    }
    r.feasible = true;
    r.best = best->params;
    r.bubble_rate = best->bubble;
    r.exact_peak = best->peak;
    r.build = fam.build_of(best->params);
    r.schedule = assemble(r.build, spec.eval_n());
    r.turn_devices_exercised = best->params.tau1 != 1 || best->params.tau3 != 1;
    return r;
}

SearchResult search(const SearchSpec& spec) { return search_with(Family(spec), spec); }

std::vector<FrontierPoint> frontier(const SearchSpec& spec, const std::vector<double>& limits) {
    Family fam(spec);
    std::vector<FrontierPoint> out;
    for (double lim : limits) {
        FrontierPoint pt;
        pt.limit = lim;
        if (auto b = fam.best_under(lim)) {
            pt.feasible = true;
            pt.bubble_rate = b->bubble;
            pt.exact_peak = b->peak;
            pt.best = b->params;
        }
        out.push_back(pt);
    }
    return out;
}

// ============================================================ render (render.hpp)
namespace {

struct Shade {
    const char *light, *dark, *ink_light, *ink_dark;
};
Shade shade(Kind k) {  // render.hpp:29-37
    switch (k) {
        case Kind::F: return {"#cfe3f7", "#2c5d8f", "#17364f", "#f3f8fd"};
        case Kind::B: return {"#cdecd2", "#2e7d44", "#1c4427", "#f1faf3"};
        case Kind::W: return {"#fbe3b5", "#b07818", "#59400d", "#fdf6e7"};
        case Kind::BW: return {"#d8d2ef", "#5b4ea0", "#2f2753", "#f4f2fb"};
    }
    return {"#eeeeee", "#444444", "#000000", "#ffffff"};
}

// A document's passes as (device, stage, kind, mb, start, duration) in document order.
struct Bar {
    int device, stage;
    Kind kind;
    int mb;
    double start, dur;
};
std::vector<Bar> bars_of(const Document& doc) {
    std::vector<Bar> out;
    if (doc.is_grid())
        for (const auto& o : doc.grid.ops) out.push_back({o.device, o.stage, o.kind, o.mb, double(o.start), double(o.dur)});
    else
        for (const auto& o : doc.timed.ops) out.push_back({o.device, o.stage, o.kind, o.mb, o.start, o.dur});
    return out;
}
double span_of(const std::vector<Bar>& bars) {
    double e = 0.0;
    for (const auto& b : bars) e = std::max(e, b.start + b.dur);
    return e;
}
std::string xml_text(const std::string& s) {
    std::string out;
    for (char c : s) {
        if (c == '&') out += "&amp;";
        else if (c == '<') out += "&lt;";
        else if (c == '>') out += "&gt;";
        else out += c;
    }
    return out;
}
int px_of(double v) { return int(std::lround(v)); }

}  // namespace

std::string render_svg(const Document& doc, const RenderOptions& opt) {  // render.hpp:83-172
    const int rows = doc.topo.devices;
    const int left = 64, top = 30, row_h = 24, gap = 5, bottom = 34;
    const auto bars = bars_of(doc);
    const double span = span_of(bars);
    double scale;
    if (doc.is_grid())
        scale = span <= 90 ? 16.0 : std::max(2.0, std::floor(1440.0 / std::max(1.0, span)));
    else
        scale = span <= 0 ? 16.0 : std::min(16.0, 1440.0 / span);
    const int W = left + px_of(span * scale) + 16;
    const int H = top + rows * (row_h + gap) + bottom;
    std::string title = !opt.title.empty() ? opt.title : doc.source_block ? *doc.source_block : std::string("schedule");

    std::ostringstream s;
    s << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << W << "\" height=\"" << H << "\" viewBox=\"0 0 " << W
      << ' ' << H << "\" font-family=\"monospace\">\n";
    if (opt.stamp) {
        std::time_t now = std::time(nullptr);
        char buf[64];
        std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", std::gmtime(&now));
        s << "<!-- generated " << buf << " -->\n";
    }
    s << "<rect x=\"0\" y=\"0\" width=\"" << W << "\" height=\"" << H << "\" fill=\"#ffffff\"/>\n";
    s << "<text x=\"" << left << "\" y=\"18\" font-size=\"13\" fill=\"#222222\">" << xml_text(title) << "</text>\n";
    for (int dev = 1; dev <= rows; ++dev) {
        int y = top + (dev - 1) * (row_h + gap);
        s << "<text x=\"8\" y=\"" << y + row_h - 8 << "\" font-size=\"11\" fill=\"#444444\">dev " << dev
          << "</text>\n";
        s << "<line x1=\"" << left << "\" y1=\"" << y + row_h << "\" x2=\"" << W - 8 << "\" y2=\"" << y + row_h
          << "\" stroke=\"#dddddd\" stroke-width=\"1\"/>\n";
    }
    for (size_t i = 0; i < bars.size(); ++i) {
        const Bar& b = bars[i];
        int x = left + px_of(b.start * scale);
        int w = std::max(2, px_of(b.dur * scale) - 1);
        int y = top + (b.device - 1) * (row_h + gap);
        Shade c = shade(b.kind);
        bool dark = b.stage > doc.topo.devices;  // return leg of the V drawn dark
        s << "<rect x=\"" << x << "\" y=\"" << y << "\" width=\"" << w << "\" height=\"" << row_h << "\" fill=\""
          << (dark ? c.dark : c.light) << "\"";
        if (i < opt.highlight.size() && opt.highlight[i]) s << " stroke=\"#d62728\" stroke-width=\"2\"";
        s << "/>\n";
        if (w >= 12)
            s << "<text x=\"" << x + w / 2 << "\" y=\"" << y + row_h / 2 + 4
              << "\" font-size=\"9\" text-anchor=\"middle\" fill=\"" << (dark ? c.ink_dark : c.ink_light) << "\">"
              << b.mb << "</text>\n";
    }
    const int axis_y = top + rows * (row_h + gap) + 6;
    s << "<line x1=\"" << left << "\" y1=\"" << axis_y << "\" x2=\"" << left + px_of(span * scale) << "\" y2=\""
      << axis_y << "\" stroke=\"#888888\" stroke-width=\"1\"/>\n";
    double tick = 1.0;
    while (span / tick > 12.0) tick *= 2.0;
    for (double t = 0.0; t <= span + 1e-9; t += tick) {
        int x = left + px_of(t * scale);
        s << "<line x1=\"" << x << "\" y1=\"" << axis_y << "\" x2=\"" << x << "\" y2=\"" << axis_y + 4
          << "\" stroke=\"#888888\" stroke-width=\"1\"/>\n";
        std::ostringstream lbl;
        lbl << t;
        s << "<text x=\"" << x << "\" y=\"" << axis_y + 16 << "\" font-size=\"9\" text-anchor=\"middle\" fill=\"#666666\">"
          << lbl.str() << "</text>\n";
    }
    s << "</svg>\n";
    return s.str();
}

std::string render_ascii(const Document& doc, const RenderOptions& opt) {  // render.hpp:177-256
    const auto bars = bars_of(doc);
    const double span = span_of(bars);
    if (span <= 0) return "(empty schedule)\n";
    int cols = int(std::ceil(span - 1e-9));
    double step = 1.0;
    bool sampled = false;
    if (cols > opt.ascii_max_width) {
        cols = opt.ascii_max_width;
        step = span / cols;
        sampled = true;
    }
    const int rows = doc.topo.devices;
    std::vector<std::string> cell(rows, std::string(cols, '.'));
    std::vector<std::vector<bool>> lower(rows, std::vector<bool>(cols, false));
    for (const Bar& b : bars) {
        int c0 = std::clamp(int(std::floor(b.start / step + 1e-9)), 0, cols - 1);
        int c1 = std::clamp(int(std::ceil((b.start + b.dur) / step - 1e-9)), c0 + 1, cols);
        bool lo = b.stage > doc.topo.devices;
        char ch = kind_letter(b.kind);
        for (int c = c0; c < c1; ++c) {
            cell[b.device - 1][c] = lo ? char(std::tolower(ch)) : ch;
            lower[b.device - 1][c] = lo;
        }
    }
    auto ansi = [](char c) -> const char* {
        switch (std::toupper(c)) {
            case 'F': return "36";
            case 'B': return "32";
            case 'W': return "33";
            case 'D': return "35";
        }
        return nullptr;
    };
    std::ostringstream out;
    for (int dev = 1; dev <= rows; ++dev) {
        out << "dev " << std::setw(2) << dev << " |";
        for (int c = 0; c < cols; ++c) {
            char ch = cell[dev - 1][c];
            const char* col = opt.ascii_color ? ansi(ch) : nullptr;
            if (!col)
                out << ch;
            else
                out << "\033[" << (lower[dev - 1][c] ? "7;" : "") << col << 'm' << ch << "\033[0m";
        }
        out << "|\n";
    }
    out << "legend: F forward, B input grad, W weight grad, D fused backward, . idle;"
        << " lowercase marks second-half stages\n";
    if (sampled) {
        std::ostringstream r;
        r << std::setprecision(3) << step;
        out << "note: schedule wider than " << opt.ascii_max_width << " columns, each column covers about " << r.str()
            << " cells\n";
    }
    return out.str();
}

}  // namespace vsched
