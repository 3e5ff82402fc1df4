// vsched implementation.  See vsched.hpp for the reference map; every routine
// below names the reference lines whose semantics it restates.
#include "vsched.hpp"

#include <algorithm>
#include <set>
#include <tuple>
#include <unordered_map>

namespace vsched {

const char* kind_name(Kind k) {
    static const char* names[] = {"F", "B", "W", "BW"};
    return names[static_cast<int>(k) & 3];
}
char kind_letter(Kind k) { return "FBWD"[static_cast<int>(k) & 3]; }
std::optional<Kind> kind_from_name(const std::string& s) {
    for (int i = 0; i < 4; ++i)
        if (s == kind_name(static_cast<Kind>(i))) return static_cast<Kind>(i);
    return std::nullopt;
}

// ---------------------------------------------------------------- topology
std::vector<int> Topology::iota(int lo, int hi) {
    std::vector<int> r;
    for (int s = lo; s <= hi; ++s) r.push_back(s);
    return r;
}
bool Topology::default_routes() const { return routes.size() == 1 && routes[0] == iota(1, num_stages); }

static Topology make_topo(int d, int stages, const std::function<int(int)>& dev) {
    Topology t;
    t.devices = d;
    t.num_stages = stages;
    for (int s = 1; s <= stages; ++s) t.placement.push_back(dev(s));
    t.stage_mem.assign(stages, 1.0);
    t.routes = {Topology::iota(1, stages)};
    return t;
}
Topology Topology::straight(int d) { return make_topo(d, d, [](int s) { return s; }); }
Topology Topology::v_shape(int d) {  // model.hpp:79-91: stage i -> i, stage d+i -> d+1-i
    return make_topo(d, 2 * d, [d](int s) { return s <= d ? s : 2 * d + 1 - s; });
}
Topology Topology::twin(int d) {
    Topology t = v_shape(d);
    t.routes = {iota(1, d), iota(d + 1, 2 * d)};
    return t;
}
Topology Topology::looped(int d, int v) {
    return make_topo(d, d * v, [d](int s) { return (s - 1) % d + 1; });
}

// model.hpp:220-240.  F follows the previous route stage; B/BW needs its own F
// and the next route stage's backward; W follows its own B.
std::vector<Ref> prerequisites(const Topology& t, int stage, Kind kind, int mb) {
    const auto& route = t.route_for(mb);
    auto it = std::find(route.begin(), route.end(), stage);
    if (it == route.end()) throw std::invalid_argument("stage not on this microbatch's route");
    size_t pos = size_t(it - route.begin());
    std::vector<Ref> out;
    if (kind == Kind::F) {
        if (pos > 0) out.push_back({route[pos - 1], Kind::F, mb});
    } else if (kind == Kind::W) {
        out.push_back({stage, Kind::B, mb});
    } else {
        out.push_back({stage, Kind::F, mb});
        if (pos + 1 < route.size()) out.push_back({route[pos + 1], kind, mb});
    }
    return out;
}

// ---------------------------------------------------------------- lookups
namespace {

// (mb, stage, kind) -> op index; backward kinds resolve split/fused either way
// (assemble.hpp:13-48; the key packing there limits stages to < 4096).
template <typename T>
struct Lookup {
    std::unordered_map<int64_t, size_t> at;
    static int64_t key(int stage, Kind k, int mb) { return ((int64_t(mb) << 13) + stage) * 4 + int(k); }
    explicit Lookup(const Plan<T>& p) {
        at.reserve(p.ops.size() * 2);
        for (size_t i = 0; i < p.ops.size(); ++i) at[key(p.ops[i].stage, p.ops[i].kind, p.ops[i].mb)] = i;
    }
    std::optional<size_t> find(int stage, Kind k, int mb) const {
        auto it = at.find(key(stage, k, mb));
        if (it == at.end() && (k == Kind::B || k == Kind::BW))
            it = at.find(key(stage, k == Kind::B ? Kind::BW : Kind::B, mb));
        if (it == at.end()) return std::nullopt;
        return it->second;
    }
    std::vector<size_t> deps(const Plan<T>& p, const Op<T>& o) const {
        std::vector<size_t> r;
        for (const Ref& d : prerequisites(p.topo, o.stage, o.kind, o.mb))
            if (auto i = find(d.stage, d.kind, d.mb)) r.push_back(*i);
        return r;
    }
};

std::string op_str(const GridOp& o) {
    return std::string(kind_name(o.kind)) + "(stage " + std::to_string(o.stage) + ", microbatch " +
           std::to_string(o.mb) + ")";
}
std::string block_op_str(const BlockOp& o) {
    return std::string(kind_name(o.kind)) + "(stage " + std::to_string(o.stage) + ", mb " + std::to_string(o.slot) +
           ")@" + std::to_string(o.offset);
}

}  // namespace

template <typename T>
void sort_canonical(Plan<T>& p) {  // assemble.hpp:50-57
    std::sort(p.ops.begin(), p.ops.end(), [](const Op<T>& a, const Op<T>& b) {
        return std::tie(a.device, a.start, a.stage, a.mb) < std::tie(b.device, b.start, b.stage, b.mb);
    });
}
template void sort_canonical(Plan<int64_t>&);
template void sort_canonical(Plan<double>&);

// ---------------------------------------------------------------- blocks
std::optional<std::pair<int, int64_t>> residue_clash(const Block& blk) {  // model.hpp:385-396
    std::set<std::pair<int, int64_t>> seen;
    for (const auto& o : blk.ops) {
        int dev = blk.topo.device_of(o.stage);
        for (int c = 0; c < width(o.kind); ++c) {
            int64_t r = (o.offset + c) % blk.interval;
            if (!seen.insert({dev, r}).second) return std::make_pair(dev, r);
        }
    }
    return std::nullopt;
}

// model.hpp:294-375, first violation only (the reference reports all; callers
// only ever surface the first one, gallery.hpp:162-164).
std::optional<std::string> first_block_violation(const Block& blk) {
    const Topology& t = blk.topo;
    std::map<std::tuple<int, int, int>, const BlockOp*> idx;
    std::vector<std::string> v;
    for (const auto& o : blk.ops) {
        if (o.stage < 1 || o.stage > t.num_stages) { v.push_back("stage out of range: " + block_op_str(o)); continue; }
        if (o.slot < 0 || o.slot >= blk.mb_per_block) { v.push_back("slot out of range: " + block_op_str(o)); continue; }
        if (o.offset < 0) v.push_back("negative offset: " + block_op_str(o));
        if (!idx.insert({{o.stage, int(o.kind), o.slot}, &o}).second) v.push_back("duplicate pass: " + block_op_str(o));
    }
    for (int slot = 0; slot < blk.mb_per_block; ++slot)
        for (int stage : t.route_for(slot)) {
            auto has = [&](Kind k) { return idx.count({stage, int(k), slot}) > 0; };
            std::string at = "stage " + std::to_string(stage) + ", slot " + std::to_string(slot);
            if (!has(Kind::F)) v.push_back("missing F at " + at);
            bool fused = has(Kind::BW), split_b = has(Kind::B), split_w = has(Kind::W);
            if (fused && (split_b || split_w)) v.push_back("fused BW next to split pass at " + at);
            if (!fused && !(split_b && split_w)) v.push_back("incomplete backward at " + at);
        }
    std::map<std::pair<int, int64_t>, const BlockOp*> cells;
    for (const auto& o : blk.ops) {
        if (o.stage < 1 || o.stage > t.num_stages) continue;
        int dev = t.device_of(o.stage);
        for (int c = 0; c < width(o.kind); ++c) {
            auto [it, fresh] = cells.insert({{dev, o.offset + c}, &o});
            if (!fresh) v.push_back(block_op_str(*it->second) + " overlaps " + block_op_str(o));
        }
    }
    for (const auto& o : blk.ops) {
        if (o.stage < 1 || o.stage > t.num_stages || o.slot < 0 || o.slot >= blk.mb_per_block) continue;
        for (const Ref& d : prerequisites(t, o.stage, o.kind, o.slot)) {
            auto it = idx.find({d.stage, int(d.kind), d.mb});
            if (it == idx.end() && (d.kind == Kind::B || d.kind == Kind::BW))
                it = idx.find({d.stage, int(d.kind == Kind::B ? Kind::BW : Kind::B), d.mb});
            if (it == idx.end()) {
                v.push_back("unresolved prerequisite of " + block_op_str(o));
            } else if (it->second->offset + width(it->second->kind) > o.offset) {
                v.push_back(block_op_str(o) + " starts before its " + kind_name(d.kind) + "(stage " +
                            std::to_string(d.stage) + ") ends");
            }
        }
    }
    if (v.empty()) return std::nullopt;
    return v.front();
}

// gallery.hpp:50-82: each split B without a W gets its W at the earliest cell
// >= B end whose residue (mod interval) is free on its device; needs are
// visited by (B end, stage, slot).
bool place_greedy_w(Block& blk) {
    std::set<std::pair<int, int64_t>> used;
    std::set<std::pair<int, int>> has_w;
    for (const auto& o : blk.ops) {
        int dev = blk.topo.device_of(o.stage);
        for (int c = 0; c < width(o.kind); ++c) used.insert({dev, (o.offset + c) % blk.interval});
        if (o.kind == Kind::W) has_w.insert({o.stage, o.slot});
    }
    std::vector<std::tuple<int64_t, int, int>> need;  // (b_end, stage, slot)
    for (const auto& o : blk.ops)
        if (o.kind == Kind::B && !has_w.count({o.stage, o.slot})) need.emplace_back(o.offset + 1, o.stage, o.slot);
    std::sort(need.begin(), need.end());
    for (auto [b_end, stage, slot] : need) {
        int dev = blk.topo.device_of(stage);
        bool ok = false;
        for (int64_t cell = b_end; cell < b_end + blk.interval; ++cell) {
            if (used.insert({dev, cell % blk.interval}).second) {
                blk.ops.push_back({stage, Kind::W, slot, cell});
                ok = true;
                break;
            }
        }
        if (!ok) return false;
    }
    return true;
}

// gallery.hpp:108-130.  F descends over devices 1..d (down edges), turns, and
// climbs back (up edges); B retraces the climb (down edges, mirrored) then the
// descent (up edges, mirrored).
Block v_block_edges(int d, const VEdges& e, int64_t interval) {
    Block blk;
    blk.topo = Topology::v_shape(d);
    blk.interval = interval;
    std::vector<int64_t> f(2 * d), b(2 * d);
    f[0] = 0;
    for (int i = 1; i < d; ++i) f[i] = f[i - 1] + e.down[i - 1];
    f[d] = f[d - 1] + e.t1;
    for (int i = d + 1; i < 2 * d; ++i) f[i] = f[i - 1] + e.up[i - d - 1];
    b[2 * d - 1] = f[2 * d - 1] + e.t2;
    for (int k = 1; k < d; ++k) b[2 * d - 1 - k] = b[2 * d - k] + e.down[k - 1];
    b[d - 1] = b[d] + e.t3;
    for (int l = 1; l < d; ++l) b[d - 1 - l] = b[d - l] + e.up[l - 1];
    for (int s = 1; s <= 2 * d; ++s) {
        blk.ops.push_back({s, Kind::F, 0, f[s - 1]});
        blk.ops.push_back({s, Kind::B, 0, b[s - 1]});
    }
    return blk;
}

// gallery.hpp:132-157: uniform chain spacings, the backward chains carrying
// their own spacings (db1 on the first B leg, db0 on the second).
Block v_block(int d, const VChain& c, int64_t interval) {
    VEdges e;
    e.down.assign(std::max(0, d - 1), c.df0);
    e.up.assign(std::max(0, d - 1), c.df1);
    e.t1 = c.t1;
    e.t2 = c.t2;
    e.t3 = c.t3;
    Block blk = v_block_edges(d, e, interval);
    int64_t head = 0;
    for (const auto& o : blk.ops)
        if (o.kind == Kind::F && o.stage == 2 * d) head = o.offset + c.t2;
    std::vector<int64_t> b(2 * d);
    b[2 * d - 1] = head;
    for (int k = 1; k < d; ++k) b[2 * d - 1 - k] = b[2 * d - k] + c.db1;
    b[d - 1] = b[d] + c.t3;
    for (int l = 1; l < d; ++l) b[d - 1 - l] = b[d - l] + c.db0;
    for (auto& o : blk.ops)
        if (o.kind == Kind::B) o.offset = b[o.stage - 1];
    return blk;
}

namespace {

Block finish_v(Block blk, const std::string& entry) {  // gallery.hpp:159-169
    if (!place_greedy_w(blk)) throw std::invalid_argument(entry + ": no free residue left for W");
    if (auto v = first_block_violation(blk)) throw std::invalid_argument(entry + ": " + *v);
    if (auto c = residue_clash(blk))
        throw std::invalid_argument(entry + ": repeat clash on device " + std::to_string(c->first));
    return blk;
}

Block straight_block(int d, int64_t interval, const std::function<void(Block&, int)>& per_stage) {
    Block blk;
    blk.topo = Topology::straight(d);
    blk.interval = interval;
    for (int i = 1; i <= d; ++i) per_stage(blk, i);
    return blk;
}

// straight-pipeline entries with a fused/split backward chain at spacing 2
// whose head sits at `x` (gallery.hpp:175-239)
Block chain_block(int d, int64_t x, bool split) {
    return straight_block(d, 3, [&](Block& b, int i) {
        b.ops.push_back({i, Kind::F, 0, i - 1});
        int64_t at = x + 2LL * (d - i);
        if (split) {
            b.ops.push_back({i, Kind::B, 0, at});
            b.ops.push_back({i, Kind::W, 0, at + 1});
        } else {
            b.ops.push_back({i, Kind::BW, 0, at});
        }
    });
}

}  // namespace

std::vector<std::string> gallery_names() {  // gallery.hpp:474-497 listing order
    return {"1f1b", "eager-1f1b", "gpipe", "gems", "chimera", "interleaved-1f1b", "interleaved-1f1b-uniform",
            "interleaved-low-mem", "zb-h1", "zb-h2", "1f1b-v", "zb-2-3", "v-min", "v-half", "v-zb"};
}

namespace {

void put(Block& b, int stage, Kind k, int slot, int64_t at) { b.ops.push_back({stage, k, slot, at}); }

// smallest interval >= 6 whose repetition is residue-clash free (gems / chimera, gallery.hpp:294-300,
// 318-324); gives up past the block span + 2
void smallest_clash_free_interval(Block& blk, int64_t span, const std::string& entry) {
    for (int64_t t = 6;; ++t) {
        blk.interval = t;
        if (!residue_clash(blk)) return;
        if (t > span + 2) throw std::invalid_argument(entry + ": no repeat interval found");
    }
}

// gallery.hpp:252-302: replica 0 in 1f1b shape; replica 1's forward chain, then its fused backward
// chain (reversed), each pass at the first free cell of its device at or after it is ready
Block gems_block(int d) {
    Block blk;
    blk.topo = Topology::twin(d);
    blk.mb_per_block = 2;
    std::set<std::pair<int, int64_t>> busy;
    auto occupy = [&](int stage, Kind k, int slot, int64_t at) {
        put(blk, stage, k, slot, at);
        for (int c = 0; c < width(k); ++c) busy.insert({blk.topo.device_of(stage), at + c});
    };
    for (int i = 1; i <= d; ++i) {
        occupy(i, Kind::F, 0, i - 1);
        occupy(i, Kind::BW, 0, d + 2LL * (d - i));
    }
    auto first_fit = [&](int stage, Kind k, int64_t ready) {
        const int dev = blk.topo.device_of(stage);
        int64_t at = ready;
        auto clear = [&] {
            for (int c = 0; c < width(k); ++c)
                if (busy.count({dev, at + c})) return false;
            return true;
        };
        while (!clear()) ++at;
        occupy(stage, k, 1, at);
        return at + width(k);
    };
    int64_t ready = 0;
    for (int s = d + 1; s <= 2 * d; ++s) ready = first_fit(s, Kind::F, ready);
    std::map<int, int64_t> f_end;
    for (const auto& o : blk.ops)
        if (o.slot == 1 && o.kind == Kind::F) f_end[o.stage] = o.offset + 1;
    ready = f_end[2 * d];
    for (int s = 2 * d; s >= d + 1; --s) ready = first_fit(s, Kind::BW, std::max(ready, f_end[s]));
    int64_t span = 0;
    for (const auto& o : blk.ops) span = std::max(span, o.offset + width(o.kind));
    smallest_clash_free_interval(blk, span, "gems");
    return blk;
}

Block chimera_block(int d) {  // gallery.hpp:306-326: two mirrored 1f1b half-pipelines
    if (d % 2 != 0) throw std::invalid_argument("chimera: device count must be even");
    Block blk;
    blk.topo = Topology::twin(d);
    blk.mb_per_block = 2;
    for (int i = 1; i <= d; ++i) {
        put(blk, i, Kind::F, 0, i - 1);
        put(blk, i, Kind::BW, 0, d + 2LL * (d - i));
    }
    for (int k = 1; k <= d; ++k) {
        put(blk, d + k, Kind::F, 1, k - 1);
        put(blk, d + k, Kind::BW, 1, d + 2LL * (d - k));
    }
    smallest_clash_free_interval(blk, 3LL * d, "chimera");
    return blk;
}

// gallery.hpp:328-349: depth-2 round robin; instance j starts at 6d*(j div d) + 3*(j mod d)
Build interleaved_classic(int d) {
    Build b;
    b.name = "interleaved-1f1b";
    b.block.topo = Topology::looped(d, 2);
    b.block.interval = 6LL * d;
    for (int i = 1; i <= d; ++i) {
        put(b.block, i, Kind::F, 0, i - 1);
        put(b.block, d + i, Kind::F, 0, 3LL * d + i - 1);
        put(b.block, d + i, Kind::BW, 0, 6LL * d - 2 * i);
        put(b.block, i, Kind::BW, 0, 9LL * d - 2 * i);
    }
    const int64_t dd = d;
    b.explicit_starts = [dd](int n) {
        std::vector<int64_t> st(size_t(std::max(n, 0)));
        for (int j = 0; j < n; ++j) st[size_t(j)] = 6 * dd * (j / dd) + 3 * (j % dd);
        return st;
    };
    return b;
}

// gallery.hpp:353-386: interval 6; second-chunk forward chain from f2, the second chunk's fused
// backward head y (first cell with (y + 2d) mod 6 in {0, 3}) and the first chunk's head z (the other
// class of the two)
Block interleaved_interval6(int d, int64_t f2) {
    Block blk;
    blk.topo = Topology::looped(d, 2);
    blk.interval = 6;
    const int64_t two_d = 2LL * d;
    int64_t y = f2 + d;
    while ((y + two_d) % 6 != 0 && (y + two_d) % 6 != 3) ++y;
    const int64_t want = ((3 - (y + two_d) % 6) % 6 + 6) % 6;
    int64_t z = y + two_d;
    while ((z + two_d) % 6 != want) ++z;
    for (int i = 1; i <= d; ++i) {
        put(blk, i, Kind::F, 0, i - 1);
        put(blk, d + i, Kind::F, 0, f2 + i - 1);
        put(blk, d + i, Kind::BW, 0, y + 2LL * (d - i));
        put(blk, i, Kind::BW, 0, z + 2LL * (d - i));
    }
    return blk;
}
int64_t first_at_or_after_3_mod_6(int64_t x) {
    while (x % 6 != 3) ++x;
    return x;
}

// gallery.hpp:390-429: V placement, fused backward; the first (lifespan-sum, then lexicographic)
// offset tuple whose block repeats clash-free and validates
Block one_f_one_b_v_block(int d) {
    struct Cand {
        int64_t key[8];  // sum, df0, df1, db1, db0, t1, t2, t3
    };
    std::vector<Cand> cands;
    for (int64_t a = 1; a <= 4; ++a)
        for (int64_t b = 1; b <= 4; ++b)
            for (int64_t c = 2; c <= 5; ++c)
                for (int64_t e = 2; e <= 5; ++e)
                    for (int64_t t1 = 1; t1 <= 6; ++t1)
                        for (int64_t t2 = 1; t2 <= 6; ++t2)
                            for (int64_t t3 = 2; t3 <= 7; ++t3)
                                cands.push_back({{a + b + c + e + t1 + t2 + t3, a, b, c, e, t1, t2, t3}});
    std::stable_sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {
        return std::lexicographical_compare(x.key, x.key + 8, y.key, y.key + 8);
    });
    for (const Cand& cd : cands) {
        const int64_t df0 = cd.key[1], df1 = cd.key[2], db1 = cd.key[3], db0 = cd.key[4];
        const int64_t t1 = cd.key[5], t2 = cd.key[6], t3 = cd.key[7];
        Block blk;
        blk.topo = Topology::v_shape(d);
        blk.interval = 6;
        std::vector<int64_t> f(size_t(2 * d)), bw(size_t(2 * d));
        for (int i = 0; i < d; ++i) f[size_t(i)] = i * df0;                      // down leg
        f[size_t(d)] = f[size_t(d - 1)] + t1;                                     // turn
        for (int k = d + 1; k < 2 * d; ++k) f[size_t(k)] = f[size_t(k - 1)] + df1; // up leg
        bw[size_t(2 * d - 1)] = f[size_t(2 * d - 1)] + t2;                       // loss turn-around
        for (int k = 2 * d - 2; k >= d; --k) bw[size_t(k)] = bw[size_t(k + 1)] + db1;
        bw[size_t(d - 1)] = bw[size_t(d)] + t3;
        for (int k = d - 2; k >= 0; --k) bw[size_t(k)] = bw[size_t(k + 1)] + db0;
        for (int s = 1; s <= 2 * d; ++s) {
            put(blk, s, Kind::F, 0, f[size_t(s - 1)]);
            put(blk, s, Kind::BW, 0, bw[size_t(s - 1)]);
        }
        if (residue_clash(blk)) continue;
        if (first_block_violation(blk)) continue;
        return blk;
    }
    throw std::invalid_argument("1f1b-v: no valid offsets in search range");
}

// gallery.hpp:241-256: two microbatches per block, backward chains at spacing 1, greedy W
Block zb_2_3_block(int d) {
    Block blk;
    blk.topo = Topology::straight(d);
    blk.interval = 6;
    blk.mb_per_block = 2;
    for (int i = 1; i <= d; ++i) {
        put(blk, i, Kind::F, 0, i - 1);
        put(blk, i, Kind::B, 0, 2LL * d - i);
        put(blk, i, Kind::F, 1, i + 1);
        put(blk, i, Kind::B, 1, 2LL * d + 2 - i);
    }
    if (!place_greedy_w(blk)) throw std::invalid_argument("zb-2-3: W placement failed");
    return blk;
}

}  // namespace

// gallery.hpp:499-557: all 15 entries.  The executor runs every single-route
// topology (straight, V, looped); gems / chimera (twin routes over replicated
// weights) are generated and analysed but rejected by the executor.
Build build_entry(const std::string& name, int d, const std::map<std::string, int64_t>& params) {
    if (d < 1) throw std::invalid_argument("device count must be positive");
    for (const auto& kv : params)
        if (kv.first != "eagerness" && kv.first != "horizon")
            throw std::invalid_argument("unknown parameter: " + kv.first);
    auto param = [&](const char* k, int64_t dflt) {
        auto it = params.find(k);
        return it == params.end() ? dflt : it->second;
    };
    Build b;
    b.name = name;
    auto need_two = [&] {
        if (d < 2) throw std::invalid_argument(name + ": needs d >= 2");
    };
    if (name == "1f1b") {
        b.block = chain_block(d, d, false);  // BW(i) @ 3d-2i
    } else if (name == "eager-1f1b") {
        int64_t k = param("eagerness", d - 1);
        if (k < 0 || k > d - 1) throw std::invalid_argument("eager-1f1b: eagerness must be in [0, d-1]");
        b.block = chain_block(d, d + 3 * k, false);
    } else if (name == "gpipe") {
        int64_t h = param("horizon", 4LL * d);
        if (h < 1) throw std::invalid_argument("gpipe: horizon must be positive");
        b.block = chain_block(d, d + 3 * (h - 1), false);
    } else if (name == "zb-h1") {
        b.block = chain_block(d, d, true);  // B(i) @ 3d-2i, W right after
    } else if (name == "zb-h2") {
        b.block = chain_block(d, 4LL * d, true);
    } else if (name == "v-min") {
        need_two();
        VChain c;  // gallery.hpp:433-440
        c.t2 = (d % 3 == 0) ? 3 : 1;
        b.block = finish_v(v_block(d, c), "v-min");
    } else if (name == "v-half") {
        need_two();
        VChain c;  // gallery.hpp:442-452
        c.df0 = 2; c.df1 = 1; c.db1 = 2; c.db0 = 1;
        c.t1 = 2;
        c.t2 = (d % 2 == 0) ? 4 : 1;
        b.block = finish_v(v_block(d, c), "v-half");
    } else if (name == "v-zb") {
        need_two();
        VChain c;  // gallery.hpp:454-464
        c.df0 = 4; c.df1 = 2; c.db1 = 4; c.db0 = 2;
        b.block = finish_v(v_block(d, c), "v-zb");
    } else if (name == "gems") {
        b.block = gems_block(d);
        b.replicated_weights = true;
    } else if (name == "chimera") {
        b.block = chimera_block(d);
        b.replicated_weights = true;
    } else if (name == "interleaved-1f1b") {
        need_two();
        b = interleaved_classic(d);
    } else if (name == "interleaved-1f1b-uniform") {
        need_two();
        b.block = interleaved_interval6(d, first_at_or_after_3_mod_6(3LL * d));
    } else if (name == "interleaved-low-mem") {
        need_two();
        b.block = interleaved_interval6(d, first_at_or_after_3_mod_6(d));
    } else if (name == "1f1b-v") {
        need_two();
        b.block = one_f_one_b_v_block(d);
    } else if (name == "zb-2-3") {
        b.block = zb_2_3_block(d);
    } else {
        throw std::invalid_argument("unknown gallery entry: " + name);
    }
    return b;
}

// ---------------------------------------------------------------- assembly
std::string Collision::str() const {
    return "collision on device " + std::to_string(device) + " at cell " + std::to_string(cell) + ": " +
           op_str(first) + " vs " + op_str(second);
}

// assemble.hpp:85-128
Grid repeat(const Block& blk, const std::vector<int64_t>* starts, int instances, std::optional<Collision>* col) {
    if (instances < 1) throw std::invalid_argument("repeat: need at least one instance");
    if (starts && int(starts->size()) < instances)
        throw std::invalid_argument("repeat: explicit pattern has too few starts");
    Grid g;
    g.topo = blk.topo;
    g.microbatches = instances * blk.mb_per_block;
    g.ops.reserve(blk.ops.size() * size_t(instances));
    for (int j = 0; j < instances; ++j) {
        int64_t base = starts ? (*starts)[j] : j * blk.interval;
        for (const auto& o : blk.ops)
            g.ops.push_back({blk.topo.device_of(o.stage), o.stage, o.kind, j * blk.mb_per_block + o.slot,
                             base + o.offset, int64_t(width(o.kind))});
    }
    std::optional<Collision> best;
    std::map<std::pair<int, int64_t>, size_t> cells;
    for (size_t i = 0; i < g.ops.size(); ++i) {
        const auto& o = g.ops[i];
        for (int64_t c = o.start; c < o.end(); ++c) {
            auto [it, fresh] = cells.insert({{o.device, c}, i});
            if (!fresh && (!best || std::tie(o.device, c) < std::tie(best->device, best->cell)))
                best = Collision{o.device, c, g.ops[it->second], o};
        }
    }
    if (col) *col = best;
    sort_canonical(g);
    return g;
}

template <typename T>
std::vector<std::string> validate_schedule(const Plan<T>& p) {  // assemble.hpp:138-183
    std::vector<std::string> probs;
    std::vector<std::vector<const Op<T>*>> per(size_t(p.topo.devices) + 1);
    for (const auto& o : p.ops) {
        if (o.device < 1 || o.device > p.topo.devices) {
            probs.push_back("device out of range: " + std::to_string(o.device));
            continue;
        }
        if (o.device != p.topo.device_of(o.stage))
            probs.push_back("stage " + std::to_string(o.stage) + " not placed on device " + std::to_string(o.device));
        per[o.device].push_back(&o);
    }
    for (int dev = 1; dev <= p.topo.devices; ++dev) {
        auto& v = per[dev];
        std::sort(v.begin(), v.end(), [](auto* a, auto* b) { return a->start < b->start; });
        for (size_t i = 1; i < v.size(); ++i)
            if (v[i]->start < v[i - 1]->end())
                probs.push_back("device " + std::to_string(dev) + " overlap at " +
                                std::to_string(static_cast<double>(v[i]->start)));
    }
    Lookup<T> look(p);
    for (const auto& o : p.ops) {
        std::vector<Ref> deps;
        try {
            deps = prerequisites(p.topo, o.stage, o.kind, o.mb);
        } catch (const std::invalid_argument& e) {
            probs.push_back(e.what());
            continue;
        }
        for (const Ref& d : deps) {
            auto i = look.find(d.stage, d.kind, d.mb);
            if (!i)
                probs.push_back("microbatch " + std::to_string(o.mb) + " misses " + kind_name(d.kind) + " of stage " +
                                std::to_string(d.stage));
            else if (p.ops[*i].end() > o.start)
                probs.push_back(std::string(kind_name(o.kind)) + "(stage " + std::to_string(o.stage) + ", microbatch " +
                                std::to_string(o.mb) + ") starts before its prerequisite ends");
        }
    }
    return probs;
}
template std::vector<std::string> validate_schedule(const Plan<int64_t>&);
template std::vector<std::string> validate_schedule(const Plan<double>&);

namespace {
// processing order shared by squeeze and simulate: (start, device, stage, mb)
template <typename T>
std::vector<size_t> time_order(const Plan<T>& p) {
    std::vector<size_t> ord(p.ops.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
        const auto &x = p.ops[a], &y = p.ops[b];
        return std::tie(x.start, x.device, x.stage, x.mb) < std::tie(y.start, y.device, y.stage, y.mb);
    });
    return ord;
}

std::vector<std::vector<size_t>> by_device_start(const Grid& g) {
    std::vector<std::vector<size_t>> v(size_t(g.topo.devices) + 1);
    for (size_t i = 0; i < g.ops.size(); ++i) v[g.ops[i].device].push_back(i);
    for (auto& dv : v)
        std::sort(dv.begin(), dv.end(), [&](size_t a, size_t b) { return g.ops[a].start < g.ops[b].start; });
    return v;
}

// peak of one device's allocation sweep with op `moved` shifted to `at`
// (assemble.hpp:236-260)
double peak_if_moved(const Grid& g, const std::vector<size_t>& dev_ops, size_t moved, int64_t at) {
    std::vector<std::tuple<int64_t, int, double>> ev;
    ev.reserve(dev_ops.size());
    for (size_t i : dev_ops) {
        const auto& o = g.ops[i];
        int64_t s = i == moved ? at : o.start;
        double m = g.topo.mem_of(o.stage);
        if (o.kind == Kind::F) ev.emplace_back(s, 1, m);
        if (o.kind == Kind::W || o.kind == Kind::BW) ev.emplace_back(s + o.dur, 0, -m);
    }
    std::sort(ev.begin(), ev.end(), [](const auto& a, const auto& b) {
        return std::tie(std::get<0>(a), std::get<1>(a)) < std::tie(std::get<0>(b), std::get<1>(b));
    });
    double cur = 0, peak = 0;
    for (const auto& e : ev) peak = std::max(peak, cur += std::get<2>(e));
    return peak;
}
}  // namespace

// assemble.hpp:188-216: earliest start keeping each device's order.
Grid squeeze(const Grid& in) {
    Grid g = in;
    Lookup<int64_t> look(g);
    std::vector<int64_t> at(g.ops.size(), 0);
    std::vector<char> done(g.ops.size(), 0);
    std::vector<int64_t> free_at(size_t(g.topo.devices) + 1, 0);
    for (size_t i : time_order(g)) {
        const auto& o = g.ops[i];
        int64_t t = free_at[o.device];
        for (size_t d : look.deps(g, o)) {
            if (!done[d]) throw std::invalid_argument("squeeze: prerequisite not ordered first");
            t = std::max(t, at[d] + g.ops[d].dur);
        }
        at[i] = t;
        done[i] = 1;
        free_at[o.device] = t + o.dur;
    }
    for (size_t i = 0; i < g.ops.size(); ++i) g.ops[i].start = at[i];
    sort_canonical(g);
    return g;
}

// assemble.hpp:269-397 (warm-up hole filling under the pre-reorder per-device
// peak, then cool-down W recycling).  The exact tie-breaks matter: they define
// the op order the executor runs.
Grid reorder(const Grid& in) {
    Grid g = in;
    const std::vector<double> cap = exact_peak(g);
    Lookup<int64_t> look(g);
    std::vector<std::vector<size_t>> deps(g.ops.size());
    for (size_t i = 0; i < g.ops.size(); ++i) deps[i] = look.deps(g, g.ops[i]);
    auto ready = [&](size_t i) {
        int64_t e = 0;
        for (size_t d : deps[i]) e = std::max(e, g.ops[d].end());
        return e;
    };

    for (bool moved = true; moved;) {
        moved = false;
        auto views = by_device_start(g);
        for (int dev = 1; dev <= g.topo.devices; ++dev) {
            const auto& dv = views[dev];
            const size_t n = dv.size();
            std::vector<char> relocated(n, 0);
            std::vector<int64_t> floor_at(n, 0);
            int64_t cursor = 0;
            for (size_t vi = 0; vi < n; ++vi) {
                if (relocated[vi]) continue;
                const int64_t gap_end = g.ops[dv[vi]].start;
                while (cursor < gap_end) {
                    size_t pick = n;
                    int64_t pick_at = 0;
                    for (size_t vj = vi; vj < n; ++vj) {
                        if (relocated[vj]) continue;
                        int64_t t = std::max({cursor, ready(dv[vj]), floor_at[vj]});
                        if (t + g.ops[dv[vj]].dur > gap_end) continue;
                        if (pick == n || t < pick_at) {
                            pick = vj;
                            pick_at = t;
                        }
                    }
                    if (pick == n) break;
                    GridOp& c = g.ops[dv[pick]];
                    if (c.kind == Kind::F && peak_if_moved(g, dv, dv[pick], pick_at) > cap[dev - 1] + 1e-9) {
                        floor_at[pick] = pick_at + 1;
                        continue;
                    }
                    c.start = pick_at;
                    relocated[pick] = 1;
                    moved = true;
                    cursor = pick_at + c.dur;
                }
                cursor = std::max(cursor, g.ops[dv[vi]].end());
            }
        }
    }

    std::vector<int64_t> last_f(size_t(g.topo.devices) + 1, -1);
    for (const auto& o : g.ops)
        if (o.kind == Kind::F) last_f[o.device] = std::max(last_f[o.device], o.end());
    Grid kept;
    kept.topo = g.topo;
    kept.microbatches = g.microbatches;
    std::vector<GridOp> tail_w;
    for (const auto& o : g.ops) {
        if (o.kind == Kind::W && last_f[o.device] >= 0 && o.start >= last_f[o.device])
            tail_w.push_back(o);
        else
            kept.ops.push_back(o);
    }
    if (tail_w.empty()) {
        sort_canonical(g);
        return g;
    }
    Grid packed = squeeze(kept);
    Lookup<int64_t> plook(packed);
    std::vector<std::vector<std::pair<int64_t, GridOp>>> pending(size_t(packed.topo.devices) + 1);
    for (const auto& w : tail_w) {
        auto bi = plook.find(w.stage, Kind::B, w.mb);
        if (!bi) throw std::invalid_argument("reorder: W without matching B");
        pending[w.device].push_back({packed.ops[*bi].end(), w});
    }
    auto views = by_device_start(packed);
    std::vector<GridOp> placed;
    for (int dev = 1; dev <= packed.topo.devices; ++dev) {
        auto& ps = pending[dev];
        std::sort(ps.begin(), ps.end(), [](const auto& a, const auto& b) {
            return std::tie(a.first, a.second.mb) < std::tie(b.first, b.second.mb);
        });
        size_t next = 0;
        int64_t cursor = 0, dev_end = 0;
        for (size_t i : views[dev]) {
            const auto& o = packed.ops[i];
            while (next < ps.size() && cursor < o.start) {
                if (ps[next].first <= cursor) {  // head-of-line W fits here
                    GridOp w = ps[next++].second;
                    w.start = cursor;
                    placed.push_back(w);
                }
                ++cursor;
            }
            cursor = std::max(cursor, o.end());
            dev_end = std::max(dev_end, o.end());
        }
        cursor = std::max(cursor, dev_end);
        for (; next < ps.size(); ++next) {
            GridOp w = ps[next].second;
            w.start = std::max(cursor, ps[next].first);
            cursor = w.start + 1;
            placed.push_back(w);
        }
    }
    packed.ops.insert(packed.ops.end(), placed.begin(), placed.end());
    sort_canonical(packed);
    return packed;
}

Grid assemble(const Build& b, int n, bool do_squeeze, bool do_reorder) {  // assemble.hpp:405-419
    const Block& blk = b.block;
    if (n < 1) throw std::invalid_argument("assemble: need at least one microbatch");
    if (n % blk.mb_per_block != 0)
        throw std::invalid_argument("assemble: microbatch count must be a multiple of " +
                                    std::to_string(blk.mb_per_block));
    int inst = n / blk.mb_per_block;
    std::vector<int64_t> starts;
    if (b.explicit_starts) starts = b.explicit_starts(inst);
    std::optional<Collision> col;
    Grid g = repeat(blk, b.explicit_starts ? &starts : nullptr, inst, &col);
    if (col) throw std::invalid_argument("assemble: " + col->str());
    if (do_squeeze) g = squeeze(g);
    if (do_reorder) g = reorder(g);
    return g;
}

// ---------------------------------------------------------------- memory
// memory.hpp:63-91: +m at F start, -m at W/BW end, releases first on ties.
template <typename T>
std::vector<double> exact_peak(const Plan<T>& p) {
    struct Ev {
        T t;
        int ord;
        int dev;
        double d;
    };
    std::vector<Ev> ev;
    ev.reserve(p.ops.size());
    for (const auto& o : p.ops) {
        double m = p.topo.mem_of(o.stage);
        if (o.kind == Kind::F) ev.push_back({o.start, 1, o.device, m});
        if (o.kind == Kind::W || o.kind == Kind::BW) ev.push_back({o.end(), 0, o.device, -m});
    }
    std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) { return std::tie(a.t, a.ord) < std::tie(b.t, b.ord); });
    std::vector<double> peak(size_t(p.topo.devices), 0.0), cur(size_t(p.topo.devices), 0.0);
    for (const auto& e : ev) {
        cur[e.dev - 1] += e.d;
        peak[e.dev - 1] = std::max(peak[e.dev - 1], cur[e.dev - 1]);
    }
    return peak;
}
template std::vector<double> exact_peak(const Plan<int64_t>&);
template std::vector<double> exact_peak(const Plan<double>&);

template <typename T>
std::vector<TraceRow> memory_trace(const Plan<T>& p) {  // memory.hpp:142-169
    struct Ev {
        T t;
        int ord;
        int dev;
        double d;
    };
    std::vector<Ev> ev;
    for (const auto& o : p.ops) {
        double m = p.topo.mem_of(o.stage);
        if (o.kind == Kind::F) ev.push_back({o.start, 1, o.device, m});
        if (o.kind == Kind::W || o.kind == Kind::BW) ev.push_back({o.end(), 0, o.device, -m});
    }
    std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
        return std::tie(a.t, a.ord, a.dev) < std::tie(b.t, b.ord, b.dev);
    });
    std::vector<double> cur(size_t(p.topo.devices), 0.0);
    std::vector<TraceRow> rows;
    for (size_t i = 0; i < ev.size(); ++i) {
        cur[ev[i].dev - 1] += ev[i].d;
        bool last = i + 1 == ev.size() || ev[i + 1].t != ev[i].t || ev[i + 1].dev != ev[i].dev;
        if (last) rows.push_back({double(ev[i].t), ev[i].dev, cur[ev[i].dev - 1]});
    }
    return rows;
}
template std::vector<TraceRow> memory_trace(const Plan<int64_t>&);
template std::vector<TraceRow> memory_trace(const Plan<double>&);

namespace {
struct Span {
    int stage;
    int64_t f_start = 0, release = 0;
};
std::vector<Span> spans_of(const Block& blk) {  // memory.hpp:20-34
    std::map<std::pair<int, int>, Span> m;
    for (const auto& o : blk.ops) {
        auto& s = m[{o.stage, o.slot}];
        s.stage = o.stage;
        if (o.kind == Kind::F) s.f_start = o.offset;
        if (o.kind == Kind::W || o.kind == Kind::BW) s.release = o.offset + width(o.kind);
    }
    std::vector<Span> out;
    for (auto& kv : m) out.push_back(kv.second);
    return out;
}
}  // namespace

std::vector<double> peak_bound(const Block& blk) {  // memory.hpp:48-59
    if (blk.interval <= 0) throw std::invalid_argument("peak_bound: interval must be positive");
    std::vector<double> out(size_t(blk.topo.devices), 0.0);
    for (const auto& s : spans_of(blk)) {
        int64_t len = s.release - s.f_start;
        out[blk.topo.device_of(s.stage) - 1] += double((len + blk.interval - 1) / blk.interval) * blk.topo.mem_of(s.stage);
    }
    return out;
}

std::vector<double> steady_peak(const Block& blk) {  // memory.hpp:97-131
    if (blk.interval <= 0) throw std::invalid_argument("steady_peak: interval must be positive");
    auto sp = spans_of(blk);
    int64_t periods = 2;
    for (const auto& s : sp) periods = std::max(periods, (s.release - s.f_start + blk.interval - 1) / blk.interval + 2);
    Grid g;
    g.topo = blk.topo;
    // an F at f_start and a unit W ending at release reproduce the same events
    for (const auto& s : sp)
        for (int64_t j = 0; j < periods; ++j) {
            int dev = blk.topo.device_of(s.stage);
            g.ops.push_back({dev, s.stage, Kind::F, 0, s.f_start + j * blk.interval, 1});
            g.ops.push_back({dev, s.stage, Kind::W, 0, s.release + j * blk.interval - 1, 1});
        }
    return exact_peak(g);
}

// ---------------------------------------------------------------- replay
SimResult account(const Timed& t) {  // simulate.hpp:257-282
    SimResult r;
    const int d = t.topo.devices;
    r.busy.assign(size_t(d), 0.0);
    std::vector<double> first(size_t(d), 0.0), last(size_t(d), 0.0);
    std::vector<bool> seen(size_t(d), false);
    for (const auto& o : t.ops) {
        r.makespan = std::max(r.makespan, o.end());
        size_t k = size_t(o.device - 1);
        r.busy[k] += o.dur;
        if (!seen[k]) {
            first[k] = o.start;
            last[k] = o.end();
            seen[k] = true;
        } else {
            first[k] = std::min(first[k], o.start);
            last[k] = std::max(last[k], o.end());
        }
    }
    r.idle_total.assign(size_t(d), 0.0);
    r.idle_span.assign(size_t(d), 0.0);
    double total = 0;
    for (int k = 0; k < d; ++k) {
        r.idle_total[k] = r.makespan - r.busy[k];
        r.idle_span[k] = seen[k] ? (last[k] - first[k]) - r.busy[k] : 0.0;
        total += r.busy[k];
    }
    r.bubble_rate = r.makespan > 0 ? 1.0 - total / (d * r.makespan) : 0.0;
    r.peak = exact_peak(t);
    r.schedule = t;
    sort_canonical(r.schedule);
    return r;
}

// simulate.hpp:22-86: order-preserving replay; a cross-device prerequisite
// adds the hop latency.
SimResult simulate(const Grid& g, const Profile& prof) {
    std::vector<double> dur(g.ops.size());
    for (size_t i = 0; i < g.ops.size(); ++i) dur[i] = prof.of(g.ops[i].kind);
    return replay(g, dur, prof.comm);
}

// simulate.hpp:44-56 with one duration per pass (canonical order) instead of
// one per kind: every pass starts when its device is free and its
// prerequisites have ended (+comm across devices), in grid start order.
SimResult replay(const Grid& g, const std::vector<double>& dur, double comm) {
    if (dur.size() != g.ops.size()) throw std::invalid_argument("replay: one duration per pass required");
    Timed t;
    t.topo = g.topo;
    t.microbatches = g.microbatches;
    t.ops.resize(g.ops.size());
    for (size_t i = 0; i < g.ops.size(); ++i) {
        const auto& o = g.ops[i];
        t.ops[i] = {o.device, o.stage, o.kind, o.mb, 0.0, dur[i]};
    }
    Lookup<int64_t> look(g);
    std::vector<double> free_at(size_t(g.topo.devices) + 1, 0.0);
    std::vector<char> done(g.ops.size(), 0);
    for (size_t i : time_order(g)) {
        const auto& o = g.ops[i];
        double at = free_at[o.device];
        for (size_t d : look.deps(g, o)) {
            if (!done[d]) throw std::invalid_argument("simulate: prerequisite not ordered first");
            double r = t.ops[d].end();
            if (g.ops[d].device != o.device) r += comm;
            at = std::max(at, r);
        }
        t.ops[i].start = at;
        done[i] = 1;
        free_at[o.device] = at + t.ops[i].dur;
    }
    return account(t);
}

}  // namespace vsched
