#include "plan.hpp"

#include <algorithm>
#include <map>
#include <stdexcept>
#include <tuple>

namespace pbx {

using vsched::Kind;

ExecPlan make_plan(const vsched::Grid& g) {
    ExecPlan p;
    p.topo = g.topo;
    p.microbatches = g.microbatches;
    const int D = g.topo.devices, S = g.topo.num_stages;
    // single-route topologies (straight, V, looped) and the two-route twin of gems / chimera
    // (model.hpp:93-107: route 0 = stages 1..d, route 1 = stages d+1..2d over replicated weights)
    const bool twin = g.topo.routes.size() == 2 && g.topo.routes[0] == vsched::Topology::iota(1, S / 2) &&
                      g.topo.routes[1] == vsched::Topology::iota(S / 2 + 1, S);
    if (!g.topo.default_routes() && !twin)
        throw std::invalid_argument("executor: only single-route and twin (gems / chimera) topologies are supported");
    for (int s = 1; s <= S; ++s)
        if (g.topo.mem_of(s) != 1.0) throw std::invalid_argument("executor: stage_mem must be 1.0 for every stage");

    p.ops.resize(g.ops.size());
    std::map<std::tuple<int, int, int>, int> at;  // (stage, kind-class, mb) -> op; B and BW share class 1
    for (size_t i = 0; i < g.ops.size(); ++i) {
        p.ops[i].op = g.ops[i];
        const auto& o = g.ops[i];
        int cls = o.kind == Kind::F ? 0 : (o.kind == Kind::W ? 2 : 1);
        at[{o.stage, cls, o.mb}] = int(i);
    }
    p.dev_ops.assign(size_t(D) + 1, {});
    for (size_t i = 0; i < g.ops.size(); ++i) p.dev_ops[g.ops[i].device].push_back(int(i));
    for (auto& v : p.dev_ops)
        std::sort(v.begin(), v.end(), [&](int a, int b) { return g.ops[a].start < g.ops[b].start; });

    // activation slots: allocated at F start, released at W/BW end, in op order (memory.hpp:61-62)
    p.slots.assign(size_t(D) + 1, 0);
    for (int d = 1; d <= D; ++d) {
        std::vector<int> free_by;  // slot -> op index that released it (-1 fresh)
        std::vector<bool> busy;
        std::map<std::pair<int, int>, int> slot_of;
        for (int i : p.dev_ops[d]) {
            const auto& o = g.ops[i];
            if (o.kind == Kind::F) {
                int k = 0;
                while (k < int(busy.size()) && busy[k]) ++k;
                if (k == int(busy.size())) {
                    busy.push_back(false);
                    free_by.push_back(-1);
                }
                busy[k] = true;
                p.ops[i].slot = k;
                p.ops[i].free_op = free_by[k];
                slot_of[{o.stage, o.mb}] = k;
            } else {
                auto it = slot_of.find({o.stage, o.mb});
                if (it == slot_of.end()) throw std::invalid_argument("executor: backward pass before its forward");
                p.ops[i].slot = it->second;
                if (o.kind == Kind::W || o.kind == Kind::BW) {
                    busy[it->second] = false;
                    free_by[it->second] = i;
                }
            }
        }
        p.slots[d] = int(busy.size());
    }

    // messages: F(s)->F(next stage on the microbatch's route) and B(s)->B(previous); consumer found by identity
    auto route_end = [&](int stage, int mb, bool want_last) {
        const auto& r = g.topo.route_for(mb);
        return want_last ? stage == r.back() : stage == r.front();
    };
    auto find = [&](int stage, int cls, int mb) {
        auto it = at.find({stage, cls, mb});
        if (it == at.end()) throw std::invalid_argument("executor: schedule misses a pass on the route");
        return it->second;
    };
    p.outboxes.assign(size_t(D) + 1, 0);
    p.uses.assign(size_t(D) + 1, {});
    p.last_use.assign(size_t(D) + 1, {});
    for (int d = 1; d <= D; ++d) {
        std::vector<int64_t> busy_until;  // consumer start of the last message in each outbox slot
        std::vector<int> last_msg;
        for (int i : p.dev_ops[d]) {
            const auto& o = g.ops[i];
            int cons = -1;
            if (o.kind == Kind::F && !route_end(o.stage, o.mb, true)) cons = find(o.stage + 1, 0, o.mb);
            if ((o.kind == Kind::B || o.kind == Kind::BW) && !route_end(o.stage, o.mb, false))
                cons = find(o.stage - 1, 1, o.mb);
            if (cons < 0) continue;
            int k = 0;
            while (k < int(busy_until.size()) && busy_until[k] > o.start) ++k;
            if (k == int(busy_until.size())) {
                busy_until.push_back(0);
                last_msg.push_back(-1);
                p.uses[d].push_back(0);
            }
            Msg m;
            m.src_dev = d;
            m.dst_dev = g.ops[cons].device;
            m.producer = i;
            m.consumer = cons;
            m.outbox = k;
            m.gen = ++p.uses[d][k];
            if (last_msg[k] >= 0) {
                m.prev_msg = last_msg[k];
                m.prev_gen = p.msgs[last_msg[k]].gen;
                m.prev_remote = !p.msgs[last_msg[k]].local();
            }
            busy_until[k] = g.ops[cons].start;
            last_msg[k] = int(p.msgs.size());
            p.ops[i].out_msg = int(p.msgs.size());
            p.ops[cons].in_msg = int(p.msgs.size());
            p.msgs.push_back(m);
        }
        p.outboxes[d] = int(busy_until.size());
        p.last_use[d] = last_msg;
        p.max_outbox = std::max(p.max_outbox, p.outboxes[d]);
    }
    // across steps, the first use of a slot follows the previous step's last use
    for (auto& m : p.msgs) {
        if (m.prev_gen == 0) {
            const Msg& last = p.msgs[p.last_use[m.src_dev][m.outbox]];
            m.prev_remote = !last.local();
            m.prev_msg = p.last_use[m.src_dev][m.outbox];
            m.prev_cross_step = true;
        }
    }
    return p;
}

}  // namespace pbx
