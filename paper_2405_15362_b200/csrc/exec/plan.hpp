// Execution plan derived from a GridSchedule: every device's op list in grid
// order, the lifespan-bounded activation slot of each (stage, microbatch),
// and the stage-boundary messages with their outbox slots and generations.
//
// Everything here is a pure function of the schedule, so every rank computes
// the same plan and knows where its peers' messages live without talking.
#pragma once
#include <cstdint>
#include <vector>

#include "schedule/vsched.hpp"

namespace pbx {

struct Msg {
    int src_dev = 0, dst_dev = 0;  // 1-based devices
    int producer = -1;             // op index (global, canonical order)
    int consumer = -1;
    int outbox = -1;               // outbox slot on src_dev
    uint32_t gen = 0;              // 1-based use count of that outbox slot within a step
    bool prev_remote = false;      // previous occupant of the slot was consumed on another device
    uint32_t prev_gen = 0;         // generation of the previous occupant (0 = none in this step)
    int prev_msg = -1;             // message index of the previous occupant of the outbox slot
    bool prev_cross_step = false;  // ... which is the last use of the slot in the previous step
    bool local() const { return src_dev == dst_dev; }
};

struct PlanOp {
    vsched::GridOp op;
    int slot = -1;      // activation slot on its device for (stage, mb)
    int out_msg = -1;   // index into msgs produced by this op
    int in_msg = -1;    // message this op consumes
    int free_op = -1;   // for F: the W/BW op that last released `slot` on this device (WAR), else -1
};

struct ExecPlan {
    vsched::Topology topo;
    int microbatches = 0;
    std::vector<PlanOp> ops;                  // canonical order
    std::vector<std::vector<int>> dev_ops;    // [device] -> op indices in grid order
    std::vector<Msg> msgs;
    std::vector<int> slots;                   // [device] activation slots used (= exact_peak)
    std::vector<int> outboxes;                // [device] outbox slots used
    std::vector<std::vector<uint32_t>> uses;  // [device][outbox] generations per step
    std::vector<std::vector<int>> last_use;   // [device][outbox] msg index of the last use in a step
    int max_outbox = 0;
};

ExecPlan make_plan(const vsched::Grid& g);

}  // namespace pbx
