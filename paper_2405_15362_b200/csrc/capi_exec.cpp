// C-ABI for the executor (include/pipeblock_b200.h, "executor").
#include <algorithm>
#include <cstring>
#include <vector>

#include "capi_common.hpp"
#include "exec/executor.hpp"

struct pb_exec {
    pbx::Exec* e;
};

namespace {
pbx::Exec& X(pb_exec* h) {
    if (!h || !h->e) throw std::invalid_argument("null executor");
    return *h->e;
}
}  // namespace

extern "C" int pb_exec_create(const pb_model_cfg* cfg, const pb_schedule* plan, int32_t device, int32_t cuda_device,
                              pb_exec** out) {
    return pbx::guard([&] {
        if (!cfg || !plan || !out) throw std::invalid_argument("null argument");
        auto* e = new pbx::Exec(*cfg, pbx::schedule_grid(plan), device, cuda_device);
        e->timeline = (cfg->flags & PB_FLAG_TIMELINE) != 0;
        e->serial = (cfg->flags & PB_FLAG_SERIAL) != 0;
        e->gemm_timing = (cfg->flags & PB_FLAG_GEMM_TIMING) != 0;
        e->kernel_timing = (cfg->flags & PB_FLAG_KERNEL_TIMING) != 0;
        e->isolate = (cfg->flags & PB_FLAG_ISOLATE) != 0;
        e->solo = (cfg->flags & PB_FLAG_SOLO) != 0;
        if (e->plan.topo.devices == 1) e->connect_local({e}, nullptr);
        *out = new pb_exec{e};
    });
}

extern "C" int pb_exec_connect_local(pb_exec* const* all, int32_t n) {
    return pbx::guard([&] {
        std::vector<pbx::Exec*> v;
        for (int i = 0; i < n; ++i) v.push_back(&X(all[i]));
        std::sort(v.begin(), v.end(), [](auto* a, auto* b) { return a->dev < b->dev; });
        auto grp = pbx::make_group(v);
        for (auto* e : v) e->connect_local(v, grp);
    });
}

extern "C" int pb_exec_export(pb_exec* h, void* blob, size_t cap, size_t* len) {
    return pbx::guard([&] {
        size_t n = X(h).export_blob(blob, cap);
        if (len) *len = n;
    });
}

extern "C" int pb_exec_connect_ipc(pb_exec* h, const void* const* blobs, const size_t* lens, int32_t n) {
    return pbx::guard([&] {
        std::vector<std::pair<const void*, size_t>> v;
        for (int i = 0; i < n; ++i) v.push_back({blobs[i], lens[i]});
        X(h).connect_ipc(v);
    });
}

extern "C" int pb_exec_step(pb_exec* h, const int32_t* tokens, const int32_t* labels, int32_t on_host,
                            pb_timed_pass* timeline, size_t n, pb_exec_stats* stats) {
    return pbx::guard([&] {
        X(h).enqueue(tokens, labels, on_host != 0);
        X(h).finish(timeline, n, stats);
    });
}

extern "C" int pb_exec_step_async(pb_exec* h, const int32_t* tokens, const int32_t* labels, int32_t on_host) {
    return pbx::guard([&] { X(h).enqueue(tokens, labels, on_host != 0); });
}

extern "C" int pb_exec_sync(pb_exec* h, pb_timed_pass* timeline, size_t n, pb_exec_stats* stats) {
    return pbx::guard([&] { X(h).finish(timeline, n, stats); });
}

extern "C" int pb_exec_num_passes(const pb_exec* h, size_t* n) {
    return pbx::guard([&] {
        auto& e = X(const_cast<pb_exec*>(h));
        *n = e.plan.dev_ops[e.dev].size();
    });
}

extern "C" int pb_exec_set_flags(pb_exec* h, int32_t flags) {
    return pbx::guard([&] {
        auto& e = X(h);
        if (e.pending) throw pbx::StateError("set_flags while a step is in flight");
        e.timeline = (flags & PB_FLAG_TIMELINE) != 0;
        e.serial = (flags & PB_FLAG_SERIAL) != 0;
        e.gemm_timing = (flags & PB_FLAG_GEMM_TIMING) != 0;
        e.kernel_timing = (flags & PB_FLAG_KERNEL_TIMING) != 0;
        e.isolate = (flags & PB_FLAG_ISOLATE) != 0;
        e.solo = (flags & PB_FLAG_SOLO) != 0;
    });
}

extern "C" void* pb_exec_stream(pb_exec* h) { return (h && h->e) ? static_cast<void*>(h->e->cs) : nullptr; }

extern "C" int pb_exec_param_count(const pb_exec* h, int32_t* n) {
    return pbx::guard([&] { *n = int32_t(X(const_cast<pb_exec*>(h)).ptensors.size()); });
}

extern "C" int pb_exec_param_info(const pb_exec* h, int32_t i, char* name, size_t cap, int64_t* numel) {
    return pbx::guard([&] {
        auto& e = X(const_cast<pb_exec*>(h));
        if (i < 0 || i >= int(e.ptensors.size())) throw std::invalid_argument("param index out of range");
        const auto& t = e.ptensors[i];
        if (name) {
            if (cap < t.name.size() + 1) throw pbx::Space("name buffer too small");
            std::memcpy(name, t.name.c_str(), t.name.size() + 1);
        }
        if (numel) *numel = int64_t(t.numel);
    });
}

extern "C" int pb_exec_param_get(pb_exec* h, int32_t i, int32_t which, float* host) {
    return pbx::guard([&] {
        auto& e = X(h);
        if (i < 0 || i >= int(e.ptensors.size())) throw std::invalid_argument("param index out of range");
        const auto& t = e.ptensors[i];
        cudaSetDevice(e.cuda);
        cudaStreamSynchronize(e.cs);
        if (which == 0) {  // the bf16 weight the model computes with (masters rounded; gamma-folded copies aside)
            if (cudaMemcpy(host, e.master + t.off, t.numel * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
                throw pbx::CudaError("param copy failed");
            for (size_t k = 0; k < t.numel; ++k) host[k] = __bfloat162float(__float2bfloat16_rn(host[k]));
        } else {
            if (cudaMemcpy(host, (which == 1 ? e.grads : e.master) + t.off, t.numel * 4, cudaMemcpyDeviceToHost) !=
                cudaSuccess)
                throw pbx::CudaError("param copy failed");
        }
    });
}

extern "C" int pb_exec_param_set(pb_exec* h, int32_t i, const float* host) {
    return pbx::guard([&] {
        auto& e = X(h);
        if (i < 0 || i >= int(e.ptensors.size())) throw std::invalid_argument("param index out of range");
        const auto& t = e.ptensors[i];
        cudaSetDevice(e.cuda);
        cudaStreamSynchronize(e.cs);
        if (cudaMemcpy(e.master + t.off, host, t.numel * 4, cudaMemcpyHostToDevice) != cudaSuccess)
            throw pbx::CudaError("param copy failed");
        pbk::f32_to_bf16(e.master + t.off, e.wts + t.off, (t.numel + 3) / 4 * 4, e.cs);
        e.refold();
        cudaStreamSynchronize(e.cs);
    });
}

extern "C" int pb_exec_memory(pb_exec* h, pb_exec_memory_t* out) {
    return pbx::guard([&] {
        if (!out) throw std::invalid_argument("null argument");
        auto& e = X(h);
        auto get = [&](std::initializer_list<const char*> keys) {
            int64_t v = 0;
            for (const char* k : keys) {
                auto it = e.mem_alloc.find(k);
                if (it != e.mem_alloc.end()) v += int64_t(it->second);
            }
            return v;
        };
        *out = {};
        out->weights = get({"params"});
        out->grads = get({"grads", "folded grads"});
        out->optimizer = get({"adam"});
        out->activation_pool = get({"activation pool"});
        out->head_pool = get({"head pool"});
        out->transfer = get({"outbox", "flags"});
        out->executor_total = int64_t(e.mem_alloc_total);
        out->scratch = out->executor_total - out->weights - out->grads - out->optimizer - out->activation_pool -
                       out->head_pool - out->transfer;
        e.sample_device_memory();
        out->device_total = int64_t(e.mem_device_total);
        out->device_used_at_create = int64_t(e.mem_used_at_create);
        out->device_used_high = int64_t(e.mem_used_high);
    });
}

extern "C" int pb_exec_zero_grads(pb_exec* h) {
    return pbx::guard([&] {
        auto& e = X(h);
        cudaSetDevice(e.cuda);
        if (cudaMemsetAsync(e.grads, 0, e.n_params * 4, e.cs) != cudaSuccess) throw pbx::CudaError("memset failed");
        cudaStreamSynchronize(e.cs);
    });
}

extern "C" void pb_exec_destroy(pb_exec* h) {
    if (!h) return;
    delete h->e;
    delete h;
}

extern "C" int pb_exec_kernel_report(pb_exec* h, char* buf, size_t cap, size_t* len) {
    return pbx::guard([&] {
        const std::string& r = X(h).kernel_report;
        if (len) *len = r.size();
        if (!buf) return;
        if (cap < r.size() + 1) throw pbx::Space("report buffer too small");
        std::memcpy(buf, r.c_str(), r.size() + 1);
    });
}

// Host-side execution plan of one pipeline device (no GPU needed): what a rank
// runs, in grid order, and which peer messages it pulls / publishes.
#include "exec/plan.hpp"
extern "C" int pb_plan_device(const pb_schedule* s, int32_t device, pb_plan_op* out, size_t cap, size_t* n,
                              int32_t* slots, int32_t* outboxes) {
    return pbx::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        pbx::ExecPlan p = pbx::make_plan(pbx::schedule_grid(s));
        if (device < 1 || device > p.topo.devices) throw std::invalid_argument("device out of range");
        const auto& ids = p.dev_ops[device];
        if (n) *n = ids.size();
        if (slots) *slots = p.slots[device];
        if (outboxes) *outboxes = p.outboxes[device];
        if (!out) return;
        if (cap < ids.size()) throw pbx::Space("plan buffer too small");
        for (size_t k = 0; k < ids.size(); ++k) {
            const pbx::PlanOp& q = p.ops[ids[k]];
            pb_plan_op r{};
            r.stage = q.op.stage;
            r.kind = int32_t(q.op.kind);
            r.microbatch = q.op.mb;
            r.start = q.op.start;
            r.slot = q.slot;
            if (q.in_msg >= 0) {
                const pbx::Msg& m = p.msgs[q.in_msg];
                r.recv_from = m.src_dev;
                r.recv_outbox = m.outbox;
                r.recv_gen = m.gen;
            }
            if (q.out_msg >= 0) {
                const pbx::Msg& m = p.msgs[q.out_msg];
                r.send_to = m.dst_dev;
                r.send_outbox = m.outbox;
                r.send_gen = m.gen;
            }
            out[k] = r;
        }
    });
}
