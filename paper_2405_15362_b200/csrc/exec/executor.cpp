// One pipeline device: weights of the stages it owns, the lifespan-bounded
// activation pool, the outbox ring for stage-boundary messages, and the
// per-pass kernel chains.  The host walks this device's passes in grid order
// and only ENQUEUES: every cross-device dependency is a device-side wait, so
// the host runs ahead and the GPU starts each pass as soon as its inputs land.
//
// Transport (neighbour pull over NVLink):
//   producer: last kernel writes the boundary tensor into its outbox slot k,
//             then cuStreamWriteValue32(consumer.ready[src][k] = gen)
//   consumer: copy stream waits ready >= gen, cudaMemcpyAsync peer->local
//             (copy engines, no SM time), writes producer.ack[k] = gen, and the
//             compute stream waits on that copy only when the pass starts
//   producer: before reusing outbox slot k waits ack[k] >= previous gen
// Outbox slots are interval-coloured over [producer start, consumer start) in
// grid time, and grid start order is a global topological order
// (assemble.hpp:185-187), so every wait points strictly back in grid time:
// deadlock-free by induction over cells.
#include "executor.hpp"

#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>

namespace pbx {

using vsched::Kind;

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct DriverFns {
    PFN_cuStreamWaitValue32_v11070 wait = nullptr;
    PFN_cuStreamWriteValue32_v11070 write = nullptr;
};
const DriverFns& drv() {
    static DriverFns f = [] {
        DriverFns d;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw CudaError("cuStreamWaitValue32 unavailable");
        d.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw CudaError("cuStreamWriteValue32 unavailable");
        d.write = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
        return d;
    }();
    return f;
}

void wait_value(cudaStream_t s, const uint32_t* addr, uint32_t v) {
    CUresult r = drv().wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                            CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed: " + std::to_string(int(r)));
}
void write_value(cudaStream_t s, uint32_t* addr, uint32_t v) {
    CUresult r = drv().write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                             CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed: " + std::to_string(int(r)));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

// ------------------------------------------------------------------ layout
void Exec::build_layout() {
    const size_t Th = size_t(T) * h;
    auto add = [](size_t& cur, size_t bytes) {
        size_t o = cur;
        cur = align_up(cur + bytes, 1024);
        return o;
    };
    slot_bytes = 0;
    for (int s : stages) {
        const int Lc = stage_L[s];
        StageLayout L;
        size_t cur = 0;
        L.x.resize(size_t(Lc) + 1);
        L.dx.resize(size_t(Lc) + 1);
        for (int l = 0; l <= Lc; ++l) {
            L.x[l] = add(cur, Th * 2);
            L.dx[l] = add(cur, Th * 2);
        }
        L.layer.resize(Lc);
        for (int l = 0; l < Lc; ++l) {
            auto& y = L.layer[l];
            if (!fold) y.a = add(cur, Th * 2);
            y.qkv = add(cur, 3 * Th * 2);
            y.o = add(cur, Th * 2);
            y.x1 = add(cur, Th * 2);
            if (!fold) y.b = add(cur, Th * 2);
            y.u = add(cur, 4 * Th * 2);
            y.gl = add(cur, 4 * Th * 2);
            y.dqkv = add(cur, 3 * Th * 2);
            y.dx1 = add(cur, Th * 2);
            if (!fold) {
                y.rstd1 = add(cur, size_t(T) * 4);
                y.rstd2 = add(cur, size_t(T) * 4);
            }
            y.lse = add(cur, size_t(H) * T * 4);
        }
        if (fold) {  // one block of per-token sums of squares, written by every F pass
            L.ss_bytes = size_t(2 * Lc + 1) * T * 4;
            L.ss = add(cur, L.ss_bytes);
            for (int l = 0; l < Lc; ++l) {
                L.layer[l].ss1 = L.ss + size_t(2 * l) * T * 4;
                L.layer[l].ss2 = L.ss + size_t(2 * l + 1) * T * 4;
            }
            L.ssf = L.ss + size_t(2 * Lc) * T * 4;
        }
        if (is_last(s)) {  // LM-head buffers live in their own lifespan pool (head slots, see constructor)
            size_t hc = 0;
            if (!fold) {
                L.hf = add(hc, Th * 2);
                L.rstdf = add(hc, size_t(T) * 4);
            }
            L.logits = add(hc, size_t(T) * V * 2);
            head_bytes = hc;
        }
        L.bytes = cur;
        layout[s] = L;
        slot_bytes = std::max(slot_bytes, cur);
    }
}

// ------------------------------------------------------------------ params
void Exec::build_params() {
    size_t off = 0;
    auto add = [&](const std::string& name, size_t numel, int id, float std, float constant) {
        PTensor t{name, off, numel, id, std, constant};
        off += align_up(numel, 64);
        ptensors.push_back(t);
        return ptensors.size() - 1;
    };
    const float std_in = 0.02f, std_out = 0.02f / std::sqrt(2.f * cfg.layers);
    for (int s : stages) {
        StageParams sp;
        if (is_first(s)) sp.emb = add("s" + std::to_string(s) + ".emb", size_t(V) * h, 1, std_in, 0.f);
        for (int l = 0; l < stage_L[s]; ++l) {
            const int gl = stage_first[s] + l;
            const std::string pre = "s" + std::to_string(s) + ".l" + std::to_string(l) + ".";
            LayerParams lp;
            lp.g1 = add(pre + "norm1", h, 16 + gl * 8 + 0, 0.f, 1.f);
            lp.wqkv = add(pre + "wqkv", size_t(3) * h * h, 16 + gl * 8 + 1, std_in, 0.f);
            lp.wo = add(pre + "wo", size_t(h) * h, 16 + gl * 8 + 2, std_out, 0.f);
            lp.g2 = add(pre + "norm2", h, 16 + gl * 8 + 3, 0.f, 1.f);
            lp.w1 = add(pre + "w1", size_t(4) * h * h, 16 + gl * 8 + 4, std_in, 0.f);
            lp.w2 = add(pre + "w2", size_t(4) * h * h, 16 + gl * 8 + 5, std_out, 0.f);
            sp.layers.push_back(lp);
        }
        if (is_last(s)) {
            sp.gf = add("s" + std::to_string(s) + ".norm", h, 2, 0.f, 1.f);
            sp.head = add("s" + std::to_string(s) + ".head", size_t(V) * h, 3, std_in, 0.f);
        }
        sparams[s] = sp;
    }
    n_params = off;
}

Exec::Exec(const pb_model_cfg& c, const vsched::Grid& grid, int device, int cuda_dev)
    : cfg(c), plan(make_plan(grid)), dev(device), cuda(cuda_dev) {
    try {
        init(device);
    } catch (...) {  // e.g. out of device memory part-way: give back what was allocated, then report
        release();
        throw;
    }
}

void Exec::init(int device) {
    if (device < 1 || device > plan.topo.devices) throw std::invalid_argument("device out of range");
    S = plan.topo.num_stages;
    twin = !plan.topo.default_routes();  // make_plan admits only the gems / chimera twin besides
    Sm = twin ? S / 2 : S;
    stage_L.assign(size_t(S) + 1, 0);
    stage_first.assign(size_t(S) + 2, 0);
    std::vector<int> model_L(size_t(Sm) + 1, 0), model_first(size_t(Sm) + 2, 0);
    if (cfg.stage_layers) {
        if (twin) throw std::invalid_argument("stage_layers: not supported with replicated-weight (twin) schedules");
        int sum = 0;
        for (int s = 1; s <= S; ++s) {
            model_L[s] = cfg.stage_layers[s - 1];
            if (model_L[s] < 1) throw std::invalid_argument("stage_layers: every stage needs >= 1 layer");
            sum += model_L[s];
        }
        if (sum != cfg.layers) throw std::invalid_argument("stage_layers must sum to layers");
        cfg.stage_layers = nullptr;  // copied
    } else {
        if (cfg.layers % Sm) throw std::invalid_argument("layers must be a multiple of the stage count");
        for (int s = 1; s <= Sm; ++s) model_L[s] = cfg.layers / Sm;
    }
    for (int s = 1; s <= Sm; ++s) model_first[s + 1] = model_first[s] + model_L[s];
    for (int s = 1; s <= S; ++s) {  // a replica stage holds its model stage's layers (same init ids)
        stage_L[s] = model_L[model_stage(s)];
        stage_first[s] = model_first[model_stage(s)];
    }
    h = cfg.hidden;
    H = cfg.heads;
    V = cfg.vocab;
    seq = cfg.seq;
    mbs = cfg.micro_batch;
    T = seq * mbs;
    if (H * 128 != h) throw std::invalid_argument("hidden must equal heads * 128");
    if (seq % 128 || h % 128 || V % 128) throw std::invalid_argument("seq, hidden, vocab must be multiples of 128");
    for (int s = 1; s <= S; ++s)
        if (plan.topo.device_of(s) == dev) stages.push_back(s);
    m = plan.microbatches;

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw CudaError("no CUDA device available (the executor has no CPU fallback)");
    }
    if (cuda < 0 || cuda >= ndev) throw CudaError("cuda device ordinal out of range");
    ck(cudaSetDevice(cuda), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, cuda), "cudaGetDeviceProperties");
    if (prop.major != 10) throw CudaError("executor kernels are built for sm_100a; device is sm_" +
                                          std::to_string(prop.major * 10 + prop.minor));
    drv();

    fold = std::getenv("PB_NO_FOLD") == nullptr;  // (decides the activation layout)
    build_layout();
    build_params();
    ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking), "stream");

    {
        size_t fr = 0, tot = 0;
        ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
        mem_device_total = tot;
        mem_used_at_create = tot - fr;
    }
    auto dmalloc = [&](size_t bytes, const char* what) {
        void* p = nullptr;
        const size_t n = std::max<size_t>(bytes, 256);
        if (cudaMalloc(&p, n) != cudaSuccess) {
            cudaGetLastError();
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            throw CudaError(std::string("out of device memory allocating ") + what + " (" + std::to_string(n) +
                            " B; executor holds " + std::to_string(mem_alloc_total) + " B, device free " +
                            std::to_string(fr) + " of " + std::to_string(tot) + " B)");
        }
        allocations.push_back(p);
        mem_alloc[what] += n;
        mem_alloc_total += n;
        return p;
    };
    master = static_cast<float*>(dmalloc(n_params * 4, "params"));
    wts = static_cast<__nv_bfloat16*>(dmalloc(n_params * 2, "params"));
    grads = static_cast<float*>(dmalloc(n_params * 4, "grads"));
    adam_m = static_cast<float*>(dmalloc(n_params * 4, "adam"));
    adam_v = static_cast<float*>(dmalloc(n_params * 4, "adam"));
    if (twin) {  // receive buffer for the replica device's gradient arena (same size: same model stages)
        rtmp = static_cast<float*>(dmalloc(n_params * 4, "replica grads"));
        const int s0 = stages.front();
        replica_dev = plan.topo.device_of(s0 > Sm ? s0 - Sm : s0 + Sm);
    }
    ck(cudaMemsetAsync(grads, 0, n_params * 4, cs), "memset");
    ck(cudaMemsetAsync(adam_m, 0, n_params * 4, cs), "memset");
    ck(cudaMemsetAsync(adam_v, 0, n_params * 4, cs), "memset");
    ck(cudaMemsetAsync(master, 0, n_params * 4, cs), "memset");
    for (const auto& t : ptensors)
        pbk::init_normal(master + t.off, t.numel, cfg.seed * 1000003ull + uint64_t(t.id), t.std, t.constant, cs);
    pbk::f32_to_bf16(master, wts, n_params, cs);
    if (fold) {
        size_t off = 0;
        for (int s : stages) {
            const StageParams& P = sparams.at(s);
            for (const auto& lp : P.layers) {
                folds.push_back({lp.wqkv, lp.g1, 3 * h, h, off});
                off += align_up(size_t(3) * h * h, 64);
                folds.push_back({lp.w1, lp.g2, 4 * h, h, off});
                off += align_up(size_t(4) * h * h, 64);
            }
            if (is_last(s)) {
                folds.push_back({P.head, P.gf, V, h, off});
                off += align_up(size_t(V) * h, 64);
            }
        }
        for (size_t i = 0; i < folds.size(); ++i) fold_of[folds[i].w] = i;
        gfold = static_cast<float*>(dmalloc(std::max<size_t>(off, 64) * 4, "folded grads"));
        ck(cudaMemsetAsync(gfold, 0, std::max<size_t>(off, 64) * 4, cs), "memset");
        refold();
    }

    nslots = plan.slots[dev];
    pool = static_cast<uint8_t*>(dmalloc(slot_bytes * size_t(std::max(nslots, 1)), "activation pool"));
    ck(cudaMemsetAsync(pool, 0, slot_bytes * size_t(std::max(nslots, 1)), cs), "memset");  // defined receive slots (PB_FLAG_SOLO)
    // head pool: hf / rstd / logits of the last stage, a slot per live (S, mb) from F(S) to W(S),
    // coloured like the main pool but over stage S alone — a V device holding stages 1 and 2p
    // does not pay the logits in every one of its slots
    head_slot_mb.assign(size_t(m), -1);
    if (std::any_of(stages.begin(), stages.end(), [&](int st) { return is_last(st); })) {
        std::vector<bool> busy;
        for (int i : plan.dev_ops[dev]) {
            const auto& o = plan.ops[size_t(i)].op;
            if (!is_last(o.stage)) continue;
            if (o.kind == vsched::Kind::F) {
                int k = 0;
                while (k < int(busy.size()) && busy[k]) ++k;
                if (k == int(busy.size())) busy.push_back(false);
                busy[k] = true;
                head_slot_mb[size_t(o.mb)] = k;
            } else if (o.kind == vsched::Kind::W || o.kind == vsched::Kind::BW) {
                busy[size_t(head_slot_mb[size_t(o.mb)])] = false;
            }
        }
        nhead = int(busy.size());
        hpool = static_cast<uint8_t*>(dmalloc(head_bytes * size_t(std::max(nhead, 1)), "head pool"));
    }
    build_w_groups();
    msg_bytes = align_up(size_t(T) * h * 2, 1024);
    nout = std::max(plan.outboxes[dev], 1);
    outbox = static_cast<uint8_t*>(dmalloc(msg_bytes * size_t(nout), "outbox"));
    nflags = size_t(plan.max_outbox + 1) * size_t(plan.topo.devices + 2);
    flags = static_cast<uint32_t*>(dmalloc(nflags * 4, "flags"));
    ck(cudaMemsetAsync(flags, 0, nflags * 4, cs), "memset");
    scratch = static_cast<__nv_bfloat16*>(dmalloc(size_t(T) * h * 2, "scratch"));
    dsum = static_cast<float*>(dmalloc(size_t(H) * T * 4 + 256, "scratch"));  // + the attention bwd work counter
    dq_acc = static_cast<float*>(dmalloc(size_t(T) * h * 4, "scratch"));
    // deterministic row sums of squares (folded RMSNorm): per-128-column partials + row-group counters
    ss_part = static_cast<float*>(dmalloc(size_t(T) * (h / 128) * 4, "scratch"));
    ss_cnt = static_cast<int*>(dmalloc(size_t(T / 32 + 1) * 4, "scratch"));
    ck(cudaMemsetAsync(ss_cnt, 0, size_t(T / 32 + 1) * 4, cs), "memset");
    tokens = static_cast<int32_t*>(dmalloc(size_t(m) * T * 4, "inputs"));
    labels = static_cast<int32_t*>(dmalloc(size_t(m) * T * 4, "inputs"));
    loss_dev = static_cast<float*>(dmalloc(64, "loss"));
    ck(cudaMallocHost(reinterpret_cast<void**>(&loss_host), 64), "pinned");

    const auto& ops = plan.dev_ops[dev];
    pos_of.assign(plan.ops.size(), -1);
    for (size_t j = 0; j < ops.size(); ++j) pos_of[ops[j]] = int(j);
    ev_start.resize(ops.size());
    ev_end.resize(ops.size());
    ev_pull.resize(ops.size());
    ev_free.resize(ops.size());
    ev_copy0.resize(ops.size());
    ev_copy1.resize(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) {
        ck(cudaEventCreate(&ev_start[i]), "event");
        ck(cudaEventCreate(&ev_end[i]), "event");
        ck(cudaEventCreateWithFlags(&ev_pull[i], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming), "event");
        ck(cudaEventCreate(&ev_copy0[i]), "event");
        ck(cudaEventCreate(&ev_copy1[i]), "event");
    }
    ck(cudaEventCreate(&ev_step0), "event");
    ck(cudaEventCreate(&ev_step1), "event");
    peers.assign(size_t(plan.topo.devices) + 1, Peer{});
    peers[dev] = Peer{outbox, flags, false};
    ck(cudaStreamSynchronize(cs), "init");
    sample_device_memory();
}

Exec::~Exec() { release(); }

void Exec::release() noexcept {
    if (released) return;
    released = true;
    if (cuda < 0) return;
    cudaSetDevice(cuda);
    cudaDeviceSynchronize();
    for (auto& kv : wgroups) pbk::gemm_group_destroy(kv.second);
    for (auto* v : {&ev_start, &ev_end, &ev_pull, &ev_free, &ev_copy0, &ev_copy1})
        for (auto e : *v) cudaEventDestroy(e);
    for (auto e : gev) cudaEventDestroy(e);
    for (auto e : kev) cudaEventDestroy(e);
    cudaEventDestroy(ev_step0);
    cudaEventDestroy(ev_step1);
    for (auto& p : peers)
        if (p.ipc) {
            cudaIpcCloseMemHandle(p.outbox);
            cudaIpcCloseMemHandle(p.flags);
        }
    for (void* p : allocations) cudaFree(p);
    allocations.clear();
    if (loss_host) cudaFreeHost(loss_host);
    if (cs) cudaStreamDestroy(cs);
    if (xs) cudaStreamDestroy(xs);
    cudaGetLastError();
}

void Exec::sample_device_memory() {
    size_t fr = 0, tot = 0;
    ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
    mem_used_high = std::max(mem_used_high, tot - fr);
}

// ------------------------------------------------------------------ gamma folding
float* Exec::GW(size_t p) const {
    auto it = fold_of.find(p);
    return it == fold_of.end() ? G(p) : gfold + folds[it->second].off;
}

void Exec::refold() {
    for (const auto& f : folds)
        pbk::fold_weight(master + ptensors[f.w].off, master + ptensors[f.g].off, wts + ptensors[f.w].off, f.rows,
                         f.cols, cs);
    launches += int64_t(folds.size());
}

void Exec::fold_grads() {
    for (const auto& f : folds)
        pbk::fold_grad(gfold + f.off, master + ptensors[f.w].off, master + ptensors[f.g].off, G(f.w), G(f.g), dq_acc,
                       size_t(T) * h, f.rows, f.cols, cs);
    launches += 2 * int64_t(folds.size());
}

// ------------------------------------------------------------------ passes
__nv_bfloat16* Exec::bf(int slot, size_t off) const {
    return reinterpret_cast<__nv_bfloat16*>(pool + size_t(slot) * slot_bytes + off);
}
float* Exec::f32(int slot, size_t off) const { return reinterpret_cast<float*>(pool + size_t(slot) * slot_bytes + off); }
uint8_t* Exec::head(int mb, size_t off) const {
    return hpool + size_t(head_slot_mb.at(size_t(mb))) * head_bytes + off;
}
__nv_bfloat16* Exec::outbox_ptr(int k) const { return reinterpret_cast<__nv_bfloat16*>(outbox + size_t(k) * msg_bytes); }

template <typename Fn>
void Exec::timed(const char* label, Fn&& fn) {
    static const bool sync_trace = std::getenv("PB_SYNC_TRACE") != nullptr;  // debugging: which launch hangs
    if (sync_trace) {
        std::fprintf(stderr, "[dev %d] launch %s\n", dev, label);
        fn();
        ck(cudaStreamSynchronize(cs), "sync trace");
        std::fprintf(stderr, "[dev %d] done %s\n", dev, label);
        return;
    }
    if (!kernel_timing) {
        fn();
        return;
    }
    int id = -1;
    for (size_t i = 0; i < klabels.size(); ++i)
        if (klabels[i] == label) id = int(i);
    if (id < 0) {
        klabels.push_back(label);
        id = int(klabels.size()) - 1;
    }
    if (kev_used + 2 > kev.size()) {
        const size_t old = kev.size();
        kev.resize(old + 1024);
        for (size_t i = old; i < kev.size(); ++i) ck(cudaEventCreate(&kev[i]), "event");
    }
    if (kev_label.size() < kev.size() / 2) kev_label.resize(kev.size() / 2);
    ck(cudaEventRecord(kev[kev_used], cs), "event");
    fn();
    ck(cudaEventRecord(kev[kev_used + 1], cs), "event");
    kev_label[kev_used / 2] = id;
    kev_used += 2;
}

void Exec::gemm(int M, int N, int K, const __nv_bfloat16* A, bool a_mn, const __nv_bfloat16* B, bool b_mn, void* C,
                int epi, const __nv_bfloat16* aux, void* C2, int accumulate, const float* rs, float* ss_out) {
    pbk::GemmArgs g;
    g.rs = rs, g.rs_inv_n = 1.f / float(h), g.rs_eps = kNormEps, g.ss_out = ss_out;
    if (ss_out) g.ss_part = ss_part, g.ss_cnt = ss_cnt;
    g.M = M, g.N = N, g.K = K;
    g.A = A, g.a_mn = a_mn, g.lda = a_mn ? M : K;
    g.B = B, g.b_mn = b_mn, g.ldb = b_mn ? N : K;
    g.C = C, g.ldc = N, g.C2 = C2;
    g.aux = aux, g.ldaux = N;
    g.epi = epi, g.accumulate = accumulate;
    const char* glabel = a_mn ? "gemm_W" : (b_mn ? "gemm_B" : "gemm_F");
    static const bool sync_trace = std::getenv("PB_SYNC_TRACE") != nullptr;
    if (kernel_timing || sync_trace) {
        if (sync_trace) std::fprintf(stderr, "[dev %d] gemm M%d N%d K%d epi%d amn%d bmn%d rs%d ss%d\n", dev, M, N, K, epi,
                                     int(a_mn), int(b_mn), rs != nullptr, ss_out != nullptr);
        timed(glabel, [&] { pbk::gemm(g, cs); });
        gemm_flops_acc += 2.0 * double(M) * double(N) * double(K);
    } else if (gemm_timing) {
        if (gev_used + 2 > gev.size()) {
            gev.resize(gev.size() + 512);
            for (size_t i = gev.size() - 512; i < gev.size(); ++i) ck(cudaEventCreate(&gev[i]), "event");
        }
        ck(cudaEventRecord(gev[gev_used++], cs), "event");
        pbk::gemm(g, cs);
        ck(cudaEventRecord(gev[gev_used++], cs), "event");
        gemm_flops_acc += 2.0 * double(M) * double(N) * double(K);
    } else {
        pbk::gemm(g, cs);
    }
    ++launches;
}

// All weight-gradient GEMMs of one W pass (every layer of the stage) as one grouped launch.
void Exec::build_w_groups() {
    if (std::getenv("PB_NO_WGROUP")) return;
    for (int s : stages) {
        const StageLayout& L = layout.at(s);
        const StageParams& P = sparams.at(s);
        const int Lc = stage_L[s];
        for (int slot = 0; slot < nslots; ++slot) {
            std::vector<pbk::GemmArgs> v;
            double fl = 0;
            auto add = [&](int M, int N, const __nv_bfloat16* A, const __nv_bfloat16* B, float* C) {
                pbk::GemmArgs g;
                g.M = M, g.N = N, g.K = T;
                g.A = A, g.a_mn = true, g.lda = M;
                g.B = B, g.b_mn = true, g.ldb = N;
                g.C = C, g.ldc = N, g.epi = pbk::EPI_F32, g.accumulate = 1;
                v.push_back(g);
                fl += 2.0 * M * N * T;
            };
            for (int l = Lc - 1; l >= 0; --l) {
                const auto& y = L.layer[l];
                const auto& w = P.layers[l];
                add(h, 4 * h, bf(slot, L.dx[l + 1]), bf(slot, y.gl), G(w.w2));
                add(4 * h, h, bf(slot, y.u), bf(slot, fold ? y.x1 : y.b), GW(w.w1));
                add(h, h, bf(slot, y.dx1), bf(slot, y.o), G(w.wo));
                add(3 * h, h, bf(slot, y.dqkv), bf(slot, fold ? L.x[l] : y.a), GW(w.wqkv));
            }
            bool ok = true;
            for (const auto& g : v) ok = ok && pbk::gemm_group_ok(g);
            if (!ok) continue;
            wgroups[{s, slot}] = pbk::gemm_group_create(v.data(), int(v.size()));
            wgroup_flops[{s, slot}] = fl;
        }
    }
}

void Exec::run_gemm_timed(const char* label, double flops, const std::function<void()>& fn) {
    static const bool sync_trace = std::getenv("PB_SYNC_TRACE") != nullptr;
    if (kernel_timing || sync_trace) {
        timed(label, fn);
        gemm_flops_acc += flops;
    } else if (gemm_timing) {
        if (gev_used + 2 > gev.size()) {
            gev.resize(gev.size() + 512);
            for (size_t i = gev.size() - 512; i < gev.size(); ++i) ck(cudaEventCreate(&gev[i]), "event");
        }
        ck(cudaEventRecord(gev[gev_used++], cs), "event");
        fn();
        ck(cudaEventRecord(gev[gev_used++], cs), "event");
        gemm_flops_acc += flops;
    } else {
        fn();
    }
    ++launches;
}

#define HB(mb, off) reinterpret_cast<__nv_bfloat16*>(head(mb, off))
#define HF(mb, off) reinterpret_cast<float*>(head(mb, off))

void Exec::pass_forward(int s, int mb, int slot, __nv_bfloat16* out) {
    const int Lc = stage_L[s];
    const StageLayout& L = layout.at(s);
    const StageParams& P = sparams.at(s);
    __nv_bfloat16* x0 = bf(slot, L.x[0]);
    if (is_first(s)) {
        timed("embed_fwd", [&] { pbk::embed_fwd(tokens + size_t(mb) * T, wts + ptensors[P.emb].off, x0, T, h, V, id_err(), cs); });
        ++launches;
    }
    if (fold) {
        // RMSNorm folded into the GEMMs around it (gamma is folded into the consuming weights, see
        // fold_weight): the residual epilogues accumulate each row's sum of squares, the consuming
        // projection scales its accumulator rows by rstd = rsqrt(ss / h + eps); x-hat is never stored.
        // Every statistic is written (not accumulated) and is bit-identical whether it comes from an
        // epilogue or from row_sumsq, so results do not depend on where the stage boundaries fall.
        timed("row_sumsq", [&] { pbk::row_sumsq(x0, f32(slot, L.layer.empty() ? L.ssf : L.layer[0].ss1), T, h, cs); });
        ++launches;
    }
    for (int l = 0; l < Lc; ++l) {
        const auto& y = L.layer[l];
        const auto& w = P.layers[l];
        __nv_bfloat16* x = bf(slot, L.x[l]);
        __nv_bfloat16* xo = (l == Lc - 1 && !is_last(s)) ? out : bf(slot, L.x[l + 1]);
        if (fold) {
            float* ss_next = l + 1 < Lc ? f32(slot, L.layer[l + 1].ss1) : (is_last(s) ? f32(slot, L.ssf) : nullptr);
            gemm(T, 3 * h, h, x, false, W(w.wqkv), false, bf(slot, y.qkv), pbk::EPI_STORE, nullptr, nullptr, 0,
                 f32(slot, y.ss1));
            timed("attn_fwd", [&] { pbk::attn_fwd_tc(bf(slot, y.qkv), bf(slot, y.o), f32(slot, y.lse), mbs, seq, H, cs); });
            gemm(T, h, h, bf(slot, y.o), false, W(w.wo), false, bf(slot, y.x1), pbk::EPI_RESID, x, nullptr, 0, nullptr,
                 f32(slot, y.ss2));
            gemm(T, 4 * h, h, bf(slot, y.x1), false, W(w.w1), false, bf(slot, y.u), pbk::EPI_GELU, nullptr,
                 bf(slot, y.gl), 0, f32(slot, y.ss2));
            gemm(T, h, 4 * h, bf(slot, y.gl), false, W(w.w2), false, xo, pbk::EPI_RESID, bf(slot, y.x1), nullptr, 0,
                 nullptr, ss_next);
            ++launches;
            continue;
        }
        timed("rmsnorm_fwd", [&] { pbk::rmsnorm_fwd(x, W(w.g1), bf(slot, y.a), f32(slot, y.rstd1), T, h, cs); });
        gemm(T, 3 * h, h, bf(slot, y.a), false, W(w.wqkv), false, bf(slot, y.qkv), pbk::EPI_STORE);
        timed("attn_fwd", [&] { pbk::attn_fwd_tc(bf(slot, y.qkv), bf(slot, y.o), f32(slot, y.lse), mbs, seq, H, cs); });
        gemm(T, h, h, bf(slot, y.o), false, W(w.wo), false, bf(slot, y.x1), pbk::EPI_RESID, x);
        timed("rmsnorm_fwd", [&] { pbk::rmsnorm_fwd(bf(slot, y.x1), W(w.g2), bf(slot, y.b), f32(slot, y.rstd2), T, h, cs); });
        gemm(T, 4 * h, h, bf(slot, y.b), false, W(w.w1), false, bf(slot, y.u), pbk::EPI_GELU, nullptr,
             bf(slot, y.gl));
        gemm(T, h, 4 * h, bf(slot, y.gl), false, W(w.w2), false, xo, pbk::EPI_RESID, bf(slot, y.x1));
        launches += 3;
    }
    if (is_last(s)) {
        const float scale = 1.f / float(size_t(m) * T);
        if (fold) {
            gemm(T, V, h, bf(slot, L.x[Lc]), false, W(P.head), false, HB(mb, L.logits), pbk::EPI_STORE, nullptr,
                 nullptr, 0, f32(slot, L.ssf));
            timed("cross_entropy", [&] {
                pbk::cross_entropy(HB(mb, L.logits), labels + size_t(mb) * T, loss_dev, T, V, scale, id_err(), cs,
                                   f32(slot, L.ssf), 1.f / float(h), kNormEps);
            });
            ++launches;
        } else {
            timed("rmsnorm_fwd", [&] { pbk::rmsnorm_fwd(bf(slot, L.x[Lc]), W(P.gf), HB(mb, L.hf), HF(mb, L.rstdf), T, h, cs); });
            gemm(T, V, h, HB(mb, L.hf), false, W(P.head), false, HB(mb, L.logits), pbk::EPI_STORE);
            timed("cross_entropy", [&] { pbk::cross_entropy(HB(mb, L.logits), labels + size_t(mb) * T, loss_dev, T, V, scale, id_err(), cs); });
            launches += 2;
        }
    }
}

void Exec::pass_backward(int s, int mb, int slot, __nv_bfloat16* out) {
    const int Lc = stage_L[s];
    (void)mb;
    const StageLayout& L = layout.at(s);
    const StageParams& P = sparams.at(s);
    if (fold) {
        // Fold mode runs every normalised projection's backward on row-scaled output gradients
        // (dY' = rstd * dY: the CE kernel, the dGELU epilogue and the attention backward apply it), so
        // the dX GEMMs yield rstd * dX-hat and the weight GEMMs use the stored x: dW' = dY'^T x.
        if (is_last(s)) {
            gemm(T, h, V, HB(mb, L.logits), false, W(P.head), true, scratch, pbk::EPI_STORE);
            timed("rmsnorm_bwd", [&] { pbk::rmsnorm_bwd_x(scratch, bf(slot, L.x[Lc]), f32(slot, L.ssf), nullptr, bf(slot, L.dx[Lc]), T, h, kNormEps, cs); });
            ++launches;
        }
        for (int l = Lc - 1; l >= 0; --l) {
            const auto& y = L.layer[l];
            const auto& w = P.layers[l];
            __nv_bfloat16* dy = bf(slot, L.dx[l + 1]);
            __nv_bfloat16* dxo = (l == 0 && !is_first(s)) ? out : bf(slot, L.dx[l]);
            // du' = rstd2 * (dy . W2) * gelu'(u), written over u
            gemm(T, 4 * h, h, dy, false, W(w.w2), true, bf(slot, y.u), pbk::EPI_DGELU, bf(slot, y.u), nullptr, 0,
                 f32(slot, y.ss2));
            gemm(T, h, 4 * h, bf(slot, y.u), false, W(w.w1), true, scratch, pbk::EPI_STORE);
            timed("rmsnorm_bwd", [&] { pbk::rmsnorm_bwd_x(scratch, bf(slot, y.x1), f32(slot, y.ss2), dy, bf(slot, y.dx1), T, h, kNormEps, cs); });
            gemm(T, h, h, bf(slot, y.dx1), false, W(w.wo), true, scratch, pbk::EPI_STORE);
            timed("attn_bwd", [&] {
                pbk::attn_bwd_tc(bf(slot, y.qkv), bf(slot, y.o), scratch, f32(slot, y.lse), dsum, dq_acc, bf(slot, y.dqkv),
                                 mbs, seq, H, cs, f32(slot, y.ss1), 1.f / float(h), kNormEps);
            });
            gemm(T, h, 3 * h, bf(slot, y.dqkv), false, W(w.wqkv), true, scratch, pbk::EPI_STORE);
            timed("rmsnorm_bwd", [&] { pbk::rmsnorm_bwd_x(scratch, bf(slot, L.x[l]), f32(slot, y.ss1), bf(slot, y.dx1), dxo, T, h, kNormEps, cs); });
            launches += 6;
        }
        return;
    }
    if (is_last(s)) {
        // dhf = dlogits . Whead ; dx_L = rmsnorm_bwd(dhf)
        gemm(T, h, V, HB(mb, L.logits), false, W(P.head), true, scratch, pbk::EPI_STORE);
        timed("rmsnorm_bwd", [&] { pbk::rmsnorm_bwd(scratch, bf(slot, L.x[Lc]), W(P.gf), HF(mb, L.rstdf), nullptr, bf(slot, L.dx[Lc]), T, h,
                         cs); });
        timed("rmsnorm_dgamma", [&] { pbk::rmsnorm_dgamma(scratch, bf(slot, L.x[Lc]), HF(mb, L.rstdf), G(P.gf), dq_acc, T, h, cs); });
        launches += 2;
    }
    for (int l = Lc - 1; l >= 0; --l) {
        const auto& y = L.layer[l];
        const auto& w = P.layers[l];
        __nv_bfloat16* dy = bf(slot, L.dx[l + 1]);
        __nv_bfloat16* dxo = (l == 0 && !is_first(s)) ? out : bf(slot, L.dx[l]);
        // du = (dy . W2) * gelu'(u), written over u
        gemm(T, 4 * h, h, dy, false, W(w.w2), true, bf(slot, y.u), pbk::EPI_DGELU, bf(slot, y.u));
        gemm(T, h, 4 * h, bf(slot, y.u), false, W(w.w1), true, scratch, pbk::EPI_STORE);
        timed("rmsnorm_bwd", [&] { pbk::rmsnorm_bwd(scratch, bf(slot, y.x1), W(w.g2), f32(slot, y.rstd2), dy, bf(slot, y.dx1), T, h, cs); });
        timed("rmsnorm_dgamma", [&] { pbk::rmsnorm_dgamma(scratch, bf(slot, y.x1), f32(slot, y.rstd2), G(w.g2), dq_acc, T, h, cs); });
        gemm(T, h, h, bf(slot, y.dx1), false, W(w.wo), true, scratch, pbk::EPI_STORE);
        timed("attn_bwd", [&] { pbk::attn_bwd_tc(bf(slot, y.qkv), bf(slot, y.o), scratch, f32(slot, y.lse), dsum, dq_acc, bf(slot, y.dqkv), mbs,
                      seq, H, cs); });
        gemm(T, h, 3 * h, bf(slot, y.dqkv), false, W(w.wqkv), true, scratch, pbk::EPI_STORE);
        timed("rmsnorm_bwd", [&] { pbk::rmsnorm_bwd(scratch, bf(slot, L.x[l]), W(w.g1), f32(slot, y.rstd1), bf(slot, y.dx1), dxo, T, h, cs); });
        timed("rmsnorm_dgamma", [&] { pbk::rmsnorm_dgamma(scratch, bf(slot, L.x[l]), f32(slot, y.rstd1), G(w.g1), dq_acc, T, h, cs); });
        launches += 8;
    }
}

void Exec::pass_weight(int s, int mb, int slot) {
    const int Lc = stage_L[s];
    const StageLayout& L = layout.at(s);
    const StageParams& P = sparams.at(s);
    auto grp = wgroups.find({s, slot});
    if (grp != wgroups.end()) {
        run_gemm_timed("gemm_W", wgroup_flops.at({s, slot}), [&] { pbk::gemm_group_run(grp->second, cs); });
    } else
    for (int l = Lc - 1; l >= 0; --l) {
        const auto& y = L.layer[l];
        const auto& w = P.layers[l];
        gemm(h, 4 * h, T, bf(slot, L.dx[l + 1]), true, bf(slot, y.gl), true, G(w.w2), pbk::EPI_F32, nullptr, nullptr, 1);
        gemm(4 * h, h, T, bf(slot, y.u), true, bf(slot, fold ? y.x1 : y.b), true, GW(w.w1), pbk::EPI_F32, nullptr, nullptr, 1);
        gemm(h, h, T, bf(slot, y.dx1), true, bf(slot, y.o), true, G(w.wo), pbk::EPI_F32, nullptr, nullptr, 1);
        gemm(3 * h, h, T, bf(slot, y.dqkv), true, bf(slot, fold ? L.x[l] : y.a), true, GW(w.wqkv), pbk::EPI_F32, nullptr, nullptr, 1);
    }
    if (is_last(s))
        gemm(V, h, T, HB(mb, L.logits), true, fold ? bf(slot, L.x[Lc]) : HB(mb, L.hf), true, GW(P.head), pbk::EPI_F32,
             nullptr, nullptr, 1);
    if (is_first(s)) {
        timed("embed_bwd", [&] { pbk::embed_bwd(tokens + size_t(mb) * T, bf(slot, L.dx[0]), G(P.emb), T, h, V, id_err(), cs); });
        ++launches;
    }
}

// ------------------------------------------------------------------ step
uint32_t Exec::gen_total(const Msg& msg) const {
    return uint32_t(steps_done) * plan.uses[msg.src_dev][msg.outbox] + msg.gen;
}
uint32_t* Exec::ack_flag(uint32_t* base, int k) const { return base + k; }
uint32_t* Exec::ready_flag(uint32_t* base, int src, int k) const {
    return base + size_t(plan.max_outbox + 1) * size_t(1 + src) + k;
}

void Exec::enqueue(const int32_t* tok, const int32_t* lab, bool on_host) {
    if (!connected && !solo && plan.topo.devices > 1) throw StateError("pb_exec_step before peers are connected");
    if (solo && group) throw StateError("PB_FLAG_SOLO is for a device without peers (not a connected group)");
    ck(cudaSetDevice(cuda), "cudaSetDevice");
    const int64_t t = steps_done;
    if (group) {
        // peers must have finished enqueueing step t-1 before step t re-records any event parity
        group->wait([&] {
            for (int d = 1; d <= plan.topo.devices; ++d)
                if (group->enqueued[d] < t) return false;
            return true;
        });
    }
    launches = 0;
    peer_bytes = 0;
    copied.assign(plan.dev_ops[dev].size(), 0);
    gev_used = 0;
    kev_used = 0;
    gemm_flops_acc = 0;
    const size_t nin = size_t(m) * T * 4;
    const auto kind = on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    ck(cudaEventRecord(ev_step0, cs), "event");
    // cross-step WAR guard: this step's pulls (copy stream) write receive slots that the previous
    // step's last users (W passes read dx.back(), F-input slots whose first use has free_op < 0) may
    // still be reading on the compute stream — start the copy stream after everything enqueued so far
    ck(cudaStreamWaitEvent(xs, ev_step0, 0), "wait");
    const bool has_first = std::any_of(stages.begin(), stages.end(), [&](int st) { return is_first(st); });
    const bool has_last = std::any_of(stages.begin(), stages.end(), [&](int st) { return is_last(st); });
    if (on_host) {  // ids index the embedding / logits: reject out-of-range ids before anything is enqueued
        auto check = [&](const int32_t* ids, const char* what) {
            for (size_t i = 0; i < size_t(m) * T; ++i)
                if (ids[i] < 0 || ids[i] >= V)
                    throw std::invalid_argument(std::string(what) + " id " + std::to_string(ids[i]) + " at index " +
                                                std::to_string(i) + " outside [0, " + std::to_string(V) + ")");
        };
        // every device given the arrays checks them (not only the stage-1 / stage-S holders), so all
        // devices of a group that share the same host inputs fail together instead of waiting on a peer
        if (tok) check(tok, "token");
        if (lab) check(lab, "label");
    }
    ck(cudaMemsetAsync(loss_dev, 0, 8, cs), "loss");  // [0] loss, [1] out-of-range id flag (device inputs)
    if (has_first) {
        if (!tok) throw std::invalid_argument("tokens required on the device holding stage 1");
        ck(cudaMemcpyAsync(tokens, tok, nin, kind, cs), "tokens");
    }
    if (has_last) {
        if (!lab) throw std::invalid_argument("labels required on the device holding the last stage");
        ck(cudaMemcpyAsync(labels, lab, nin, kind, cs), "labels");
    }
    const auto& ops = plan.dev_ops[dev];
    int live = 0;
    pool_live_peak = 0;
    static const bool trace = std::getenv("PB_TRACE") != nullptr;
    for (size_t j = 0; j < ops.size(); ++j) {
        const int i = ops[j];
        const PlanOp& po = plan.ops[i];
        const auto& o = po.op;
        const StageLayout& L = layout.at(o.stage);
        if (trace)
            std::fprintf(stderr, "[dev %d] op %zu %s(s%d,mb%d)@%lld slot %d in %d out %d\n", dev, j,
                         vsched::kind_name(o.kind), o.stage, o.mb, (long long)o.start, po.slot, po.in_msg, po.out_msg);
        const bool iso = isolate && group;
        std::unique_lock<std::mutex> gpu_token(group ? group->iso_mu : local_iso_mu, std::defer_lock);
        // ---- incoming boundary tensor
        __nv_bfloat16* in_dst = nullptr;
        const Msg* in = po.in_msg >= 0 ? &plan.msgs[po.in_msg] : nullptr;
        if (in) in_dst = o.kind == Kind::F ? bf(po.slot, L.x[0]) : bf(po.slot, L.dx.back());
        if (in && !in->local() && !solo) {
            if (o.kind == Kind::F && po.free_op >= 0) {
                ck(cudaStreamWaitEvent(xs, ev_free[size_t(pos_of[po.free_op])], 0), "wait");
            }
            const Peer& src = peers[in->src_dev];
            const uint32_t g = gen_total(*in);
            const size_t mi = size_t(po.in_msg);
            if (group) {
                group->wait([&] { return group->ready_step[mi] >= t; });
                ck(cudaStreamWaitEvent(xs, group->ready_ev[t & 1][mi], 0), "wait");
            } else {
                wait_value(xs, ready_flag(flags, in->src_dev, in->outbox), g);
            }
            ck(cudaEventRecord(ev_copy0[j], xs), "event");
            ck(cudaMemcpyAsync(in_dst, reinterpret_cast<uint8_t*>(src.outbox) + size_t(in->outbox) * msg_bytes,
                               size_t(T) * h * 2, cudaMemcpyDeviceToDevice, xs),
               "peer copy");
            ck(cudaEventRecord(ev_copy1[j], xs), "event");
            copied[j] = 1;
            if (group) {
                ck(cudaEventRecord(group->ack_ev[t & 1][mi], xs), "event");
                group->set(group->ack_step, mi, t);
            } else {
                write_value(xs, ack_flag(src.flags, in->outbox), g);
            }
            ck(cudaEventRecord(ev_pull[j], xs), "event");
            ck(cudaStreamWaitEvent(cs, ev_pull[j], 0), "wait");
            peer_bytes += int64_t(T) * h * 2;
        }
        // ---- outgoing: outbox slot must be drained by its previous (remote) consumer
        const Msg* out = po.out_msg >= 0 ? &plan.msgs[po.out_msg] : nullptr;
        if (out && out->prev_remote && gen_total(*out) > 1 && !solo) {
            if (group) {
                const int64_t tp = out->prev_cross_step ? t - 1 : t;
                const size_t pm = size_t(out->prev_msg);
                group->wait([&] { return group->ack_step[pm] >= tp; });
                ck(cudaStreamWaitEvent(cs, group->ack_ev[tp & 1][pm], 0), "wait");
            } else {
                wait_value(cs, ack_flag(flags, out->outbox), gen_total(*out) - 1);
            }
        }
        // isolate: every cross-device wait above is host-side, so taking the group's GPU token
        // only now keeps the schedule deadlock-free while passes run one at a time
        if (iso) gpu_token.lock();
        if (timeline) ck(cudaEventRecord(ev_start[j], cs), "event");
        if (in && in->local())
            ck(cudaMemcpyAsync(in_dst, outbox_ptr(in->outbox), size_t(T) * h * 2, cudaMemcpyDeviceToDevice, cs),
               "local copy");
        __nv_bfloat16* out_ptr = out ? outbox_ptr(out->outbox) : nullptr;
        switch (o.kind) {
            case Kind::F:
                ++live;
                pool_live_peak = std::max(pool_live_peak, live);
                pass_forward(o.stage, o.mb, po.slot, out_ptr);
                break;
            case Kind::B: pass_backward(o.stage, o.mb, po.slot, out_ptr); break;
            case Kind::W: pass_weight(o.stage, o.mb, po.slot); break;
            case Kind::BW:
                pass_backward(o.stage, o.mb, po.slot, out_ptr);
                pass_weight(o.stage, o.mb, po.slot);
                break;
        }
        if (timeline) ck(cudaEventRecord(ev_end[j], cs), "event");
        if (out && !out->local() && !solo) {
            if (group) {
                const size_t mi = size_t(po.out_msg);
                ck(cudaEventRecord(group->ready_ev[t & 1][mi], cs), "event");
                group->set(group->ready_step, mi, t);
            } else {
                write_value(cs, ready_flag(peers[out->dst_dev].flags, dev, out->outbox), gen_total(*out));
            }
        }
        if (o.kind == Kind::W || o.kind == Kind::BW) {
            --live;
            ck(cudaEventRecord(ev_free[j], cs), "event");
        }
        if (serial || iso) {
            ck(cudaStreamSynchronize(xs), "serial");
            ck(cudaStreamSynchronize(cs), "serial");
        }
        if (iso) {
            gpu_token.unlock();
            {
                std::lock_guard<std::mutex> lk(group->mu);
                if (group->iso_step != t) group->iso_step = t, group->iso_done = 0;
                ++group->iso_done;
            }
            group->cv.notify_all();
        }
    }
    if (isolate && group)  // keep the optimizer off the isolated pass window
        group->wait([&] { return group->iso_step == t && group->iso_done == int64_t(plan.ops.size()); });
    if (fold) timed("fold_grad", [&] { fold_grads(); });
    if (twin && !solo) sync_replicas(t);  // data-parallel replicas: every copy gets the summed gradient
    if (cfg.optimizer) {
        ++adam_step;
        timed("adamw", [&] {
            pbk::adamw(master, wts, grads, adam_m, adam_v, n_params, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps,
                       cfg.weight_decay, adam_step, cs);
        });
        ++launches;
        if (fold) timed("fold_weight", [&] { refold(); });
    }
    ck(cudaMemcpyAsync(loss_host, loss_dev, 8, cudaMemcpyDeviceToHost, cs), "loss");
    ck(cudaEventRecord(ev_step1, cs), "event");
    ck(cudaGetLastError(), "launch");
    ++steps_done;
    if (group) group->set(group->enqueued, size_t(dev), steps_done);
    pending = true;
}

void Exec::finish(pb_timed_pass* tl, size_t tl_n, pb_exec_stats* st) {
    ck(cudaSetDevice(cuda), "cudaSetDevice");
    if (const char* wd = std::getenv("PB_WATCHDOG_S"); wd && kernel_timing) {
        // debugging: name the first launch of this device that has not completed after the deadline
        const auto t0 = std::chrono::steady_clock::now();
        while (cudaStreamQuery(cs) == cudaErrorNotReady) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::duration<double>(std::atof(wd))) {
                for (size_t e = 0; e + 1 < kev_used; e += 2)
                    if (cudaEventQuery(kev[e + 1]) == cudaErrorNotReady) {
                        std::fprintf(stderr, "[dev %d] watchdog: launch %zu (%s) not complete, started: %d\n", dev,
                                     e / 2, klabels[size_t(kev_label[e / 2])].c_str(),
                                     int(cudaEventQuery(kev[e]) == cudaSuccess));
                        break;
                    }
                std::fflush(stderr);
                std::this_thread::sleep_for(std::chrono::seconds(2));  // let the peer devices report too
                std::abort();
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(5));
        }
    }
    ck(cudaStreamSynchronize(cs), "step");
    ck(cudaStreamSynchronize(xs), "step");
    pending = false;
    sample_device_memory();
    if (reinterpret_cast<const int32_t*>(loss_host)[1])
        throw std::invalid_argument("token or label id outside [0, " + std::to_string(V) + ") in the step's device inputs");
    const auto& ops = plan.dev_ops[dev];
    const bool has_last = std::any_of(stages.begin(), stages.end(), [&](int st) { return is_last(st); });
    double busy = 0;
    if (timeline) {
        if (tl && tl_n < ops.size()) throw Space("timeline buffer too small");
        for (size_t j = 0; j < ops.size(); ++j) {
            float a = 0, b = 0;
            ck(cudaEventElapsedTime(&a, ev_step0, ev_start[j]), "elapsed");
            ck(cudaEventElapsedTime(&b, ev_step0, ev_end[j]), "elapsed");
            busy += double(b) - double(a);
            if (tl) {
                const auto& o = plan.ops[ops[j]].op;
                tl[j] = {o.device, o.stage, int32_t(o.kind), o.mb, double(a), double(b) - double(a)};
            }
        }
    }
    if (st) {
        float total = 0;
        ck(cudaEventElapsedTime(&total, ev_step0, ev_step1), "elapsed");
        st->loss = has_last ? double(*loss_host) : NAN;
        st->step_ms = total;
        st->busy_ms = busy;
        st->pool_slots = nslots;
        st->pool_peak = pool_live_peak;
        st->slot_bytes = int64_t(slot_bytes);
        st->pool_bytes = int64_t(slot_bytes) * nslots + int64_t(head_bytes) * nhead;
        st->peer_bytes = peer_bytes;
        double cms = 0;  // stage-boundary pulls: copy-engine time on the copy stream (CUDA events)
        for (size_t j = 0; j < copied.size(); ++j)
            if (copied[j]) {
                float t = 0;
                ck(cudaEventElapsedTime(&t, ev_copy0[j], ev_copy1[j]), "elapsed");
                cms += t;
            }
        st->copy_ms = cms;
        st->kernel_launches = launches;
        double gms = 0;
        for (size_t i = 0; i + 1 < gev_used; i += 2) {
            float t = 0;
            ck(cudaEventElapsedTime(&t, gev[i], gev[i + 1]), "elapsed");
            gms += t;
        }
        st->gemm_ms = gms;
        if (kernel_timing) {
            std::vector<double> ms(klabels.size(), 0.0);
            std::vector<int64_t> cnt(klabels.size(), 0);
            for (size_t i = 0; i + 1 < kev_used; i += 2) {
                float t = 0;
                ck(cudaEventElapsedTime(&t, kev[i], kev[i + 1]), "elapsed");
                ms[kev_label[i / 2]] += t;
                cnt[kev_label[i / 2]] += 1;
            }
            std::string r = "{";
            for (size_t i = 0; i < klabels.size(); ++i) {
                if (i) r += ",";
                r += "\"" + klabels[i] + "\":[" + std::to_string(ms[i]) + "," + std::to_string(cnt[i]) + "]";
            }
            kernel_report = r + "}";
        }
        st->gemm_flops = gemm_flops_acc;
        st->gemm_launches = int64_t(gev_used / 2);
    }
}

// ------------------------------------------------------------------ peers
LocalGroup::~LocalGroup() {
    for (int b = 0; b < 2; ++b) {
        for (auto e : ready_ev[b]) cudaEventDestroy(e);
        for (auto e : ack_ev[b]) cudaEventDestroy(e);
        for (auto e : gdone_ev[b])
            if (e) cudaEventDestroy(e);
        for (auto e : gcopied_ev[b])
            if (e) cudaEventDestroy(e);
    }
}

std::shared_ptr<LocalGroup> make_group(const std::vector<Exec*>& all) {
    auto g = std::make_shared<LocalGroup>();
    const ExecPlan& p = all.front()->plan;
    const size_t n = p.msgs.size();
    auto cuda_of = [&](int dev) {
        for (Exec* e : all)
            if (e->dev == dev) return e->cuda;
        throw std::invalid_argument("connect: missing device");
    };
    for (int b = 0; b < 2; ++b) {
        g->ready_ev[b].resize(n);
        g->ack_ev[b].resize(n);
        for (size_t i = 0; i < n; ++i) {
            ck(cudaSetDevice(cuda_of(p.msgs[i].src_dev)), "cudaSetDevice");
            ck(cudaEventCreateWithFlags(&g->ready_ev[b][i], cudaEventDisableTiming), "event");
            ck(cudaSetDevice(cuda_of(p.msgs[i].dst_dev)), "cudaSetDevice");
            ck(cudaEventCreateWithFlags(&g->ack_ev[b][i], cudaEventDisableTiming), "event");
        }
    }
    g->ready_step.assign(n, -1);
    g->ack_step.assign(n, -1);
    g->enqueued.assign(size_t(p.topo.devices) + 1, 0);
    for (Exec* e : all) g->enqueued[e->dev] = e->steps_done;
    g->execs.assign(size_t(p.topo.devices) + 1, nullptr);
    for (Exec* e : all) g->execs[size_t(e->dev)] = e;
    if (all.front()->twin) {
        for (int b = 0; b < 2; ++b) {
            g->gdone_ev[b].assign(size_t(p.topo.devices) + 1, nullptr);
            g->gcopied_ev[b].assign(size_t(p.topo.devices) + 1, nullptr);
            for (Exec* e : all) {
                ck(cudaSetDevice(e->cuda), "cudaSetDevice");
                ck(cudaEventCreateWithFlags(&g->gdone_ev[b][size_t(e->dev)], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&g->gcopied_ev[b][size_t(e->dev)], cudaEventDisableTiming), "event");
            }
        }
        g->gdone_step.assign(size_t(p.topo.devices) + 1, -1);
        g->gcopied_step.assign(size_t(p.topo.devices) + 1, -1);
    }
    return g;
}

void Exec::connect_local(const std::vector<Exec*>& all, std::shared_ptr<LocalGroup> grp) {
    if (int(all.size()) != plan.topo.devices) throw std::invalid_argument("connect: need one exec per device");
    group = std::move(grp);
    for (Exec* e : all)
        if (e != this && e->cuda == cuda) shares_gpu = true;
    for (Exec* e : all) {
        if (e->plan.ops.size() != plan.ops.size()) throw std::invalid_argument("connect: executors run different plans");
        peers[e->dev] = Peer{e->outbox, e->flags, false};
        if (e->cuda != cuda) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, cuda, e->cuda);
            if (!can) throw CudaError("no peer access between GPUs " + std::to_string(cuda) + " and " + std::to_string(e->cuda));
            cudaSetDevice(cuda);
            cudaError_t r = cudaDeviceEnablePeerAccess(e->cuda, 0);
            if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) ck(r, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    }
    if (twin) {  // pair every local tensor "s<s>.<rest>" with "s<partner>.<rest>" on the replica device
        const Exec* peer = nullptr;
        for (Exec* e : all)
            if (e->dev == replica_dev) peer = e;
        if (!peer) throw std::invalid_argument("connect: replica device missing");
        std::map<std::string, const PTensor*> by_name;
        for (const auto& q : peer->ptensors) by_name[q.name] = &q;
        replica_map.clear();
        for (const auto& q : ptensors) {
            const size_t dot = q.name.find('.');
            const int s = std::stoi(q.name.substr(1, dot - 1));
            const int ps = s > Sm ? s - Sm : s + Sm;
            auto it = by_name.find("s" + std::to_string(ps) + q.name.substr(dot));
            if (it == by_name.end() || it->second->numel != q.numel)
                throw std::invalid_argument("connect: replica of " + q.name + " not found");
            replica_map.push_back({q.off, it->second->off, q.numel});
        }
    }
    connected = true;
}

// Twin topologies: the two copies of every model stage sum their gradients before the optimizer
// (gems / chimera train two weight replicas data-parallel).  Host-ordered like the message events:
// record "gradients final" -> pull the replica device's arena -> record "pulled" -> wait until the
// replica device has pulled ours -> add its arena into ours, tensor by tensor.
void Exec::sync_replicas(int64_t t) {
    if (!group) throw StateError("replicated-weight schedules need an in-process pipeline (connect_local)");
    const size_t b = size_t(t & 1), me = size_t(dev), pd = size_t(replica_dev);
    const Exec* peer = group->execs[pd];
    ck(cudaEventRecord(group->gdone_ev[b][me], cs), "event");
    group->set(group->gdone_step, me, t);
    group->wait([&] { return group->gdone_step[pd] >= t; });
    ck(cudaStreamWaitEvent(cs, group->gdone_ev[b][pd], 0), "wait");
    if (peer->cuda == cuda)
        ck(cudaMemcpyAsync(rtmp, peer->grads, n_params * 4, cudaMemcpyDeviceToDevice, cs), "replica copy");
    else
        ck(cudaMemcpyPeerAsync(rtmp, cuda, peer->grads, peer->cuda, n_params * 4, cs), "replica copy");
    ck(cudaEventRecord(group->gcopied_ev[b][me], cs), "event");
    group->set(group->gcopied_step, me, t);
    group->wait([&] { return group->gcopied_step[pd] >= t; });
    ck(cudaStreamWaitEvent(cs, group->gcopied_ev[b][pd], 0), "wait");
    timed("replica_sync", [&] {
        for (const auto& r : replica_map) pbk::grad_add(grads + r[0], rtmp + r[1], r[2], cs);
    });
    launches += int64_t(replica_map.size());
}

struct IpcBlob {
    uint32_t magic;
    int32_t device;
    int32_t cuda;
    uint64_t plan_ops;
    cudaIpcMemHandle_t outbox, flags;
    unsigned char uuid[16];  // physical GPU: ranks on the same GPU share its SMs (shares_gpu)
};

static void gpu_uuid(int cuda, unsigned char out[16]) {
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, cuda), "cudaGetDeviceProperties");
    std::memcpy(out, &prop.uuid, 16);
}

size_t Exec::export_blob(void* buf, size_t cap) {
    IpcBlob b{};
    b.magic = 0x50423230;
    b.device = dev;
    b.cuda = cuda;
    b.plan_ops = plan.ops.size();
    gpu_uuid(cuda, b.uuid);
    ck(cudaSetDevice(cuda), "cudaSetDevice");
    ck(cudaIpcGetMemHandle(&b.outbox, outbox), "cudaIpcGetMemHandle");
    ck(cudaIpcGetMemHandle(&b.flags, flags), "cudaIpcGetMemHandle");
    if (buf) {
        if (cap < sizeof b) throw Space("blob buffer too small");
        std::memcpy(buf, &b, sizeof b);
    }
    return sizeof b;
}

void Exec::connect_ipc(const std::vector<std::pair<const void*, size_t>>& blobs) {
    if (connected) throw StateError("connect_ipc: already connected");
    if (twin)
        throw std::invalid_argument(
            "connect_ipc: replicated-weight (twin: gems / chimera) schedules run with in-process pipelines only");
    if (int(blobs.size()) != plan.topo.devices) throw std::invalid_argument("connect_ipc: need one blob per device");
    ck(cudaSetDevice(cuda), "cudaSetDevice");
    // validate everything before mapping anything: each device 1..D exactly once, same plan
    std::vector<IpcBlob> bs(blobs.size());
    std::vector<int> seen(size_t(plan.topo.devices) + 1, 0);
    for (size_t i = 0; i < blobs.size(); ++i) {
        if (!blobs[i].first || blobs[i].second < sizeof(IpcBlob)) throw std::invalid_argument("connect_ipc: short blob");
        std::memcpy(&bs[i], blobs[i].first, sizeof(IpcBlob));
        const IpcBlob& b = bs[i];
        if (b.magic != 0x50423230 || b.plan_ops != plan.ops.size()) throw std::invalid_argument("connect_ipc: bad blob");
        if (b.device < 1 || b.device > plan.topo.devices || seen[size_t(b.device)]++)
            throw std::invalid_argument("connect_ipc: device " + std::to_string(b.device) +
                                        " missing, duplicated or out of range in the blob set");
    }
    if (!seen[size_t(dev)]) throw std::invalid_argument("connect_ipc: this device's own blob is missing");
    unsigned char mine[16];
    gpu_uuid(cuda, mine);
    for (const IpcBlob& b : bs)
        if (b.device != dev && std::memcmp(b.uuid, mine, 16) == 0) shares_gpu = true;
    for (const IpcBlob& b : bs) {
        if (b.device == dev) continue;
        // only neighbours exchange messages, but every peer is mapped (cheap)
        void *ob = nullptr, *fl = nullptr;
        ck(cudaIpcOpenMemHandle(&ob, b.outbox, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        ck(cudaIpcOpenMemHandle(&fl, b.flags, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        peers[b.device] = Peer{ob, static_cast<uint32_t*>(fl), true};
    }
    connected = true;
}

}  // namespace pbx
