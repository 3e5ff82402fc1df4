// Device-side runtime of one pipeline device (see executor.cpp).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <array>
#include <condition_variable>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "capi_common.hpp"
#include "kernels/ops.hpp"
#include "plan.hpp"

namespace pbx {

constexpr float kNormEps = 1e-5f;  // RMSNorm epsilon (oracle/numerics.py rmsnorm)

struct LayerSlots {  // byte offsets inside an activation slot
    size_t a, qkv, o, x1, b, u, gl, dqkv, dx1, rstd1, rstd2, lse;  // a, b, rstd1/2: unfolded path only
    size_t ss1, ss2;  // fold mode: per-token sum of squares of x (norm1) and x1 (norm2)
};
struct StageLayout {
    std::vector<size_t> x, dx;  // Lc+1 residual-stream buffers and their gradients
    std::vector<LayerSlots> layer;
    size_t hf = 0, rstdf = 0, logits = 0;  // hf, rstdf: unfolded path only
    size_t ss = 0, ss_bytes = 0, ssf = 0;   // fold mode: the stage's sum-of-squares block, final norm's
    size_t bytes = 0;
};
struct LayerParams {
    size_t g1, wqkv, wo, g2, w1, w2;  // indices into ptensors
};
struct StageParams {
    std::vector<LayerParams> layers;
    size_t emb = 0, gf = 0, head = 0;
};
struct PTensor {
    std::string name;
    size_t off, numel;
    int id;
    float std, constant;
};
// RMSNorm gamma folded into the projection that consumes the normalised rows:
// the GEMM operand is bf16(W diag g), its gradient dW' accumulates in `gfold`, and
// dW / dg are recovered once per step (executor.cpp fold_grads).
struct FoldPair {
    size_t w, g;  // ptensor indices
    int rows, cols;
    size_t off;   // into gfold
};
struct Peer {
    void* outbox = nullptr;
    uint32_t* flags = nullptr;
    bool ipc = false;
};

class Exec;

// In-process peer group: message hand-off through CUDA events whose records are
// host-ordered before any wait on them (double-buffered by step parity), so no
// stream ever waits on work that is not yet submitted.
struct LocalGroup {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<cudaEvent_t> ready_ev[2], ack_ev[2];  // per message
    std::vector<int64_t> ready_step, ack_step;        // last step whose record is enqueued
    std::vector<int64_t> enqueued;                    // per device: steps fully enqueued
    // twin topologies (gems / chimera): replica-gradient exchange at the end of a step, per device
    std::vector<Exec*> execs;                         // [device]
    std::vector<cudaEvent_t> gdone_ev[2], gcopied_ev[2];
    std::vector<int64_t> gdone_step, gcopied_step;
    // PB_FLAG_ISOLATE: one pass at a time on the whole group (GPU token), passes done this step
    std::mutex iso_mu;
    int64_t iso_step = -1, iso_done = 0;
    void wait(const std::function<bool()>& pred) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, pred);
    }
    void set(std::vector<int64_t>& v, size_t i, int64_t t) {
        {
            std::lock_guard<std::mutex> lk(mu);
            v[i] = t;
        }
        cv.notify_all();
    }
    ~LocalGroup();
};

class Exec {
  public:
    Exec(const pb_model_cfg& cfg, const vsched::Grid& grid, int device, int cuda_dev);
    ~Exec();
    void init(int device);
    void release() noexcept;
    bool released = false;
    void connect_local(const std::vector<Exec*>& all, std::shared_ptr<LocalGroup> grp);
    size_t export_blob(void* buf, size_t cap);
    void connect_ipc(const std::vector<std::pair<const void*, size_t>>& blobs);
    void enqueue(const int32_t* tok, const int32_t* lab, bool on_host);
    void finish(pb_timed_pass* tl, size_t tl_n, pb_exec_stats* st);

    pb_model_cfg cfg;
    ExecPlan plan;
    int dev, cuda;
    int S = 0, T = 0, h = 0, H = 0, V = 0, seq = 0, mbs = 0, m = 0;
    std::vector<int> stage_L, stage_first;  // [stage] layers held, global index of its first layer
    // twin topology (gems / chimera): stages d+k replicate model stage k (weights, init, names' layers);
    // the first / last stage of each route carries the embedding / LM head
    bool twin = false;
    int Sm = 0;  // model stages (S, or d for twin)
    int model_stage(int s) const { return twin && s > Sm ? s - Sm : s; }
    bool is_first(int s) const { return model_stage(s) == 1; }
    bool is_last(int s) const { return model_stage(s) == Sm; }
    // replica gradients: the device holding the replicas of this device's stages, the (dst, src, n)
    // element ranges that pair each local tensor with its replica in that device's arena, and a
    // receive buffer for the replica's gradient arena
    int replica_dev = 0;
    std::vector<std::array<size_t, 3>> replica_map;
    float* rtmp = nullptr;
    void sync_replicas(int64_t t);
    std::vector<int> stages;
    std::vector<PTensor> ptensors;
    float *master = nullptr, *grads = nullptr, *adam_m = nullptr, *adam_v = nullptr;
    __nv_bfloat16* wts = nullptr;
    size_t n_params = 0;
    cudaStream_t cs = nullptr, xs = nullptr;
    bool shares_gpu = false;  // another pipeline device of the group runs on the same GPU
    bool timeline = true, serial = false, isolate = false, connected = false, pending = false, gemm_timing = false, kernel_timing = false;
    // PB_FLAG_SOLO: run this device's op list alone — cross-device inputs are not pulled (the receive
    // slot keeps its contents) and outputs are not signalled — at the device's real memory footprint
    bool solo = false;
    // device memory: executor allocations per category (dmalloc) and cudaMemGetInfo samples
    std::map<std::string, size_t> mem_alloc;
    size_t mem_alloc_total = 0, mem_device_total = 0, mem_used_at_create = 0, mem_used_high = 0;
    void sample_device_memory();
    int adam_step = 0;

    int64_t steps_done = 0;
    std::string kernel_report;

  private:
    void build_layout();
    void build_params();
    __nv_bfloat16* bf(int slot, size_t off) const;
    float* f32(int slot, size_t off) const;
    __nv_bfloat16* outbox_ptr(int k) const;
    const __nv_bfloat16* W(size_t p) const { return wts + ptensors[p].off; }
    float* G(size_t p) const { return grads + ptensors[p].off; }
    // rs: folded-RMSNorm row statistic of the A rows (sum of squares over h); ss_out: residual epilogue's
    // sum of squares of the output rows (the next norm's statistic)
    void gemm(int M, int N, int K, const __nv_bfloat16* A, bool a_mn, const __nv_bfloat16* B, bool b_mn, void* C,
              int epi, const __nv_bfloat16* aux = nullptr, void* C2 = nullptr, int accumulate = 0,
              const float* rs = nullptr, float* ss_out = nullptr);
    void pass_forward(int s, int mb, int slot, __nv_bfloat16* out);
    void pass_backward(int s, int mb, int slot, __nv_bfloat16* out);
    void pass_weight(int s, int mb, int slot);
    uint32_t gen_total(const Msg& m) const;
    uint32_t* ack_flag(uint32_t* base, int k) const;
    uint32_t* ready_flag(uint32_t* base, int src, int k) const;

    void build_w_groups();
    float* GW(size_t p) const;  // where the W pass accumulates tensor p's gradient (dW' if folded)
    void fold_grads();
  public:
    void refold();  // wts of folded pairs <- bf16(W diag g) from the masters
  private:
    bool fold = true;
    std::vector<FoldPair> folds;
    std::map<size_t, size_t> fold_of;  // ptensor index of W -> folds index
    float* gfold = nullptr;
    void run_gemm_timed(const char* label, double flops, const std::function<void()>& fn);
    std::map<std::pair<int, int>, pbk::GemmGroup> wgroups;  // (stage, slot) -> grouped W GEMMs
    std::map<std::pair<int, int>, double> wgroup_flops;
    std::map<int, StageLayout> layout;
    std::map<int, StageParams> sparams;
    size_t slot_bytes = 0, head_bytes = 0, msg_bytes = 0, nflags = 0;
    uint8_t* hpool = nullptr;           // last-stage head buffers (hf, rstd, logits), own lifespan pool
    int nhead = 0;
    std::vector<int> head_slot_mb;      // microbatch -> head slot
    uint8_t* head(int mb, size_t off) const;
    int nslots = 0, nout = 0, pool_live_peak = 0;
    uint8_t* pool = nullptr;
    uint8_t* outbox = nullptr;
    uint32_t* flags = nullptr;
    __nv_bfloat16* scratch = nullptr;
    float *dsum = nullptr, *dq_acc = nullptr, *loss_dev = nullptr, *loss_host = nullptr;
    float* ss_part = nullptr;
    int* ss_cnt = nullptr;
    int* id_err() { return reinterpret_cast<int*>(loss_dev + 1); }  // out-of-range token/label flag
    int32_t *tokens = nullptr, *labels = nullptr;
    std::vector<void*> allocations;
    std::vector<cudaEvent_t> ev_start, ev_end, ev_pull, ev_free, ev_copy0, ev_copy1;
    std::vector<uint8_t> copied;  // this step: op j pulled its input from a peer
    cudaEvent_t ev_step0 = nullptr, ev_step1 = nullptr;
    std::vector<Peer> peers;
    std::vector<int> pos_of;
    std::shared_ptr<LocalGroup> group;
    std::mutex local_iso_mu;
    int64_t launches = 0, peer_bytes = 0;
    std::vector<cudaEvent_t> gev;
    size_t gev_used = 0;
    double gemm_flops_acc = 0;
    // PB_FLAG_KERNEL_TIMING: event pairs around every launch, aggregated per label
    std::vector<cudaEvent_t> kev;
    std::vector<int> kev_label;
    size_t kev_used = 0;
    std::vector<std::string> klabels;
    template <typename Fn>
    void timed(const char* label, Fn&& fn);
};

std::shared_ptr<LocalGroup> make_group(const std::vector<Exec*>& all);

}  // namespace pbx
