// Memory-bound kernels of a pipeline stage: RMSNorm fwd/bwd (+ gamma grads),
// embedding gather / scatter-add, fused LM-head softmax cross-entropy
// (loss + dlogits in place), AdamW.  128-bit vector I/O, warp-shuffle
// reductions, one row per warp where a row fits.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "ops.hpp"
#include "sm100.cuh"

namespace pbk {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int k = 16; k; k >>= 1) v += __shfl_xor_sync(0xffffffff, v, k);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int k = 16; k; k >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, k));
    return v;
}
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) f[2 * i] = bf16_lo(w[i]), f[2 * i + 1] = bf16_hi(w[i]);
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}

// block-wide sum; every thread gets the result (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = lane < nw ? red[lane] : 0.f;
    t = warp_sum(t);
    __syncthreads();
    return t;
}

// y = x * rsqrt(mean(x^2) + eps) * g (g null: 1) ; one CTA per row, one 16-byte chunk per thread held in registers
__global__ void rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                                   __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int T, int h, float eps) {
    pdl_wait();
    pdl_launch();
    __shared__ float red[32];
    const int row = blockIdx.x, c = threadIdx.x;
    float f[8], w[8] = {1, 1, 1, 1, 1, 1, 1, 1};
    unpack8(reinterpret_cast<const uint4*>(x + size_t(row) * h)[c], f);
    if (g) unpack8(reinterpret_cast<const uint4*>(g)[c], w);
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss += f[i] * f[i];
    ss = block_sum(ss, red);
    const float r = rsqrtf(ss / float(h) + eps);
    if (c == 0) rstd[row] = r;
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = f[i] * r * w[i];
    reinterpret_cast<uint4*>(y + size_t(row) * h)[c] = pack8(f);
}

// dx = dres + r*g*dy - x * r^3/h * sum(g*dy*x) ; one CTA per row
__global__ void rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd,
                                   const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx, int T,
                                   int h) {
    pdl_wait();
    pdl_launch();
    __shared__ float red[32];
    const int row = blockIdx.x, c = threadIdx.x;
    float a[8], b[8], w[8] = {1, 1, 1, 1, 1, 1, 1, 1}, o[8];
    unpack8(reinterpret_cast<const uint4*>(dy + size_t(row) * h)[c], a);
    unpack8(reinterpret_cast<const uint4*>(x + size_t(row) * h)[c], b);
    if (g) unpack8(reinterpret_cast<const uint4*>(g)[c], w);
    if (dres) {
        unpack8(reinterpret_cast<const uint4*>(dres + size_t(row) * h)[c], o);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = 0.f;
    }
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) dot += w[i] * a[i] * b[i];
    dot = block_sum(dot, red);
    const float k = dot * r * r * r / float(h);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] += r * w[i] * a[i] - b[i] * k;
    reinterpret_cast<uint4*>(dx + size_t(row) * h)[c] = pack8(o);
}

// ---- RMSNorm folded into the neighbouring GEMMs (executor.cpp, fold mode).  The forward never
// materialises the normalised rows: the producer's residual epilogue accumulates ss = sum x^2, the
// consumer GEMM scales its accumulator rows by rstd = rsqrt(ss / h + eps).  Only a stage's input
// (pulled from the previous stage or embedded) needs this standalone statistic.
// ss[row] = sum_c x[row, c]^2, bit-identical to the residual GEMM epilogue's statistic (gemm_tc.cu):
// one fp32 partial per 128 columns accumulated pair by pair in column order as
// fmaf(lo, lo, fmaf(hi, hi, acc)), then the partials summed in column order.
// Block = 4 rows x P threads (P = h / 128 <= 64), thread = one 128-column chunk.
__global__ void __launch_bounds__(256) row_sumsq_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ ss,
                                                        int T, int h) {
    pdl_wait();
    pdl_launch();
    __shared__ float part[256];
    const int P = h >> 7;
    const int r = int(threadIdx.x) / P, q = int(threadIdx.x) % P;
    const int row = blockIdx.x * 4 + r;
    if (r < 4 && row < T) {
        const uint4* xr = reinterpret_cast<const uint4*>(x + size_t(row) * h + q * 128);
        float acc = 0.f;
#pragma unroll 4
        for (int c = 0; c < 16; ++c) {
            const uint4 v = xr[c];
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float lo = bf16_lo(w[e]), hi = bf16_hi(w[e]);
                acc = fmaf(lo, lo, fmaf(hi, hi, acc));
            }
        }
        part[threadIdx.x] = acc;
    }
    __syncthreads();
    if (r < 4 && q == 0 && row < T) {
        float sum = 0.f;
        for (int k = 0; k < P; ++k) sum += part[threadIdx.x + k];
        ss[row] = sum;
    }
}

// Backward of y = rstd * x (gamma folded away) given dy' = rstd * dy (the consuming projection's
// dX GEMM ran on row-scaled output gradients):  dx = dy' - x * rstd^2 * mean(dy' * x) + dres,
// rstd = rsqrt(ss / h + eps).  One CTA per row, one 16-byte chunk per thread.
__global__ void rmsnorm_bwd_x_kernel(const __nv_bfloat16* __restrict__ dyp, const __nv_bfloat16* __restrict__ x,
                                     const float* __restrict__ ss, const __nv_bfloat16* __restrict__ dres,
                                     __nv_bfloat16* __restrict__ dx, int h, float eps) {
    pdl_wait();
    pdl_launch();
    __shared__ float red[32];
    const int row = blockIdx.x, c = threadIdx.x;
    float a[8], b[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(dyp + size_t(row) * h)[c], a);
    unpack8(reinterpret_cast<const uint4*>(x + size_t(row) * h)[c], b);
    if (dres) {
        unpack8(reinterpret_cast<const uint4*>(dres + size_t(row) * h)[c], o);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = 0.f;
    }
    const float inv_h = 1.f / float(h);
    const float r2 = 1.f / (ss[row] * inv_h + eps);
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) dot = fmaf(a[i], b[i], dot);
    dot = block_sum(dot, red);
    const float k = dot * r2 * inv_h;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] += a[i] - b[i] * k;
    reinterpret_cast<uint4*>(dx + size_t(row) * h)[c] = pack8(o);
}

// The same, one warp per row with the whole row of dy' and x held in registers (NC 16-byte chunks
// per lane, all loads in flight before the warp-shuffle dot; no block barriers): the one-CTA-per-row
// kernel above reached 3.8 TB/s in-step (two __syncthreads per row, one chunk per thread in flight).
template <int NC>
__global__ void __launch_bounds__(128) rmsnorm_bwd_x_warp_kernel(const __nv_bfloat16* __restrict__ dyp,
                                                                 const __nv_bfloat16* __restrict__ x,
                                                                 const float* __restrict__ ss,
                                                                 const __nv_bfloat16* __restrict__ dres,
                                                                 __nv_bfloat16* __restrict__ dx, int T, float eps) {
    pdl_wait();
    pdl_launch();
    constexpr int h = NC * 256;
    const int row = int(blockIdx.x) * 4 + int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    if (row >= T) return;
    const uint4* a4 = reinterpret_cast<const uint4*>(dyp + size_t(row) * h) + lane;
    const uint4* b4 = reinterpret_cast<const uint4*>(x + size_t(row) * h) + lane;
    uint4 a[NC], b[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) a[k] = a4[32 * k], b[k] = b4[32 * k];
    const float ssr = ss[row];
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float fa[8], fb[8];
        unpack8(a[k], fa);
        unpack8(b[k], fb);
#pragma unroll
        for (int i = 0; i < 8; ++i) dot = fmaf(fa[i], fb[i], dot);
    }
    dot = warp_sum(dot);
    const float inv_h = 1.f / float(h);
    const float kk = dot * inv_h / (ssr * inv_h + eps);
    const uint4* r4 = dres ? reinterpret_cast<const uint4*>(dres + size_t(row) * h) + lane : nullptr;
    uint4* o4 = reinterpret_cast<uint4*>(dx + size_t(row) * h) + lane;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float fa[8], fb[8], o[8];
        unpack8(a[k], fa);
        unpack8(b[k], fb);
        if (r4) {
            unpack8(r4[32 * k], o);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] += fa[i] - fb[i] * kk;
        o4[32 * k] = pack8(o);
    }
}


// dgamma[j] += sum_t dy[t,j] * x[t,j] * rstd[t], deterministic two-stage column reduction:
// stage 1: thread = 8 columns x `rows_per_block` rows -> partial[row_block][h] (no atomics)
__global__ void rmsnorm_dgamma_partial_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                                              const float* __restrict__ rstd, float* __restrict__ partial, int T,
                                              int h, int rows_per_block) {
    pdl_wait();
    pdl_launch();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;  // 8-column chunk
    if (c * 8 >= h) return;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(T, r0 + rows_per_block);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int row = r0;
    for (; row + 4 <= r1; row += 4) {
        uint4 ua[4], ub[4];
        float rr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            ua[u] = reinterpret_cast<const uint4*>(dy + size_t(row + u) * h)[c];
            ub[u] = reinterpret_cast<const uint4*>(x + size_t(row + u) * h)[c];
            rr[u] = rstd[row + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float a[8], b[8];
            unpack8(ua[u], a);
            unpack8(ub[u], b);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += a[i] * b[i] * rr[u];
        }
    }
    for (; row < r1; ++row) {
        float a[8], b[8];
        unpack8(reinterpret_cast<const uint4*>(dy + size_t(row) * h)[c], a);
        unpack8(reinterpret_cast<const uint4*>(x + size_t(row) * h)[c], b);
        const float r = rstd[row];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += a[i] * b[i] * r;
    }
    float4* dst = reinterpret_cast<float4*>(partial + size_t(blockIdx.y) * h + c * 8);
    dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

// stage 2: dgamma[j] += sum over row blocks; block = 32 columns x 8 row groups, fixed reduction order
__global__ void rmsnorm_dgamma_sum_kernel(const float* __restrict__ partial, float* __restrict__ dgamma, int nb,
                                          int h) {
    pdl_wait();
    pdl_launch();
    __shared__ float red[8][33];
    const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + cl;
    float s = 0.f;
    if (j < h) {
#pragma unroll 4
        for (int b = g; b < nb; b += 8) s += partial[size_t(b) * h + j];
    }
    red[g][cl] = s;
    __syncthreads();
    if (g == 0 && j < h) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += red[k][cl];
        dgamma[j] += t;
    }
}

// Token / label ids come through the public C-ABI: an id outside [0, V) never indexes memory.
// The row is zeroed (embed_fwd) or skipped (embed_bwd, CE) and *err is set; the executor turns
// the flag into PB_EINVAL when the step is synchronised.
__device__ __forceinline__ bool id_ok(int32_t id, int V, int* err) {
    if (id >= 0 && id < V) return true;
    if (err) atomicOr(err, 1);
    return false;
}

__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ emb,
                                 __nv_bfloat16* __restrict__ x, int T, int h, int V, int* err) {
    pdl_wait();
    pdl_launch();
    const int row = blockIdx.x;
    const int32_t id = tok[row];
    uint4* dst = reinterpret_cast<uint4*>(x + size_t(row) * h);
    if (!id_ok(id, V, threadIdx.x == 0 ? err : nullptr)) {
        for (int c = threadIdx.x; c < (h >> 3); c += blockDim.x) dst[c] = make_uint4(0, 0, 0, 0);
        return;
    }
    const uint4* src = reinterpret_cast<const uint4*>(emb + size_t(id) * h);
    for (int c = threadIdx.x; c < (h >> 3); c += blockDim.x) dst[c] = src[c];
}

__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ dx,
                                 float* __restrict__ demb, int T, int h, int V, int* err) {
    pdl_wait();
    pdl_launch();
    const int row = blockIdx.x;
    const int32_t id = tok[row];
    if (!id_ok(id, V, threadIdx.x == 0 ? err : nullptr)) return;
    float* dst = demb + size_t(id) * h;
    const uint4* src = reinterpret_cast<const uint4*>(dx + size_t(row) * h);
    for (int c = threadIdx.x; c < (h >> 3); c += blockDim.x) {
        float f[8];
        unpack8(src[c], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(dst + c * 8 + i, f[i]);
    }
}

// one block per row: loss += (lse - z[label]) * scale ; z <- (softmax(z) - onehot) * scale  (bf16, in place)
__global__ void __launch_bounds__(512) ce_kernel(__nv_bfloat16* __restrict__ logits, const int32_t* __restrict__ labels,
                                                 float* __restrict__ loss, int V, float scale, int* err,
                                                 const float* __restrict__ rs, float rs_inv_n, float rs_eps) {
    pdl_wait();
    pdl_launch();
    __shared__ float red[32];
    const int row = blockIdx.x;
    __nv_bfloat16* z = logits + size_t(row) * V;
    const int nch = V >> 3;
    uint4* z4 = reinterpret_cast<uint4*>(z);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    float m = -INFINITY;
#pragma unroll 4  // four chunks' loads in flight per thread
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
        float f[8];
        unpack8(z4[c], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmaxf(m, f[i]);
    }
    m = warp_max(m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (warp == 0) {
        float v = lane < nw ? red[lane] : -INFINITY;
        v = warp_max(v);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    float s = 0.f;
#pragma unroll 4  // four chunks' loads in flight per thread
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
        float f[8];
        unpack8(z4[c], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += __expf(f[i] - m);
    }
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (warp == 0) {
        float v = lane < nw ? red[lane] : 0.f;
        v = warp_sum(v);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    s = red[0];
    const int lab = labels[row];
    const bool lab_ok = id_ok(lab, V, threadIdx.x == 0 ? err : nullptr);  // bad label: no loss, no one-hot
    const float zl = lab_ok ? __bfloat162float(z[lab]) : 0.f;
    __syncthreads();
    const float inv = 1.f / s;
    // folded final RMSNorm: dlogits' = rstd_f * dlogits (the head's dX and dW GEMMs then use x, not x-hat)
    const float gsc = rs ? scale * rsqrtf(rs[row] * rs_inv_n + rs_eps) : scale;
#pragma unroll 4  // four chunks' loads in flight per thread
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
        float f[8];
        unpack8(z4[c], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float p = __expf(f[i] - m) * inv;
            if (c * 8 + i == lab) p -= 1.f;
            f[i] = p * gsc;
        }
        z4[c] = pack8(f);
    }
    if (threadIdx.x == 0 && lab_ok) atomicAdd(loss, (m + __logf(s) - zl) * scale);
}

// AdamW on fp32 masters; refreshes the bf16 copy and zeroes the gradient.
__global__ void adamw_kernel(float* __restrict__ w, __nv_bfloat16* __restrict__ wb, float* __restrict__ gr,
                             float* __restrict__ m, float* __restrict__ v, size_t n, float lr, float b1, float b2,
                             float eps, float wd, float bc1, float bc2) {
    pdl_wait();
    pdl_launch();
    size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    const size_t stride = size_t(gridDim.x) * blockDim.x * 4;
    for (; i < n; i += stride) {
        float4 W = *reinterpret_cast<float4*>(w + i), G = *reinterpret_cast<float4*>(gr + i);
        float4 M = *reinterpret_cast<float4*>(m + i), Vv = *reinterpret_cast<float4*>(v + i);
        float* wp = &W.x;
        float* gp = &G.x;
        float* mp = &M.x;
        float* vp = &Vv.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            mp[k] = b1 * mp[k] + (1.f - b1) * gp[k];
            vp[k] = b2 * vp[k] + (1.f - b2) * gp[k] * gp[k];
            const float mh = mp[k] / bc1, vh = vp[k] / bc2;
            wp[k] -= lr * (mh / (sqrtf(vh) + eps) + wd * wp[k]);
        }
        *reinterpret_cast<float4*>(w + i) = W;
        *reinterpret_cast<float4*>(m + i) = M;
        *reinterpret_cast<float4*>(v + i) = Vv;
        *reinterpret_cast<float4*>(gr + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<uint2*>(wb + i) = make_uint2(pack_bf16(W.x, W.y), pack_bf16(W.z, W.w));
    }
}

// RMSNorm gamma folded into the following projection (Y = (x^ * g) W^T = x^ (W diag g)^T):
// Wb[i][j] = bf16(W[i][j] * g[j]) for a row-major [rows][cols] weight.
__global__ void fold_weight_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                   __nv_bfloat16* __restrict__ wb, size_t n, int cols) {
    pdl_wait();
    pdl_launch();
    size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    const size_t stride = size_t(gridDim.x) * blockDim.x * 4;
    for (; i < n; i += stride) {
        const float4 a = *reinterpret_cast<const float4*>(w + i);
        const float4 b = *reinterpret_cast<const float4*>(g + (i % size_t(cols)));
        *reinterpret_cast<uint2*>(wb + i) = make_uint2(pack_bf16(a.x * b.x, a.y * b.y), pack_bf16(a.z * b.z, a.w * b.w));
    }
}

// Gradients of a folded pair from dW' (the accumulated gradient w.r.t. W diag g), once per step:
//   dW += dW' * g[j],  dg[j] += sum_i dW'[i][j] * W[i][j],  dW' <- 0.
// Stage 1: thread = 4 columns x `rows_per_block` rows -> partial[row_block][cols] (deterministic).
__global__ void fold_grad_partial_kernel(float* __restrict__ dwp, const float* __restrict__ w,
                                         const float* __restrict__ g, float* __restrict__ dw,
                                         float* __restrict__ partial, int rows, int cols, int rows_per_block) {
    pdl_wait();
    pdl_launch();
    const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
    if (c4 * 4 >= cols) return;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
    const float4 gg = reinterpret_cast<const float4*>(g)[c4];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = r0; r < r1; ++r) {
        const size_t o = size_t(r) * cols + size_t(c4) * 4;
        float4 d = *reinterpret_cast<float4*>(dwp + o);
        const float4 a = *reinterpret_cast<const float4*>(w + o);
        float4 t = *reinterpret_cast<float4*>(dw + o);
        acc.x += d.x * a.x, acc.y += d.y * a.y, acc.z += d.z * a.z, acc.w += d.w * a.w;
        t.x += d.x * gg.x, t.y += d.y * gg.y, t.z += d.z * gg.z, t.w += d.w * gg.w;
        *reinterpret_cast<float4*>(dw + o) = t;
        *reinterpret_cast<float4*>(dwp + o) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    reinterpret_cast<float4*>(partial + size_t(blockIdx.y) * cols)[c4] = acc;
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, size_t n) {
    pdl_wait();
    pdl_launch();
    size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    const size_t stride = size_t(gridDim.x) * blockDim.x * 4;
    for (; i < n; i += stride) {
        float4 a = *reinterpret_cast<const float4*>(src + i);
        *reinterpret_cast<uint2*>(dst + i) = make_uint2(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w));
    }
}

// counter-based N(0, std) init (splitmix64 -> Box-Muller), deterministic in (seed, index)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void init_normal_kernel(float* __restrict__ w, size_t n, uint64_t seed, float std, float constant) {
    pdl_wait();
    pdl_launch();
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (; i < n; i += stride) {
        if (std == 0.f) {
            w[i] = constant;
            continue;
        }
        uint64_t r = mix64(seed * 0x2545F4914F6CDD1Dull + i);
        float u1 = (float((r >> 40) & 0xFFFFFF) + 1.f) * (1.f / 16777217.f);
        float u2 = float((r >> 16) & 0xFFFFFF) * (1.f / 16777216.f);
        w[i] = std * sqrtf(-2.f * __logf(u1)) * __cosf(6.283185307179586f * u2);
    }
}

int grid_for(size_t n, int per_thread, int block) {
    size_t blocks = (n / per_thread + block - 1) / block;
    int cap = num_sms() * 8;
    return int(blocks < size_t(cap) ? (blocks ? blocks : 1) : cap);
}

}  // namespace

void rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y, float* rstd, int T, int h,
                 cudaStream_t s) {
    if (h % 256 || h > 8192) throw std::invalid_argument("rmsnorm: h must be a multiple of 256 and <= 8192");
    launch_k(rmsnorm_fwd_kernel, dim3(T), dim3(h / 8), 0, s, 1, x, g, y, rstd, T, h, 1e-5f);
}

void rmsnorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd,
                 const __nv_bfloat16* dres, __nv_bfloat16* dx, int T, int h, cudaStream_t s) {
    if (h % 256 || h > 8192) throw std::invalid_argument("rmsnorm: h must be a multiple of 256 and <= 8192");
    launch_k(rmsnorm_bwd_kernel, dim3(T), dim3(h / 8), 0, s, 1, dy, x, g, rstd, dres, dx, T, h);
}

// dst[i] += src[i] (fp32, both 16-byte aligned): replica gradients of the twin topologies
__global__ void grad_add_kernel(float* __restrict__ dst, const float* __restrict__ src, size_t n4) {
    pdl_wait();
    pdl_launch();
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
        float4 a = reinterpret_cast<float4*>(dst)[i];
        const float4 b = reinterpret_cast<const float4*>(src)[i];
        a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
        reinterpret_cast<float4*>(dst)[i] = a;
    }
}

void grad_add(float* dst, const float* src, size_t n, cudaStream_t s) {
    if (n % 4 || (reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) % 16)
        throw std::invalid_argument("grad_add: 16-byte aligned float4 ranges expected");
    const size_t n4 = n / 4;
    const unsigned blocks = unsigned(std::min<size_t>((n4 + 255) / 256, 148 * 8));
    launch_k(grad_add_kernel, dim3(blocks), dim3(256), 0, s, 1, dst, src, n4);
}

void row_sumsq(const __nv_bfloat16* x, float* ss, int T, int h, cudaStream_t s) {
    if (h % 128 || h > 8192) throw std::invalid_argument("row_sumsq: h must be a multiple of 128 and <= 8192");
    launch_k(row_sumsq_kernel, dim3((T + 3) / 4), dim3(4 * (h / 128)), 0, s, 1, x, ss, T, h);
}

void rmsnorm_bwd_x(const __nv_bfloat16* dyp, const __nv_bfloat16* x, const float* ss, const __nv_bfloat16* dres,
                   __nv_bfloat16* dx, int T, int h, float eps, cudaStream_t s) {
    if (h % 256 || h > 8192) throw std::invalid_argument("rmsnorm: h must be a multiple of 256 and <= 8192");
    const dim3 g4((T + 3) / 4), b4(128);
    if (h == 2048)  // wider rows spill the register-held row (ptxas: 255 regs + stack at h = 4096)
        launch_k(rmsnorm_bwd_x_warp_kernel<8>, g4, b4, 0, s, 1, dyp, x, ss, dres, dx, T, eps);
    else
        launch_k(rmsnorm_bwd_x_kernel, dim3(T), dim3(h / 8), 0, s, 1, dyp, x, ss, dres, dx, h, eps);
}

void rmsnorm_dgamma(const __nv_bfloat16* dy, const __nv_bfloat16* x, const float* rstd, float* dgamma, float* scratch,
                    int T, int h, cudaStream_t s) {
    const int rows = 16;
    const int threads = std::min(256, h / 8);
    const int nb = (T + rows - 1) / rows;
    dim3 grid((h / 8 + threads - 1) / threads, nb);
    launch_k(rmsnorm_dgamma_partial_kernel, grid, dim3(threads), 0, s, 1, dy, x, rstd, scratch, T, h, rows);
    launch_k(rmsnorm_dgamma_sum_kernel, dim3((h + 31) / 32), dim3(256), 0, s, 1, static_cast<const float*>(scratch),
             dgamma, nb, h);
}

void embed_fwd(const int32_t* tok, const __nv_bfloat16* emb, __nv_bfloat16* x, int T, int h, int V, int* err,
               cudaStream_t s) {
    launch_k(embed_fwd_kernel, dim3(T), dim3(128), 0, s, 1, tok, emb, x, T, h, V, err);
}
void embed_bwd(const int32_t* tok, const __nv_bfloat16* dx, float* demb, int T, int h, int V, int* err,
               cudaStream_t s) {
    launch_k(embed_bwd_kernel, dim3(T), dim3(128), 0, s, 1, tok, dx, demb, T, h, V, err);
}
void cross_entropy(__nv_bfloat16* logits, const int32_t* labels, float* loss, int T, int V, float scale, int* err,
                   cudaStream_t s, const float* rs, float rs_inv_n, float rs_eps) {
    if (V % 8) throw std::invalid_argument("cross_entropy: V % 8");
    launch_k(ce_kernel, dim3(T), dim3(512), 0, s, 1, logits, labels, loss, V, scale, err, rs, rs_inv_n, rs_eps);
}
void adamw(float* w, __nv_bfloat16* wb, float* g, float* m, float* v, size_t n, float lr, float b1, float b2,
           float eps, float wd, int step, cudaStream_t s) {
    if (n % 4) throw std::invalid_argument("adamw: n % 4");
    const float bc1 = 1.f - powf(b1, float(step)), bc2 = 1.f - powf(b2, float(step));
    launch_k(adamw_kernel, dim3(grid_for(n, 4, 256)), dim3(256), 0, s, 1, w, wb, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2);
}
void fold_weight(const float* w, const float* g, __nv_bfloat16* wb, int rows, int cols, cudaStream_t s) {
    if (cols % 4) throw std::invalid_argument("fold_weight: cols % 4");
    const size_t n = size_t(rows) * cols;
    launch_k(fold_weight_kernel, dim3(grid_for(n, 4, 256)), dim3(256), 0, s, 1, w, g, wb, n, cols);
}
void fold_grad(float* dwp, const float* w, const float* g, float* dw, float* dg, float* scratch, size_t scratch_floats,
               int rows, int cols, cudaStream_t s) {
    if (cols % 128) throw std::invalid_argument("fold_grad: cols % 128");
    int rpb = 64;
    while (size_t((rows + rpb - 1) / rpb) * cols > scratch_floats) rpb *= 2;
    const int nb = (rows + rpb - 1) / rpb;
    const int threads = std::min(128, cols / 4);
    dim3 grid((cols / 4 + threads - 1) / threads, nb);
    launch_k(fold_grad_partial_kernel, grid, dim3(threads), 0, s, 1, dwp, w, g, dw, scratch, rows, cols, rpb);
    launch_k(rmsnorm_dgamma_sum_kernel, dim3((cols + 31) / 32), dim3(256), 0, s, 1, static_cast<const float*>(scratch),
             dg, nb, cols);
}
void f32_to_bf16(const float* src, __nv_bfloat16* dst, size_t n, cudaStream_t s) {
    launch_k(f32_to_bf16_kernel, dim3(grid_for(n, 4, 256)), dim3(256), 0, s, 1, src, dst, n);
}
void init_normal(float* w, size_t n, uint64_t seed, float std, float constant, cudaStream_t s) {
    launch_k(init_normal_kernel, dim3(grid_for(n, 1, 256)), dim3(256), 0, s, 1, w, n, seed, std, constant);
}

}  // namespace pbk
