// Causal multi-head attention (model.py:317-368), SIMT fp32 path (fp32 parity
// mode, head dims != 64, and the exact backward).
//
// q and k arrive already RoPE-rotated: the QKV GEMM epilogue applies the
// interleaved-pair rotation (model.py:281-288), exactly what the reference's
// full cache stores. The backward applies the transpose rotation to dq/dk
// (model.py:291-298). Forward keeps only the per-row log-sum-exp; backward
// recomputes scores. One CTA per (sequence, head, 64-query block); each query
// row is owned by 4 threads that split the key loop and merge their
// online-softmax states with warp shuffles.
#pragma once
#include "common.cuh"

namespace mecefo {

struct AttnDev {
  const void* qkv;   // (b, ld_qkv): q at col 0, k at col m, v at col 2m; head h at h*d
  int64_t ld_qkv;
  void* ctx;         // (b, ld_ctx) output (fwd) / O (bwd)
  int64_t ld_ctx;
  const void* dctx;  // (b, ld_ctx) dO (bwd)
  void* dqkv;        // (b, ld_qkv) output (bwd)
  float* lse;        // (b, H)
  float* dsum;       // (b, H) rowsum(dO * O) scratch (bwd)
  const float* cosT; // (T, d/2)
  const float* sinT;
  int T, H, m, rope, prec;
  float scale;       // 1/sqrt(d)
};

template <int D>
__device__ __forceinline__ void rope_rotate(float* v, const AttnDev& a, int pos, float sign) {
  if (!a.rope) return;
#pragma unroll
  for (int p = 0; p < D / 2; ++p) {
    const float c = a.cosT[pos * (D / 2) + p], s = sign * a.sinT[pos * (D / 2) + p];
    const float e = v[2 * p], o = v[2 * p + 1];
    v[2 * p] = e * c - o * s;       // model.py:286
    v[2 * p + 1] = e * s + o * c;   // model.py:287
  }
}

template <int D>
__device__ __forceinline__ void load_head_row(const void* base, int64_t idx, float* v, int prec) {
#pragma unroll
  for (int c = 0; c < D; ++c) v[c] = load_as_f32(base, idx + c, prec);
}

// Stage rows [r0, r1) of one head of a (b, ld) tensor into smem (stride D+4),
// optionally RoPE-rotated and scaled.
template <int D>
__device__ void stage_rows(float* dst, const void* src, int64_t ld, int64_t row_base, int col, int r0, int r1,
                           const AttnDev& a, bool rotate, float mul) {
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    float v[D];
    load_head_row<D>(src, (row_base + r) * ld + col, v, a.prec);
    if (rotate) rope_rotate<D>(v, a, r, 1.f);
#pragma unroll
    for (int c = 0; c < D; ++c) dst[(r - r0) * (D + 4) + c] = v[c] * mul;
  }
}

template <int D>
__global__ void __launch_bounds__(256) attn_fwd_kernel(AttnDev a) {
  griddep_wait();
  extern __shared__ float sm[];
  const int bh = blockIdx.x, seq = bh / a.H, h = bh % a.H;
  const int q0 = blockIdx.y * 64;
  const int kend = min(a.T, q0 + 64);
  float* Ks = sm;
  float* Vs = sm + (size_t)kend * (D + 4);
  const int64_t row_base = (int64_t)seq * a.T;
  stage_rows<D>(Ks, a.qkv, a.ld_qkv, row_base, a.m + h * D, 0, kend, a, false, 1.f);
  stage_rows<D>(Vs, a.qkv, a.ld_qkv, row_base, 2 * a.m + h * D, 0, kend, a, false, 1.f);
  __syncthreads();
  const int i = q0 + (threadIdx.x >> 2), sl = threadIdx.x & 3;
  const bool valid = i < a.T;
  float q[D], o[D];
  if (valid) load_head_row<D>(a.qkv, (row_base + i) * a.ld_qkv + h * D, q, a.prec);
#pragma unroll
  for (int c = 0; c < D; ++c) { q[c] = valid ? q[c] * a.scale : 0.f; o[c] = 0.f; }
  float mx = -INFINITY, l = 0.f;
  if (valid) {
    for (int j = sl; j <= i; j += 4) {
      const float* kj = Ks + j * (D + 4);
      float s = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) s = fmaf(q[c], kj[c], s);
      const float mn = fmaxf(mx, s);
      const float corr = expf(mx - mn);
      const float p = expf(s - mn);
      l = l * corr + p;
      const float* vj = Vs + j * (D + 4);
#pragma unroll
      for (int c = 0; c < D; ++c) o[c] = fmaf(p, vj[c], o[c] * corr);
      mx = mn;
    }
  }
  // merge the 4 key slices of this row
  float M = mx;
  M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
  M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 2));
  const float f = (mx == -INFINITY) ? 0.f : expf(mx - M);
  l *= f;
  l += __shfl_xor_sync(0xffffffffu, l, 1);
  l += __shfl_xor_sync(0xffffffffu, l, 2);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    float v = o[c] * f;
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    o[c] = v;
  }
  if (valid) {
    const float il = 1.f / l;
    constexpr int DQ = (D >= 4) ? D / 4 : 1;
    const int cbeg = sl * DQ;
    const int64_t ob = (row_base + i) * a.ld_ctx + h * D;
#pragma unroll
    for (int c = 0; c < D; ++c)
      if (c >= cbeg && c < cbeg + DQ) store_from_f32(a.ctx, ob + c, o[c] * il, a.prec);
    if (sl == 0 && a.lse) a.lse[(row_base + i) * a.H + h] = M + logf(l);
  }
}

// dQ (and rowsum(dO*O)) for a block of 64 query rows.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(AttnDev a) {
  griddep_wait();
  extern __shared__ float sm[];
  const int bh = blockIdx.x, seq = bh / a.H, h = bh % a.H;
  const int q0 = blockIdx.y * 64;
  const int kend = min(a.T, q0 + 64);
  float* Ks = sm;
  float* Vs = sm + (size_t)kend * (D + 4);
  const int64_t row_base = (int64_t)seq * a.T;
  stage_rows<D>(Ks, a.qkv, a.ld_qkv, row_base, a.m + h * D, 0, kend, a, false, 1.f);
  stage_rows<D>(Vs, a.qkv, a.ld_qkv, row_base, 2 * a.m + h * D, 0, kend, a, false, 1.f);
  __syncthreads();
  const int i = q0 + (threadIdx.x >> 2), sl = threadIdx.x & 3;
  if (i >= a.T) return;  // whole 4-lane groups exit together; no shuffles below cross groups
  float q[D], dO[D], dq[D];
  load_head_row<D>(a.qkv, (row_base + i) * a.ld_qkv + h * D, q, a.prec);
  load_head_row<D>(a.dctx, (row_base + i) * a.ld_ctx + h * D, dO, a.prec);
  float Dsum = 0.f;
  {
    float o[D];
    load_head_row<D>(a.ctx, (row_base + i) * a.ld_ctx + h * D, o, a.prec);
#pragma unroll
    for (int c = 0; c < D; ++c) Dsum = fmaf(dO[c], o[c], Dsum);
  }
  const float lse = a.lse[(row_base + i) * a.H + h];
#pragma unroll
  for (int c = 0; c < D; ++c) { q[c] *= a.scale; dq[c] = 0.f; }
  for (int j = sl; j <= i; j += 4) {
    const float* kj = Ks + j * (D + 4);
    const float* vj = Vs + j * (D + 4);
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int c = 0; c < D; ++c) { s = fmaf(q[c], kj[c], s); dp = fmaf(dO[c], vj[c], dp); }
    const float p = expf(s - lse);
    const float ds = p * (dp - Dsum);  // model.py:352
#pragma unroll
    for (int c = 0; c < D; ++c) dq[c] = fmaf(ds, kj[c], dq[c]);
  }
  const unsigned gmask = 0xFu << (threadIdx.x & 28);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    float v = dq[c];
    v += __shfl_xor_sync(gmask, v, 1);
    v += __shfl_xor_sync(gmask, v, 2);
    dq[c] = v * a.scale;
  }
  rope_rotate<D>(dq, a, i, -1.f);  // transpose rotation, model.py:291-298
  if (sl == 0) {
    const int64_t ob = (row_base + i) * a.ld_qkv + h * D;
#pragma unroll
    for (int c = 0; c < D; ++c) store_from_f32(a.dqkv, ob + c, dq[c], a.prec);
    a.dsum[(row_base + i) * a.H + h] = Dsum;
  }
}

// dK, dV for a block of 64 key rows (queries i >= j).
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_dkv_kernel(AttnDev a) {
  griddep_wait();
  extern __shared__ float sm[];
  const int bh = blockIdx.x, seq = bh / a.H, h = bh % a.H;
  const int k0 = blockIdx.y * 64;
  const int nq = a.T - k0;  // queries k0..T-1
  float* Qs = sm;
  float* Os = sm + (size_t)nq * (D + 4);
  float* Ls = Os + (size_t)nq * (D + 4);
  float* Ds = Ls + nq;
  const int64_t row_base = (int64_t)seq * a.T;
  stage_rows<D>(Qs, a.qkv, a.ld_qkv, row_base, h * D, k0, a.T, a, false, a.scale);
  stage_rows<D>(Os, a.dctx, a.ld_ctx, row_base, h * D, k0, a.T, a, false, 1.f);
  for (int r = threadIdx.x; r < nq; r += blockDim.x) {
    Ls[r] = a.lse[(row_base + k0 + r) * a.H + h];
    Ds[r] = a.dsum[(row_base + k0 + r) * a.H + h];
  }
  __syncthreads();
  const int j = k0 + (threadIdx.x >> 2), sl = threadIdx.x & 3;
  if (j >= a.T) return;
  float k[D], v[D], dk[D], dv[D];
  load_head_row<D>(a.qkv, (row_base + j) * a.ld_qkv + a.m + h * D, k, a.prec);
  load_head_row<D>(a.qkv, (row_base + j) * a.ld_qkv + 2 * a.m + h * D, v, a.prec);
#pragma unroll
  for (int c = 0; c < D; ++c) { dk[c] = 0.f; dv[c] = 0.f; }
  for (int i = j + sl; i < a.T; i += 4) {
    const int r = i - k0;
    const float* qi = Qs + r * (D + 4);
    const float* oi = Os + r * (D + 4);
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int c = 0; c < D; ++c) { s = fmaf(qi[c], k[c], s); dp = fmaf(oi[c], v[c], dp); }
    const float p = expf(s - Ls[r]);
    const float ds = p * (dp - Ds[r]);
#pragma unroll
    for (int c = 0; c < D; ++c) { dv[c] = fmaf(p, oi[c], dv[c]); dk[c] = fmaf(ds, qi[c], dk[c]); }
  }
  const unsigned gmask = 0xFu << (threadIdx.x & 28);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    float x = dk[c], y = dv[c];
    x += __shfl_xor_sync(gmask, x, 1);
    x += __shfl_xor_sync(gmask, x, 2);
    y += __shfl_xor_sync(gmask, y, 1);
    y += __shfl_xor_sync(gmask, y, 2);
    dk[c] = x;
    dv[c] = y;
  }
  rope_rotate<D>(dk, a, j, -1.f);
  if (sl == 0) {
    const int64_t ob = (row_base + j) * a.ld_qkv + h * D;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      store_from_f32(a.dqkv, ob + a.m + c, dk[c], a.prec);
      store_from_f32(a.dqkv, ob + 2 * a.m + c, dv[c], a.prec);
    }
  }
}

}  // namespace mecefo
