// HBM-bound kernels of the MeCeFO step: RMSNorm forward/backward (fused with
// the residual add and a deterministic two-stage scale-gradient reduction),
// embedding gather/scatter, fused softmax-cross-entropy forward+backward,
// Eq. (1) gradient scale/accumulate, and the multi-tensor AdamW step.
#pragma once
#include "common.cuh"

namespace mecefo {

constexpr float kRmsEps = 1e-6f;  // model.py:27

// ---------------------------------------------------------------------------
// RMSNorm forward: out = (x * inv) * g, inv = 1/sqrt(mean(x^2) + eps).
// model.py:183-186. One warp per row, float4 loads when aligned.
// ---------------------------------------------------------------------------
__global__ void rmsnorm_fwd_kernel(const float* __restrict__ x, const float* __restrict__ g, void* __restrict__ out,
                                   float* __restrict__ inv_out, int rows, int m, int out_prec) {
  griddep_wait();
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + (int64_t)row * m;
  float ss = 0.f;
  const bool vec = ((m & 3) == 0);
  if (vec) {
    for (int c = lane * 4; c < m; c += 128) {
      float4 v = *reinterpret_cast<const float4*>(xr + c);
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
  } else {
    for (int c = lane; c < m; c += 32) ss += xr[c] * xr[c];
  }
  ss = warp_sum(ss);
  const float inv = 1.f / sqrtf(ss / (float)m + kRmsEps);
  if (lane == 0 && inv_out) inv_out[row] = inv;
  if (vec && out_prec == PREC_BF16) {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + (int64_t)row * m;
    for (int c = lane * 4; c < m; c += 128) {
      float4 v = *reinterpret_cast<const float4*>(xr + c);
      float4 s = *reinterpret_cast<const float4*>(g + c);
      __nv_bfloat162 a = __floats2bfloat162_rn((v.x * inv) * s.x, (v.y * inv) * s.y);
      __nv_bfloat162 b = __floats2bfloat162_rn((v.z * inv) * s.z, (v.w * inv) * s.w);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&a);
      w.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(o + c) = w;
    }
  } else {
    for (int c = lane; c < m; c += 32) store_from_f32(out, (int64_t)row * m + c, (xr[c] * inv) * g[c], out_prec);
  }
}

// ---------------------------------------------------------------------------
// RMSNorm backward fused with the residual add (model.py:189-195,
// approx.py:130): dx = resid + a*inv - x*inv^3*(sum(a*x)/m), a = d*g.
// Also emits a low-precision copy of dx (the next GEMM operand) and per-block
// partial column sums of d*x*inv (the scale gradient), reduced by
// colsum_finalize_kernel in a fixed order (deterministic).
// Block = 8 warps, each warp one row at a time; block b owns rows
// [b*rows_per_block, ...).
// ---------------------------------------------------------------------------
__global__ void rmsnorm_bwd_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                   const float* __restrict__ inv, const float* __restrict__ d,
                                   const float* __restrict__ resid, float* __restrict__ dx, void* __restrict__ dx_lp,
                                   int lp_prec, float* __restrict__ partial, int rows, int m, int rows_per_block) {
  griddep_wait();
  extern __shared__ float sh[];  // [8][m] per-warp column partials
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* acc = sh + wid * m;
  for (int c = lane; c < m; c += 32) acc[c] = 0.f;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(r0 + rows_per_block, rows);
  for (int row = r0 + wid; row < r1; row += 8) {
    const float* xr = x + (int64_t)row * m;
    const float* dr = d + (int64_t)row * m;
    const float iv = inv[row];
    float s = 0.f;
    for (int c = lane; c < m; c += 32) {
      const float a = dr[c] * g[c];
      s += a * xr[c];
      acc[c] += dr[c] * xr[c] * iv;
    }
    s = warp_sum(s) / (float)m;
    const float k = iv * iv * iv * s;
    for (int c = lane; c < m; c += 32) {
      float v = dr[c] * g[c] * iv - xr[c] * k;
      if (resid) v += resid[(int64_t)row * m + c];
      dx[(int64_t)row * m + c] = v;
      if (dx_lp) store_from_f32(dx_lp, (int64_t)row * m + c, v, lp_prec);
    }
  }
  __syncthreads();
  if (partial) {
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += sh[w * m + c];
      partial[(int64_t)blockIdx.x * m + c] = t;
    }
  }
}

// out[c] = beta*out[c] + alpha * sum_b partial[b, c] (fixed order over b).
// Block (32 x 8): 32 columns, 8 row-strided partial sums each, fixed order.
__global__ void colsum_finalize_kernel(const float* __restrict__ partial, int nblocks, int m, float* __restrict__ out,
                                       float alpha, float beta) {
  griddep_wait();
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float t = 0.f;
  if (c < m)
    for (int b = ty; b < nblocks; b += 8) t += partial[(int64_t)b * m + c];
  red[ty][tx] = t;
  __syncthreads();
  if (ty == 0 && c < m) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][tx];
    out[c] = (beta != 0.f ? beta * out[c] : 0.f) + alpha * s;
  }
}

// ---------------------------------------------------------------------------
// Embedding gather / scatter-add (model.py:463, 486-489).
// ---------------------------------------------------------------------------
// Token ids outside [0, vocab) (the reference raises IndexError on the gather,
// model.py:463) never touch memory out of range: the gather writes a zero row
// and sets status[MECEFO_STATUS_BAD_TOKEN]; the scatter-add skips the row.
__global__ void embedding_fwd_kernel(const int64_t* __restrict__ tok, const float* __restrict__ emb,
                                     float* __restrict__ out, int rows, int m, int vocab, int* __restrict__ status) {
  griddep_wait();
  const int row = blockIdx.x;
  if (row >= rows) return;
  const int64_t t = tok[row];
  float* o = out + (int64_t)row * m;
  if (t < 0 || t >= vocab) {
    if (threadIdx.x == 0 && status) atomicOr(status, 1);
    for (int c = threadIdx.x; c < m; c += blockDim.x) o[c] = 0.f;
    return;
  }
  const float* e = emb + t * (int64_t)m;
  for (int c = threadIdx.x; c < m; c += blockDim.x) o[c] = e[c];
}

__global__ void embedding_bwd_kernel(const int64_t* __restrict__ tok, const float* __restrict__ dx,
                                     float* __restrict__ grad, int rows, int m, float alpha, int vocab) {
  griddep_wait();
  const int row = blockIdx.x;
  if (row >= rows) return;
  const int64_t t = tok[row];
  if (t < 0 || t >= vocab) return;
  float* gp = grad + t * (int64_t)m;
  const float* d = dx + (int64_t)row * m;
  for (int c = threadIdx.x; c < m; c += blockDim.x) atomicAdd(gp + c, alpha * d[c]);
}

// ---------------------------------------------------------------------------
// Fused softmax cross-entropy forward + backward (model.py:492-509).
// loss_row = logsumexp(z) - z[target]; dlogits = (softmax - onehot) / n,
// written in place over the logits (same precision). One block per row.
// ---------------------------------------------------------------------------
__global__ void cross_entropy_kernel(void* __restrict__ logits, int64_t ld, const int64_t* __restrict__ targets,
                                     float* __restrict__ loss_rows, int rows, int V, float inv_n, int prec,
                                     int* __restrict__ bad_target) {
  griddep_wait();
  __shared__ float red[32];
  const int row = blockIdx.x;
  if (row >= rows) return;
  const int64_t base = (int64_t)row * ld;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < V; c += blockDim.x) mx = fmaxf(mx, load_as_f32(logits, base + c, prec));
  mx = block_max(mx, red);
  float s = 0.f;
  for (int c = threadIdx.x; c < V; c += blockDim.x) s += expf(load_as_f32(logits, base + c, prec) - mx);
  s = block_sum(s, red);
  const float lse = mx + logf(s);
  const int64_t t = targets[row];
  if (t < 0 || t >= V) {  // model.py:505 would raise IndexError: flag it, contribute nothing
    if (threadIdx.x == 0) {
      atomicOr(bad_target, 2);
      loss_rows[row] = 0.f;
    }
    for (int c = threadIdx.x; c < V; c += blockDim.x) store_from_f32(logits, base + c, 0.f, prec);
    return;
  }
  const float zt = load_as_f32(logits, base + t, prec);
  __syncthreads();
  if (threadIdx.x == 0) loss_rows[row] = lse - zt;
  const float inv_s = 1.f / s;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float p = expf(load_as_f32(logits, base + c, prec) - mx) * inv_s;
    store_from_f32(logits, base + c, (p - (c == t ? 1.f : 0.f)) * inv_n, prec);
  }
}

// Deterministic mean of per-row losses into out[0] (single block).
// One block per group of n consecutive values: out[g] = mean(v[g*n : (g+1)*n]).
__global__ void mean_kernel(const float* __restrict__ v, int n, float* __restrict__ out) {
  griddep_wait();
  __shared__ float red[32];
  const float* vg = v + (int64_t)blockIdx.x * n;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += vg[i];
  float t = block_sum((float)s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = t / (float)n;
}

// ---------------------------------------------------------------------------
// Eq. (1): out = beta*out + alpha*src over a flat range (fp32).
// ---------------------------------------------------------------------------
__global__ void axpby_kernel(const float* __restrict__ src, float* __restrict__ out, int64_t n, float alpha,
                             float beta) {
  griddep_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (beta != 0.f ? beta * out[i] : 0.f) + alpha * src[i];
}

__global__ void cast_f32_kernel(const float* __restrict__ src, void* __restrict__ dst, int64_t n, int prec) {
  griddep_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    store_from_f32(dst, i, src[i], prec);
}

// bf16 -> fp32 (the all-reduced bf16 gradient bucket back into the flat fp32
// buffer the optimizer reads); 8 elements per thread-iteration.
__global__ void widen_bf16_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst, int64_t n) {
  griddep_wait();
  const int64_t n8 = n >> 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = reinterpret_cast<const uint4*>(src)[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
    float4 a, b;
    float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]), f2 = __bfloat1622float2(h[2]),
           f3 = __bfloat1622float2(h[3]);
    a = make_float4(f0.x, f0.y, f1.x, f1.y);
    b = make_float4(f2.x, f2.y, f3.x, f3.y);
    reinterpret_cast<float4*>(dst)[2 * i] = a;
    reinterpret_cast<float4*>(dst)[2 * i + 1] = b;
  }
  for (int64_t i = (n8 << 3) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

// Q (2f x 2r) fp32 -> compute precision, keeping only the diagonal blocks
// [0,f)x[0,r) and [f,2f)x[r,2r) (the gate-gate and up-up products).
__global__ void cast_blockdiag_kernel(const float* __restrict__ src, void* __restrict__ dst, int rows_half,
                                      int cols_half, int prec) {
  griddep_wait();
  const int64_t n = (int64_t)4 * rows_half * cols_half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (2 * cols_half), c = i % (2 * cols_half);
    const bool keep = (r < rows_half) == (c < cols_half);
    store_from_f32(dst, i, keep ? src[i] : 0.f, prec);
  }
}

// dst (2rp x 2f, compute precision) = the block-diagonal expansion of the
// stacked [Q_g^T ; Q_u^T] (2rp x f, fp32): row block k/rp keeps column block
// k/rp, the off-diagonal blocks are zero (the transposed low-rank chain).
// `groups` consecutive (2rp x f) -> (2rp x 2f) blocks (grouped low-rank chain).
__global__ void cast_blockdiag_t_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int rp, int f,
                                        int64_t groups) {
  griddep_wait();
  const int64_t n = groups * 4 * rp * f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / (2 * f), c = i % (2 * f);  // k: global row (group-major)
    const bool keep = ((k % (2 * rp)) < rp) == (c < f);
    dst[i] = __float2bfloat16_rn(keep ? src[k * f + (c < f ? c : c - f)] : 0.f);
  }
}

__global__ void nonfinite_kernel(const float* __restrict__ v, int64_t n, int* __restrict__ flag) {
  griddep_wait();
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(v[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

// ---------------------------------------------------------------------------
// Multi-tensor AdamW (optim.py:75-93) with per-parameter step counts and a
// skip mask (optim.py:96-103). Segments describe each named parameter in the
// flat buffer; skipped segments are simply not listed by the host.
// ---------------------------------------------------------------------------
struct AdamSeg {
  int64_t offset;
  int64_t numel;
  float step_size;   // lr / (1 - beta1^t)
  float inv_bc2;     // 1 / (1 - beta2^t)
  float lr_wd;       // lr * weight_decay
  int pad;
};

// The active segments are concatenated into one virtual range; every thread
// updates 4 consecutive elements per iteration (float4 when aligned), so the
// large embedding/unembedding segments spread over the whole GPU.
__global__ void __launch_bounds__(256) adamw_kernel(const AdamSeg* __restrict__ segs, int nseg,
                                                    float* __restrict__ w, const float* __restrict__ grad,
                                                    float* __restrict__ m1, float* __restrict__ m2,
                                                    void* __restrict__ shadow, int shadow_prec, float beta1,
                                                    float beta2, float eps, int* __restrict__ status) {
  griddep_wait();
  extern __shared__ int64_t cum[];  // nseg + 1 prefix sums of numel
  if (threadIdx.x == 0) {
    int64_t c = 0;
    for (int s = 0; s < nseg; ++s) {
      cum[s] = c;
      c += segs[s].numel;
    }
    cum[nseg] = c;
  }
  __syncthreads();
  const int64_t total = cum[nseg];
  // optim.py:55-57 _check_grad, fused into the read of g: any non-finite
  // gradient sets status[MECEFO_STATUS_NONFINITE_GRAD] (read by the host at the
  // iteration boundary, which raises NumericalFailure)
  bool bad = false;
  auto upd = [&](const AdamSeg& sg, int64_t i) {
    const float g = grad[i];
    bad |= !isfinite(g);
    float mm = m1[i], vv = m2[i];
    mm = beta1 * mm + (1.f - beta1) * g;
    vv = beta2 * vv + (1.f - beta2) * (g * g);
    m1[i] = mm;
    m2[i] = vv;
    const float wi = w[i];
    const float wn = wi - (sg.step_size * mm / (sqrtf(vv * sg.inv_bc2) + eps) + sg.lr_wd * wi);
    w[i] = wn;
    if (shadow) store_from_f32(shadow, i, wn, shadow_prec);
  };
  for (int64_t v = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); v < total;
       v += 4 * (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;  // last segment with cum[s] <= v
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cum[mid] <= v) lo = mid; else hi = mid - 1;
    }
    const AdamSeg sg = segs[lo];
    const int64_t i = sg.offset + (v - cum[lo]);
    if (v + 4 <= cum[lo + 1] && (i & 3) == 0) {
      const float4 g = *reinterpret_cast<const float4*>(grad + i);
      float4 mm = *reinterpret_cast<const float4*>(m1 + i), vv = *reinterpret_cast<const float4*>(m2 + i);
      float4 wi = *reinterpret_cast<const float4*>(w + i);
      float gg[4] = {g.x, g.y, g.z, g.w}, ma[4] = {mm.x, mm.y, mm.z, mm.w}, va[4] = {vv.x, vv.y, vv.z, vv.w};
      bad |= !(isfinite(g.x) && isfinite(g.y) && isfinite(g.z) && isfinite(g.w));
      float wa[4] = {wi.x, wi.y, wi.z, wi.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ma[q] = beta1 * ma[q] + (1.f - beta1) * gg[q];
        va[q] = beta2 * va[q] + (1.f - beta2) * (gg[q] * gg[q]);
        wa[q] = wa[q] - (sg.step_size * ma[q] / (sqrtf(va[q] * sg.inv_bc2) + eps) + sg.lr_wd * wa[q]);
      }
      *reinterpret_cast<float4*>(m1 + i) = make_float4(ma[0], ma[1], ma[2], ma[3]);
      *reinterpret_cast<float4*>(m2 + i) = make_float4(va[0], va[1], va[2], va[3]);
      *reinterpret_cast<float4*>(w + i) = make_float4(wa[0], wa[1], wa[2], wa[3]);
      if (shadow) {
        if (shadow_prec == PREC_BF16) {
          __nv_bfloat162 a = __floats2bfloat162_rn(wa[0], wa[1]), b = __floats2bfloat162_rn(wa[2], wa[3]);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&a);
          u.y = *reinterpret_cast<uint32_t*>(&b);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(shadow) + i) = u;
        } else {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(shadow) + i) = make_float4(wa[0], wa[1], wa[2], wa[3]);
        }
      }
    } else {
      for (int q = 0; q < 4 && v + q < total; ++q) {
        int s = lo;
        while (v + q >= cum[s + 1]) ++s;
        upd(segs[s], segs[s].offset + (v + q - cum[s]));
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && status) atomicOr(status, 4);
}

}  // namespace mecefo

namespace mecefo {

// ---------------------------------------------------------------------------
// Bandwidth-oriented versions (the row lives in registers; 16-byte accesses,
// one warp per row, lane-contiguous float4 columns).
// ---------------------------------------------------------------------------

__device__ __forceinline__ void store4(void* base, int64_t idx, float4 v, int prec) {
  if (prec == PREC_BF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&a);
    w.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + idx) = w;
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + idx) = v;
  }
}

// model.py:183-186. Requires m % 4 == 0 and m <= 128 * NV.
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_fwd_vec_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                                              void* __restrict__ out, float* __restrict__ inv_out,
                                                              int rows, int m, int out_prec) {
  griddep_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + (int64_t)row * m;
  float4 v[NV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 4;
    v[i] = c < m ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = warp_sum(ss);
  const float inv = 1.f / sqrtf(ss / (float)m + kRmsEps);
  if (lane == 0 && inv_out) inv_out[row] = inv;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 4;
    if (c < m) {
      const float4 s = __ldg(reinterpret_cast<const float4*>(g + c));
      store4(out, (int64_t)row * m + c,
             make_float4((v[i].x * inv) * s.x, (v[i].y * inv) * s.y, (v[i].z * inv) * s.z, (v[i].w * inv) * s.w),
             out_prec);
    }
  }
}

// model.py:189-195 + approx.py:130, fused: dx = resid + a*inv - x*inv^3*(sum(a*x)/m),
// a = d*g; dx_lp = compute-precision copy; per-block partial column sums of
// d*x*inv (scale gradient), reduced in a fixed order afterwards.
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_bwd_vec_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                                              const float* __restrict__ inv,
                                                              const float* __restrict__ d,
                                                              const float* __restrict__ resid, float* __restrict__ dx,
                                                              void* __restrict__ dx_lp, int lp_prec,
                                                              float* __restrict__ partial, int rows, int m,
                                                              int rows_per_block) {
  griddep_wait();
  extern __shared__ float4 red_dyn[];  // [8][NV * 32]
  float4 (*red)[NV * 32] = reinterpret_cast<float4 (*)[NV * 32]>(red_dyn);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 gs[NV], acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 4;
    gs[i] = c < m ? __ldg(reinterpret_cast<const float4*>(g + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(r0 + rows_per_block, rows);
  if constexpr (NV <= 4) {  // (wider rows would spill with two rows in registers)
    // software pipeline over this warp's rows: the next row's x, d, residual
    // and inv are in flight while the current row is reduced and written (one
    // exposed memory latency per warp instead of two per row)
    float4 xv[NV], dv[NV], rv[NV];
    float iv = 0.f;
    auto fetch = [&](int row, float4* xa, float4* da, float4* ra, float& ivr) {
      const float* xr = x + (int64_t)row * m;
      const float* dr = d + (int64_t)row * m;
      ivr = inv[row];
  #pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = (i * 32 + lane) * 4;
        const bool ok = c < m;
        xa[i] = ok ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        da[i] = ok ? *reinterpret_cast<const float4*>(dr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        ra[i] = (ok && resid) ? *reinterpret_cast<const float4*>(resid + (int64_t)row * m + c)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    if (r0 + wid < r1) fetch(r0 + wid, xv, dv, rv, iv);
    for (int row = r0 + wid; row < r1; row += 8) {
      float4 xn[NV], dn[NV], rn[NV];
      float ivn = 0.f;
      if (row + 8 < r1) fetch(row + 8, xn, dn, rn, ivn);
      float s = 0.f;
  #pragma unroll
      for (int i = 0; i < NV; ++i) {
        s += dv[i].x * gs[i].x * xv[i].x + dv[i].y * gs[i].y * xv[i].y + dv[i].z * gs[i].z * xv[i].z +
             dv[i].w * gs[i].w * xv[i].w;
        acc[i].x += dv[i].x * xv[i].x * iv;
        acc[i].y += dv[i].y * xv[i].y * iv;
        acc[i].z += dv[i].z * xv[i].z * iv;
        acc[i].w += dv[i].w * xv[i].w * iv;
      }
      s = warp_sum(s) / (float)m;
      const float k = iv * iv * iv * s;
  #pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = (i * 32 + lane) * 4;
        if (c < m) {
          float4 o = make_float4(dv[i].x * gs[i].x * iv - xv[i].x * k, dv[i].y * gs[i].y * iv - xv[i].y * k,
                                 dv[i].z * gs[i].z * iv - xv[i].z * k, dv[i].w * gs[i].w * iv - xv[i].w * k);
          o.x += rv[i].x; o.y += rv[i].y; o.z += rv[i].z; o.w += rv[i].w;  // zeros without a residual
          *reinterpret_cast<float4*>(dx + (int64_t)row * m + c) = o;
          if (dx_lp) store4(dx_lp, (int64_t)row * m + c, o, lp_prec);
        }
      }
  #pragma unroll
      for (int i = 0; i < NV; ++i) {
        xv[i] = xn[i];
        dv[i] = dn[i];
        rv[i] = rn[i];
      }
      iv = ivn;
    }
  } else {
    for (int row = r0 + wid; row < r1; row += 8) {
      const float* xr = x + (int64_t)row * m;
      const float* dr = d + (int64_t)row * m;
      const float iv = inv[row];
      float4 xv[NV], dv[NV];
      float s = 0.f;
  #pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = (i * 32 + lane) * 4;
        if (c < m) {
          xv[i] = *reinterpret_cast<const float4*>(xr + c);
          dv[i] = *reinterpret_cast<const float4*>(dr + c);
        } else {
          xv[i] = dv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        s += dv[i].x * gs[i].x * xv[i].x + dv[i].y * gs[i].y * xv[i].y + dv[i].z * gs[i].z * xv[i].z +
             dv[i].w * gs[i].w * xv[i].w;
        acc[i].x += dv[i].x * xv[i].x * iv;
        acc[i].y += dv[i].y * xv[i].y * iv;
        acc[i].z += dv[i].z * xv[i].z * iv;
        acc[i].w += dv[i].w * xv[i].w * iv;
      }
      s = warp_sum(s) / (float)m;
      const float k = iv * iv * iv * s;
  #pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = (i * 32 + lane) * 4;
        if (c < m) {
          float4 o = make_float4(dv[i].x * gs[i].x * iv - xv[i].x * k, dv[i].y * gs[i].y * iv - xv[i].y * k,
                                 dv[i].z * gs[i].z * iv - xv[i].z * k, dv[i].w * gs[i].w * iv - xv[i].w * k);
          if (resid) {
            const float4 rr = *reinterpret_cast<const float4*>(resid + (int64_t)row * m + c);
            o.x += rr.x; o.y += rr.y; o.z += rr.z; o.w += rr.w;
          }
          *reinterpret_cast<float4*>(dx + (int64_t)row * m + c) = o;
          if (dx_lp) store4(dx_lp, (int64_t)row * m + c, o, lp_prec);
        }
      }
    }
  }
  if (!partial) return;
#pragma unroll
  for (int i = 0; i < NV; ++i) red[wid][i * 32 + lane] = acc[i];
  __syncthreads();
  for (int q = threadIdx.x; q < NV * 32; q += blockDim.x) {
    const int c = q * 4;
    if (c >= m) continue;
    float4 t = red[0][q];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      t.x += red[w][q].x; t.y += red[w][q].y; t.z += red[w][q].z; t.w += red[w][q].w;
    }
    *reinterpret_cast<float4*>(partial + (int64_t)blockIdx.x * m + c) = t;
  }
}

// Single-read fused softmax-CE for bf16 logits (model.py:492-509): the row is
// held in registers (8 bf16 per 16-byte vector, NV vectors per thread), so the
// logits are read once and dlogits written once.
template <int NV>
__global__ void __launch_bounds__(256) cross_entropy_bf16_kernel(__nv_bfloat16* __restrict__ logits, int64_t ld,
                                                                  const int64_t* __restrict__ targets,
                                                                  float* __restrict__ loss_rows, int rows, int V,
                                                                  float inv_n, int* __restrict__ bad_target) {
  griddep_wait();
  __shared__ float red[32];
  __shared__ float zt_s;
  const int row = blockIdx.x;
  __nv_bfloat16* lr = logits + (int64_t)row * ld;
  const int64_t t = targets[row];
  if (t < 0 || t >= V) {
    if (threadIdx.x == 0) {
      atomicOr(bad_target, 2);
      loss_rows[row] = 0.f;
    }
    for (int c = threadIdx.x * 8; c < V; c += blockDim.x * 8)
      *reinterpret_cast<uint4*>(lr + c) = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  if (threadIdx.x == 0) zt_s = __bfloat162float(lr[t]);
  uint4 w[NV];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 8;
    if (c < V) {
      w[i] = *reinterpret_cast<const uint4*>(lr + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        mx = fmaxf(mx, fmaxf(f.x, f.y));
      }
    }
  }
  mx = block_max(mx, red);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 8;
    if (c < V) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        s += __expf(f.x - mx) + __expf(f.y - mx);
      }
    }
  }
  s = block_sum(s, red);
  const float lse = mx + logf(s);
  if (threadIdx.x == 0) loss_rows[row] = lse - zt_s;
  const float sc = inv_n / s;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 8;
    if (c < V) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        float p0 = __expf(f.x - mx) * sc, p1 = __expf(f.y - mx) * sc;
        if (c + 2 * j == t) p0 -= inv_n;
        if (c + 2 * j + 1 == t) p1 -= inv_n;
        __nv_bfloat162 q = __floats2bfloat162_rn(p0, p1);
        o[j] = *reinterpret_cast<uint32_t*>(&q);
      }
      *reinterpret_cast<uint4*>(lr + c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// One warp per row (model.py:492-509, bf16 logits): pass 1 keeps an online
// (max, sum-exp) per lane over 16-byte vectors (4 loads in flight per lane),
// a shuffle reduction merges the lanes; pass 2 re-reads the row and writes
// dlogits = (softmax - onehot)/n in place. No block barriers, full occupancy
// (measured faster than a register-resident CTA-per-row variant, which
// reads once but serialises load -> reduce -> store within each CTA).
__global__ void __launch_bounds__(256) cross_entropy_warp_kernel(__nv_bfloat16* __restrict__ logits, int64_t ld,
                                                                  const int64_t* __restrict__ targets,
                                                                  float* __restrict__ loss_rows, int rows, int V,
                                                                  float inv_n, int* __restrict__ bad_target) {
  griddep_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  __nv_bfloat16* lr = logits + (int64_t)row * ld;
  const int64_t t = targets[row];
  if (t < 0 || t >= V) {
    if (lane == 0) {
      atomicOr(bad_target, 2);
      loss_rows[row] = 0.f;
    }
    for (int vi = lane; vi < (V >> 3); vi += 32) reinterpret_cast<uint4*>(lr)[vi] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  const float zt = __bfloat162float(lr[t]);
  const int nvec = V >> 3;
  const uint4* lv = reinterpret_cast<const uint4*>(lr);
  float mx = -INFINITY, s = 0.f;
  // 4 independent 16-byte loads per lane in flight per iteration
  for (int v0 = lane; v0 < nvec; v0 += 128) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = v0 + 32 * u < nvec ? lv[v0 + 32 * u] : make_uint4(0xff80ff80u, 0xff80ff80u,
                                                                                        0xff80ff80u, 0xff80ff80u);
    float lm = -INFINITY;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 q = __bfloat1622float2(h[j]);
        lm = fmaxf(lm, fmaxf(q.x, q.y));
      }
    }
    const float nm = fmaxf(mx, lm);
    s = (mx == -INFINITY) ? 0.f : s * __expf(mx - nm);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 q = __bfloat1622float2(h[j]);  // -inf padding contributes exp(-inf) = 0
        s += __expf(q.x - nm) + __expf(q.y - nm);
      }
    }
    mx = nm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const float os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(mx, om);
    s = (mx == -INFINITY ? 0.f : s * __expf(mx - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    mx = nm;
  }
  if (lane == 0) loss_rows[row] = mx + logf(s) - zt;
  const float sc = inv_n / s;
  uint4* lw = reinterpret_cast<uint4*>(lr);
  for (int v0 = lane; v0 < nvec; v0 += 128) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + 32 * u < nvec) w[u] = lv[v0 + 32 * u];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int vi = v0 + 32 * u;
      if (vi >= nvec) continue;
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
      uint32_t o4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 q = __bfloat1622float2(h[j]);
        float p0 = __expf(q.x - mx) * sc, p1 = __expf(q.y - mx) * sc;
        const int c = vi * 8 + 2 * j;
        if (c == t) p0 -= inv_n;
        if (c + 1 == t) p1 -= inv_n;
        __nv_bfloat162 r = __floats2bfloat162_rn(p0, p1);
        o4[j] = *reinterpret_cast<uint32_t*>(&r);
      }
      lw[vi] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
    }
  }
}

}  // namespace mecefo
