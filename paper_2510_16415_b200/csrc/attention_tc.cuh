// Tensor-core causal attention forward for head_dim 64 and T <= 256 (bf16).
//
// One CTA per (sequence, head, 128-query block). Because a whole causal key
// range (<= 256 keys) fits one tcgen05 accumulator (M=128, N<=256 fp32 columns
// of TMEM), the softmax is exact and single-pass — no online rescaling:
//   1. TMA: Q block (128x64), K and V rows [0, nk) (nk <= 256) -> smem (SW128)
//   2. tcgen05.mma  S = Q K^T            -> TMEM cols [0, nk)
//   3. 8 warps, two per TMEM lane quadrant (one query row per thread, each
//      warp of a pair owns half of the key columns; partial max / sum meet in
//      smem): row max, p = exp(scale (s - max)), causal mask, row sum; P
//      (bf16) -> smem in the UMMA K-major SW128 layout
//   4. tcgen05.mma  O = P V (V as an MN-major B operand) -> TMEM cols [0,64)
//   5. O / rowsum -> ctx (bf16), LSE (full cache only)
// q/k arrive RoPE-rotated from the QKV GEMM epilogue (model.py:281-288,
// 323-331). The (B,H,T,T) probabilities never touch HBM.
#pragma once
#include "gemm.cuh"

namespace mecefo {

struct AttnTcArgs {
  void* ctx;
  int64_t ld_ctx;
  float* lse;
  int T, H, m;
  float scale;
};

constexpr int ATC_THREADS = 256;
// smem: [Q 16 KB][K 32 KB][pad 16 KB][V 32 KB] + barriers/reductions. P (up to
// 64 KB) overwrites Q|K|pad once S = Q K^T has completed, so two CTAs fit
// per SM (TMEM: 256 columns each; O reuses S's first 64 columns).
constexpr int ATC_SMEM = 16384 + 32768 + 16384 + 32768 + 1024 + 256 + 2048;

__global__ void __launch_bounds__(ATC_THREADS, 2)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, AttnTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + 16384;
  uint8_t* sV = sK + 32768 + 16384;
  uint8_t* sP = smem;  // aliases Q|K|pad after the S MMA
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 32768);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seq = blockIdx.x / a.H, h = blockIdx.x % a.H;
  const int q0 = blockIdx.y * 128;
  const int nk = min(a.T, q0 + 128);   // keys 0..nk-1 (multiple of 64)
  const int nq = min(128, a.T - q0);   // valid query rows in this block
  const int row0 = seq * a.T;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(256u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  griddep_wait();  // predecessor outputs are visible from here on
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (threadIdx.x == 0) {
    // Q|K on bars[0] (S = Q K^T starts as soon as they land), V on bars[3] (needed by P V only)
    mbar_expect_tx(&bars[0], 16384 + nk * 128);
    mbar_expect_tx(&bars[3], nk * 128);
    tma_load_2d(sQ, &tq, &bars[0], h * 64, row0 + q0);
    tma_load_2d(sQ + 8192, &tq, &bars[0], h * 64, row0 + q0 + 64);
    for (int kb = 0; kb < nk / 64; ++kb) tma_load_2d(sK + kb * 8192, &tq, &bars[0], a.m + h * 64, row0 + kb * 64);
    for (int kb = 0; kb < nk / 64; ++kb) tma_load_2d(sV + kb * 8192, &tq, &bars[3], 2 * a.m + h * 64, row0 + kb * 64);
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    // S = Q K^T: A, B K-major; M = 128, N = nk, K = 64
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nk >> 3) << 17) | ((128u >> 4) << 24);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      tc_mma_bf16(tmem, make_sdesc(smem_u32(sQ) + k * 32, 16, 1024), make_sdesc(smem_u32(sK) + k * 32, 16, 1024),
                  idesc, k > 0 ? 1u : 0u);
    tc_commit(&bars[1]);
  }
  mbar_wait(&bars[1], 0);
  tc_fence_after();

  const int quad = warp & 3, hf = warp >> 2;  // TMEM lane quadrant, key-column half
  const int row = quad * 32 + lane;
  const int qi = q0 + row;  // query position in the sequence
  const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16);
  const float c2 = a.scale * 1.4426950408889634f;
  const int hw = nk >> 1;          // key columns per half (64 or 128)
  const int cb = hf * hw;          // first key column of this half
  float* red = reinterpret_cast<float*>(tmem_holder + 4);  // [2][128] max, then [2][128] sum
  float mx = -INFINITY;
  for (int cc = 0; cc < hw; cc += 32) {
    float v[32];
    tmem_ld16_nowait(taddr + cb + cc, v);
    tmem_ld16_nowait(taddr + cb + cc + 16, v + 16);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (cb + cc + j <= qi) mx = fmaxf(mx, v[j]);
  }
  red[hf * 128 + row] = mx;
  __syncthreads();
  mx = fmaxf(red[row], red[128 + row]);
  const bool valid = row < nq;
  float l = 0.f;
  for (int cc = 0; cc < hw; cc += 32) {
    float v[32];
    tmem_ld16_nowait(taddr + cb + cc, v);
    tmem_ld16_nowait(taddr + cb + cc + 16, v + 16);
    tmem_wait_ld();
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k0 = cb + cc + 2 * j;
      const float p0 = (valid && k0 <= qi) ? ex2_approx((v[2 * j] - mx) * c2) : 0.f;
      const float p1 = (valid && k0 + 1 <= qi) ? ex2_approx((v[2 * j + 1] - mx) * c2) : 0.f;
      __nv_bfloat162 hp = __floats2bfloat162_rn(p0, p1);
      // the row sum uses the bf16-rounded probabilities that feed P V
      const float2 back = __bfloat1622float2(hp);
      l += back.x + back.y;
      pk[j] = *reinterpret_cast<uint32_t*>(&hp);
    }
    // P row `row`, keys [cb+cc, cb+cc+32): 64-key block, 16-byte units u0..u0+3 of the 128-B row
    const int kk = cb + cc;
    uint8_t* blk = sP + (kk >> 6) * 16384 + row * 128;
    const int u0 = (kk & 63) >> 3;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(blk + (((u0 + q) ^ (row & 7)) << 4)) =
          make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
  red[256 + hf * 128 + row] = l;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  l = red[256 + row] + red[384 + row];
  if (threadIdx.x == 0) {
    mbar_wait(&bars[3], 0);
    tc_fence_after();
    // O = P V: A = P K-major (K = keys), B = V MN-major (N = d = 64)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    for (int s = 0; s < nk / 16; ++s)
      tc_mma_bf16(tmem, make_sdesc(smem_u32(sP) + (s >> 2) * 16384 + (s & 3) * 32, 16, 1024),
                  make_sdesc(smem_u32(sV) + s * 2048, 8192, 1024), idesc, s > 0 ? 1u : 0u);
    tc_commit(&bars[2]);
  }
  mbar_wait(&bars[2], 0);
  tc_fence_after();
  const float il = 1.f / l;
  // this half's 32 output columns [hf*32, hf*32+32)
  float ov[32];
  tmem_ld16_nowait(taddr + hf * 32, ov);
  tmem_ld16_nowait(taddr + hf * 32 + 16, ov + 16);
  tmem_wait_ld();
  uint32_t ow[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    __nv_bfloat162 hp = __floats2bfloat162_rn(ov[2 * j] * il, ov[2 * j + 1] * il);
    ow[j] = *reinterpret_cast<uint32_t*>(&hp);
  }
  if (valid) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.ctx) + (int64_t)(row0 + qi) * a.ld_ctx +
                                          h * 64 + hf * 32);
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[u] = make_uint4(ow[4 * u], ow[4 * u + 1], ow[4 * u + 2], ow[4 * u + 3]);
    if (a.lse && hf == 0) a.lse[(int64_t)(row0 + qi) * a.H + h] = mx * a.scale + logf(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
  }
}

}  // namespace mecefo
