// Tensor-core causal attention backward for head_dim 64, T in {128, 256}
// (bf16), the exact backward of healthy ranks (model.py:336-368).
//
// A persistent CTA per SM (16 warps) walks the (sequence, head) items; each
// item's Q, K, V, dO are TMA-staged once (the next item's while this one
// computes, see below) and the causal 128x128 blocks n = (key block kb, query
// block qb >= kb) run as a software pipeline on ONE issuing thread:
//   S^T  = K_kb Q_qb^T,  dP^T = V_kb dO_qb^T            (tcgen05 -> TMEM)
//   P^T  = exp(scale S^T - LSE),  dS^T = P^T (dP^T - D)   (all 16 warps)
//   dV_kb += P^T dO_qb,  dK_kb += dS^T Q_qb,  dQ_qb += dS K_kb   (tcgen05)
// The gradient products of block n and the S^T / dP^T products of block n+1
// are issued back to back and committed once, so the tensor pipe never waits
// for a separate round trip per phase; block n+1's elementwise pass starts
// when that commit lands (which also guarantees block n's products are done
// reading the P^T / dS^T tiles it overwrites). Each warp owns one TMEM lane
// quadrant (32 key rows) and a quarter of the 128 query columns; the dK / dV
// / dQ epilogues split the 64 head columns the same way. The P^T / dS^T smem
// tiles are written once in the UMMA K-major SW128 layout and read back both
// as K-major A (dV, dK) and as MN-major A (dQ: the same bytes describe
// dS = (dS^T)^T). TMEM holds S^T, dP^T, dV, dK and dQ for both query blocks:
// exactly 512 columns. Scale and the transpose RoPE rotation (model.py:
// 291-298) are applied in the epilogues.
//
// Measured per C1 layer launch (16384 tokens, 512 items): round-1 kernel (one
// CTA per item, 4 warps, MMA -> wait -> softmax -> MMA -> wait per block)
// 104 us; 16 warps + the issue pipeline 55 us; persistent with prefetch: see
// DESIGN.md.
#pragma once
#include "gemm.cuh"

namespace mecefo {

struct AttnBwdTcArgs {
  const void* ctx;   // O  (b, m)
  const void* dctx;  // dO (b, m)
  const float* lse;  // (b, H)
  void* dqkv;        // (b, 3m) out
  const float* theta;  // rotary frequencies theta_j, j < 32 (model.py:274)
  int T, H, m, rope;
  float scale;
};

constexpr int ABT_WARPS = 16;
constexpr int ABT_THREADS = 32 * ABT_WARPS;
constexpr int ABT_SMEM = 4 * 32768 + 2 * 32768 + 2 * 256 * 4 + 1024 + 256;

// 16 fp32 head columns [c0, c0 + 16) of one row -> scaled, optionally rotated
// back by the transpose RoPE (pairs (2p, 2p+1), model.py:294-297), bf16, two
// 16-byte stores. th: the 8 frequencies theta_{c0/2 .. c0/2+7} (registers);
// the angles are computed, not looked up (the cos/sin table's L2 latency
// serialised these epilogues), with the QKV epilogue's Cody-Waite reduction
// (|angle error| <= ~6e-5 rad, far below the bf16 rounding of dQ / dK).
__device__ __forceinline__ void abt_store_row16(void* base, int64_t idx, const float* v, const float* th, bool rope,
                                                int pos, float mul) {
  float w[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) w[c] = v[c] * mul;
  if (rope) {
    const float fpos = (float)pos;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float ang = fpos * th[p];
      const float kq = rintf(ang * 0.15915494309189535f);
      float rr = fmaf(-kq, 6.28318548202514648f, ang);
      rr = fmaf(kq, 1.7484556e-7f, rr);
      float sn, cs;
      __sincosf(rr, &sn, &cs);
      const float e = w[2 * p], o = w[2 * p + 1];
      w[2 * p] = e * cs + o * sn;
      w[2 * p + 1] = -e * sn + o * cs;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + idx);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    uint32_t q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(w[8 * u + 2 * j], w[8 * u + 2 * j + 1]);
      q[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    dst[u] = make_uint4(q[0], q[1], q[2], q[3]);
  }
}

__device__ __forceinline__ uint32_t abt_pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Persistent: one CTA per SM walks (sequence, head) items. Q, K, V, dO are
// staged in two halves (rows [0,128) and [128,256)); the next item's first
// half is fetched as soon as the current item's last use of it has retired
// (the commit that precedes block (1,1)), its second half once the final
// gradient products retired, and its LSE / D rows are computed while those
// products run — so the loads and the D pass overlap the current item's
// tensor and elementwise work instead of opening every CTA.
__global__ void __launch_bounds__(ABT_THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tdo,
                       AttnBwdTcArgs a, int items) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;               // T rows x 128 B (K-major SW128, 16 KB per 128-row block)
  uint8_t* sK = sQ + 32768;
  uint8_t* sV = sK + 32768;
  uint8_t* sDO = sV + 32768;
  uint8_t* sPt = sDO + 32768;       // P^T  tile: 128 keys x 128 queries (2 x 16 KB chunks)
  uint8_t* sDSt = sPt + 32768;      // dS^T tile
  float* Ls = reinterpret_cast<float*>(sDSt + 32768);
  float* Dv = Ls + 256;
  // 0 S (+ every earlier gradient product), 1 final gradients of an item,
  // 2 / 3 load of rows [0,128) / [128,256)
  uint64_t* bars = reinterpret_cast<uint64_t*>(Dv + 256);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, cg = warp >> 2;  // TMEM lane quadrant, column quarter
  const int nb = a.T / 128;
  const int nblk = nb * (nb + 1) / 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  griddep_wait();  // predecessor outputs are visible from here on
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // TMA of rows [128 hb, 128 hb + 128) of an item's Q, K, V, dO (one barrier per half)
  auto load_half = [&](int item, int hb) {
    const int seq = item / a.H, h = item % a.H, row0 = seq * a.T + hb * 128;
    uint64_t* bar = &bars[2 + hb];
    mbar_expect_tx(bar, 4 * 128 * 128);
    for (int r = 0; r < 2; ++r) {
      const int o = hb * 16384 + r * 8192;
      tma_load_2d(sK + o, &tqkv, bar, a.m + h * 64, row0 + r * 64);
      tma_load_2d(sQ + o, &tqkv, bar, h * 64, row0 + r * 64);
      tma_load_2d(sV + o, &tqkv, bar, 2 * a.m + h * 64, row0 + r * 64);
      tma_load_2d(sDO + o, &tdo, bar, h * 64, row0 + r * 64);
    }
  };
  // LSE (log2 domain) and D_i = rowsum(dO * O) (model.py:352) of an item: two threads per query row
  auto lse_d = [&](int item) {
    const int seq = item / a.H, h = item % a.H, row0 = seq * a.T;
    for (int t = threadIdx.x; t < 2 * a.T; t += ABT_THREADS) {
      const int i = t >> 1, hf = t & 1;
      const int64_t g = (int64_t)(row0 + i);
      const uint4* o =
          reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.ctx) + g * a.m + h * 64 + hf * 32);
      const uint4* d =
          reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.dctx) + g * a.m + h * 64 + hf * 32);
      float acc = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 ov = o[u], dv = d[u];
        const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&ov);
        const __nv_bfloat162* dh = reinterpret_cast<const __nv_bfloat162*>(&dv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 x = __bfloat1622float2(oh[j]), y = __bfloat1622float2(dh[j]);
          acc = fmaf(x.x, y.x, acc);
          acc = fmaf(x.y, y.y, acc);
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (hf == 0) {
        Dv[i] = acc;
        Ls[i] = a.lse[g * a.H + h] * 1.4426950408889634f;
      }
    }
  };

  // K-major A/B, N = 128 (S^T, dP^T); K-major A + MN-major B, N = 64 (dV, dK);
  // MN-major A + MN-major B, N = 64 (dQ).
  constexpr uint32_t id_s = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t id_kv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t id_q =
      (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

  // block n -> (kb, qb), key-block major: (0,0), (0,1), ..., (1,1), ...
  auto block_of = [nb](int n, int& kb, int& qb) {
    kb = 0;
    while (n >= nb - kb) {
      n -= nb - kb;
      ++kb;
    }
    qb = kb + n;
  };
  auto issue_s = [&](int kb, int qb) {  // S^T -> cols [0,128), dP^T -> [128,256)
    const uint32_t k_a = smem_u32(sK + kb * 16384), v_a = smem_u32(sV + kb * 16384);
    const uint32_t q_b = smem_u32(sQ + qb * 16384), do_b = smem_u32(sDO + qb * 16384);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      tc_mma_bf16(tmem, make_sdesc(k_a + k * 32, 16, 1024), make_sdesc(q_b + k * 32, 16, 1024), id_s, k > 0);
      tc_mma_bf16(tmem + 128, make_sdesc(v_a + k * 32, 16, 1024), make_sdesc(do_b + k * 32, 16, 1024), id_s, k > 0);
    }
  };
  auto issue_grads = [&](int kb, int qb) {
    const uint32_t pt = smem_u32(sPt), dst = smem_u32(sDSt);
    const uint32_t q_b = smem_u32(sQ + qb * 16384), do_b = smem_u32(sDO + qb * 16384);
    const uint32_t k_b = smem_u32(sK + kb * 16384);
#pragma unroll 1
    for (int s8 = 0; s8 < 8; ++s8) {  // K = 128 (queries for dV/dK, keys for dQ), 16 per MMA
      const uint32_t a_k = (s8 >> 2) * 16384 + (s8 & 3) * 32;
      const uint32_t first_kv = (qb == kb && s8 == 0) ? 0u : 1u;
      tc_mma_bf16(tmem + 256, make_sdesc(pt + a_k, 16, 1024), make_sdesc(do_b + s8 * 2048, 8192, 1024), id_kv,
                  first_kv);
      tc_mma_bf16(tmem + 320, make_sdesc(dst + a_k, 16, 1024), make_sdesc(q_b + s8 * 2048, 8192, 1024), id_kv,
                  first_kv);
      tc_mma_bf16(tmem + 384 + qb * 64, make_sdesc(dst + s8 * 2048, 16384, 1024),
                  make_sdesc(k_b + s8 * 2048, 8192, 1024), id_q, (kb > 0 || s8 > 0) ? 1u : 0u);
    }
  };

  const float c2 = a.scale * 1.4426950408889634f;
  float th[8];  // this warp's 8 rotary frequencies (head columns [16 cg, 16 cg + 16))
  if (a.rope) {
#pragma unroll
    for (int p = 0; p < 8; ++p) th[p] = __ldg(a.theta + cg * 8 + p);
  }
  const int jl = quad * 32 + lane;  // key row (TMEM lane) owned by this thread
  const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
  auto epi_kv = [&](int row0, int h, int kb) {  // dK_kb (scale, RoPE^T), dV_kb: key rows kb*128 + jl
    float v[16];
    const int pos = kb * 128 + jl;
    const int64_t g = (int64_t)(row0 + pos) * (3 * a.m);
    tmem_ld16(trow + 320 + cg * 16, v);
    abt_store_row16(a.dqkv, g + a.m + h * 64 + cg * 16, v, th, a.rope != 0, pos, a.scale);
    tmem_ld16(trow + 256 + cg * 16, v);
    abt_store_row16(a.dqkv, g + 2 * a.m + h * 64 + cg * 16, v, th, false, 0, 1.f);
  };

  // prologue: the first item's loads, LSE / D, and its first S^T / dP^T
  if (blockIdx.x < items && threadIdx.x == 0) {
    load_half(blockIdx.x, 0);
    if (nb > 1) load_half(blockIdx.x, 1);
  }
  if (blockIdx.x < items) lse_d(blockIdx.x);
  __syncthreads();
  if (blockIdx.x < items && threadIdx.x == 0) {
    mbar_wait(&bars[2], 0);
    tc_fence_after();
    issue_s(0, 0);
    tc_commit(&bars[0]);
  }

  uint32_t nS = 0;  // waits on bars[0] so far
  int iter = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, ++iter) {
    const int seq = item / a.H, h = item % a.H, row0 = seq * a.T;
    const int next = item + gridDim.x;
    const bool has_next = next < items;
    const uint32_t ph = (uint32_t)(iter & 1);
    int kb_prev = 0;
    for (int n = 0; n < nblk; ++n) {
      int kb, qb;
      block_of(n, kb, qb);
      mbar_wait(&bars[0], nS & 1);  // S^T / dP^T of block n (and every earlier gradient product) landed
      ++nS;
      tc_fence_after();
      if (kb != kb_prev) {  // the previous key block's dK / dV are complete: drain before they are overwritten
        epi_kv(row0, h, kb_prev);
        kb_prev = kb;
      }
      if (nb > 1 && n == nblk - 1 && has_next && threadIdx.x == 0)
        load_half(next, 0);  // rows [0,128) are no longer read by this item
      // elementwise: P^T, dS^T for key j = kb*128 + jl, queries i = qb*128 + 32 cg + c
      const int j = kb * 128 + jl;
      const int ib = qb * 128 + cg * 32;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // two 16-column halves (register pressure: 512 threads x 128 regs)
        const int ih = ib + 16 * hh;
        float s[16], dp[16];
        tmem_ld16_nowait(trow + cg * 32 + 16 * hh, s);
        tmem_ld16_nowait(trow + 128 + cg * 32 + 16 * hh, dp);
        tmem_wait_ld();
        uint32_t pk[8], dk[8];
        if (ih + 15 < j) {  // whole half above the diagonal: P = dS = 0
#pragma unroll
          for (int t = 0; t < 8; ++t) pk[t] = dk[t] = 0u;
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            float pv[2], dv[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = 2 * t + e, i = ih + c;
              const float p = (i >= j) ? ex2_approx(fmaf(s[c], c2, -Ls[i])) : 0.f;
              pv[e] = p;
              dv[e] = p * (dp[c] - Dv[i]);
            }
            pk[t] = abt_pack(pv[0], pv[1]);
            dk[t] = abt_pack(dv[0], dv[1]);
          }
        }
        const int off = (cg >> 1) * 16384 + jl * 128;
        const int u0 = (cg & 1) * 4 + 2 * hh;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int sw = ((u0 + q) ^ (jl & 7)) << 4;
          *reinterpret_cast<uint4*>(sPt + off + sw) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          *reinterpret_cast<uint4*>(sDSt + off + sw) =
              make_uint4(dk[4 * q], dk[4 * q + 1], dk[4 * q + 2], dk[4 * q + 3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncthreads();
      if (threadIdx.x == 0) {
        tc_fence_after();
        issue_grads(kb, qb);
        if (n + 1 < nblk) {
          int kb2, qb2;
          block_of(n + 1, kb2, qb2);
          if (n == 0) mbar_wait(&bars[3], ph);  // rows [128,256) of this item landed
          issue_s(kb2, qb2);
          tc_commit(&bars[0]);
        } else {
          tc_commit(&bars[1]);
        }
      }
    }
    if (has_next) lse_d(next);  // overlaps the final gradient products; this item no longer reads Ls / Dv
    mbar_wait(&bars[1], ph);
    tc_fence_after();
    if (has_next && threadIdx.x == 0) {  // next item: remaining rows, then its first S^T / dP^T
      load_half(next, nb > 1 ? 1 : 0);
      mbar_wait(&bars[2], ph ^ 1u);
      tc_fence_after();
      issue_s(0, 0);  // TMEM columns [0,256): free; the epilogue below reads [256,512)
      tc_commit(&bars[0]);
    }
    epi_kv(row0, h, kb_prev);
    // dQ epilogue: query rows i = qb*128 + jl
    for (int qb = 0; qb < nb; ++qb) {
      float v[16];
      tmem_ld16(trow + 384 + qb * 64 + cg * 16, v);
      const int pos = qb * 128 + jl;
      abt_store_row16(a.dqkv, (int64_t)(row0 + pos) * (3 * a.m) + h * 64 + cg * 16, v, th, a.rope != 0, pos,
                      a.scale);
    }
    tc_fence_before();
    __syncthreads();  // next item's Ls / Dv visible; TMEM [256,512) drained before its gradient products
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
}

}  // namespace mecefo
