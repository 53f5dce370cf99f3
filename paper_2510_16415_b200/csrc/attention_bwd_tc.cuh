// Tensor-core causal attention backward for head_dim 64, T in {128, 256}
// (bf16), the exact backward of healthy ranks (model.py:336-368).
//
// One CTA per (sequence, head). Q, K, V, dO are TMA-staged once; for every
// causal (key block kb, query block qb >= kb) of 128x128:
//   S^T  = K_kb Q_qb^T,  dP^T = V_kb dO_qb^T          (tcgen05 -> TMEM)
//   P^T  = exp(scale S^T - LSE),  dS^T = P^T (dP^T - D)   (4 warps, key rows)
//   dV_kb += P^T dO_qb,  dK_kb += dS^T Q_qb,  dQ_qb += dS K_kb   (tcgen05)
// The P^T / dS^T smem tiles are written once in the UMMA K-major SW128 layout
// and read back both as K-major A (dV, dK) and as MN-major A (dQ: the same
// bytes describe dS = (dS^T)^T). TMEM holds S^T, dP^T, dV, dK and dQ for both
// query blocks: exactly 512 columns. Scale and the transpose RoPE rotation
// (model.py:291-298) are applied in the epilogues.
#pragma once
#include "gemm.cuh"

namespace mecefo {

struct AttnBwdTcArgs {
  const void* ctx;   // O  (b, m)
  const void* dctx;  // dO (b, m)
  const float* lse;  // (b, H)
  void* dqkv;        // (b, 3m) out
  const float* cosT;
  const float* sinT;
  int T, H, m, rope;
  float scale;
};

constexpr int ABT_THREADS = 128;
constexpr int ABT_SMEM = 4 * 32768 + 2 * 32768 + 2 * 256 * 4 + 1024 + 256;

__device__ __forceinline__ void abt_store_row64(void* base, int64_t idx, const float* v, const AttnBwdTcArgs& a,
                                                int pos, float mul) {
  float w[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) w[c] = v[c] * mul;
  if (a.rope) {
#pragma unroll
    for (int p = 0; p < 32; ++p) {  // transpose rotation (model.py:294-297)
      const float cs = __ldg(a.cosT + pos * 32 + p), sn = __ldg(a.sinT + pos * 32 + p);
      const float e = w[2 * p], o = w[2 * p + 1];
      w[2 * p] = e * cs + o * sn;
      w[2 * p + 1] = -e * sn + o * cs;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + idx);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    uint32_t q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(w[8 * u + 2 * j], w[8 * u + 2 * j + 1]);
      q[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    dst[u] = make_uint4(q[0], q[1], q[2], q[3]);
  }
}

__global__ void __launch_bounds__(ABT_THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tdo,
                       AttnBwdTcArgs a) {
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
  uint64_t* bars = reinterpret_cast<uint64_t*>(Dv + 256);  // 0 load, 1 S, 2 M
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seq = blockIdx.x / a.H, h = blockIdx.x % a.H;
  const int row0 = seq * a.T;
  const int nb = a.T / 128;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
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

  if (threadIdx.x == 0) {
    mbar_expect_tx(&bars[0], 4 * a.T * 128);
    for (int r = 0; r < a.T / 64; ++r) {
      tma_load_2d(sQ + r * 8192, &tqkv, &bars[0], h * 64, row0 + r * 64);
      tma_load_2d(sK + r * 8192, &tqkv, &bars[0], a.m + h * 64, row0 + r * 64);
      tma_load_2d(sV + r * 8192, &tqkv, &bars[0], 2 * a.m + h * 64, row0 + r * 64);
      tma_load_2d(sDO + r * 8192, &tdo, &bars[0], h * 64, row0 + r * 64);
    }
  }
  // LSE and D_i = rowsum(dO * O) (model.py:352) for all T query rows
  for (int i = threadIdx.x; i < a.T; i += ABT_THREADS) {
    const int64_t g = (int64_t)(row0 + i);
    Ls[i] = a.lse[g * a.H + h] * 1.4426950408889634f;  // log2 domain
    const uint4* o = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.ctx) + g * a.m + h * 64);
    const uint4* d = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.dctx) + g * a.m + h * 64);
    float acc = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 ov = o[u], dv = d[u];
      const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&ov);
      const __nv_bfloat162* dh = reinterpret_cast<const __nv_bfloat162*>(&dv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 x = __bfloat1622float2(oh[j]), y = __bfloat1622float2(dh[j]);
        acc += x.x * y.x + x.y * y.y;
      }
    }
    Dv[i] = acc;
  }
  __syncthreads();
  mbar_wait(&bars[0], 0);
  tc_fence_after();

  // K-major A/B, N = 128 (S^T, dP^T); K-major A + MN-major B, N = 64 (dV, dK);
  // MN-major A + MN-major B, N = 64 (dQ).
  constexpr uint32_t id_s = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t id_kv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t id_q =
      (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const float c2 = a.scale * 1.4426950408889634f;
  const int jl = warp * 32 + lane;  // key row (TMEM lane) owned by this thread
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  int blk = 0;
  for (int kb = 0; kb < nb; ++kb) {
    for (int qb = kb; qb < nb; ++qb, ++blk) {
      if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t k_a = smem_u32(sK + kb * 16384), v_a = smem_u32(sV + kb * 16384);
        const uint32_t q_b = smem_u32(sQ + qb * 16384), do_b = smem_u32(sDO + qb * 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          tc_mma_bf16(tmem, make_sdesc(k_a + k * 32, 16, 1024), make_sdesc(q_b + k * 32, 16, 1024), id_s, k > 0);
          tc_mma_bf16(tmem + 128, make_sdesc(v_a + k * 32, 16, 1024), make_sdesc(do_b + k * 32, 16, 1024), id_s,
                      k > 0);
        }
        tc_commit(&bars[1]);
      }
      mbar_wait(&bars[1], blk & 1);
      tc_fence_after();
      // elementwise: P^T, dS^T for key j = kb*128 + jl, queries i = qb*128 + c
      const int j = kb * 128 + jl;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        float s[16], dp[16];
        tmem_ld16(trow + c * 16, s);
        tmem_ld16(trow + 128 + c * 16, dp);
        uint32_t pk[8], dk[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          float pv[2], dv[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int il = c * 16 + 2 * t + e;
            const int i = qb * 128 + il;
            const float p = (i >= j) ? exp2f(s[2 * t + e] * c2 - Ls[i]) : 0.f;
            pv[e] = p;
            dv[e] = p * (dp[2 * t + e] - Dv[i]);
          }
          __nv_bfloat162 hp = __floats2bfloat162_rn(pv[0], pv[1]);
          __nv_bfloat162 hd = __floats2bfloat162_rn(dv[0], dv[1]);
          pk[t] = *reinterpret_cast<uint32_t*>(&hp);
          dk[t] = *reinterpret_cast<uint32_t*>(&hd);
        }
        const int off = (c >> 2) * 16384 + jl * 128;
        const int u0 = (c & 3) * 2;
        *reinterpret_cast<uint4*>(sPt + off + ((u0 ^ (jl & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(sPt + off + (((u0 + 1) ^ (jl & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        *reinterpret_cast<uint4*>(sDSt + off + ((u0 ^ (jl & 7)) << 4)) = make_uint4(dk[0], dk[1], dk[2], dk[3]);
        *reinterpret_cast<uint4*>(sDSt + off + (((u0 + 1) ^ (jl & 7)) << 4)) = make_uint4(dk[4], dk[5], dk[6], dk[7]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncthreads();
      if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t pt = smem_u32(sPt), dst = smem_u32(sDSt);
        const uint32_t q_b = smem_u32(sQ + qb * 16384), do_b = smem_u32(sDO + qb * 16384);
        const uint32_t k_b = smem_u32(sK + kb * 16384);
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
        tc_commit(&bars[2]);
      }
      mbar_wait(&bars[2], blk & 1);
      tc_fence_after();
    }
    // dK_kb, dV_kb epilogue: key rows j = kb*128 + jl
    {
      float v[64];
      const int64_t g = (int64_t)(row0 + kb * 128 + jl) * (3 * a.m);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(trow + 320 + c * 16, v + 16 * c);
      abt_store_row64(a.dqkv, g + a.m + h * 64, v, a, kb * 128 + jl, a.scale);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(trow + 256 + c * 16, v + 16 * c);
      AttnBwdTcArgs nr = a;
      nr.rope = 0;
      abt_store_row64(a.dqkv, g + 2 * a.m + h * 64, v, nr, 0, 1.f);
    }
    tc_fence_before();
    __syncthreads();
  }
  // dQ epilogue: query rows i = qb*128 + jl
  for (int qb = 0; qb < nb; ++qb) {
    float v[64];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld16(trow + 384 + qb * 64 + c * 16, v + 16 * c);
    abt_store_row64(a.dqkv, (int64_t)(row0 + qb * 128 + jl) * (3 * a.m) + h * 64, v, a, qb * 128 + jl, a.scale);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
}

}  // namespace mecefo
