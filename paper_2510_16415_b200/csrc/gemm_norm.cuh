// Residual GEMM with the following RMSNorm fused (m = 512):
//     x1 = x + A W^T                       (model.py:332, 406: the O projection)
//     inv = 1 / sqrt(mean(x1^2) + eps),  h = (x1 * inv) * g    (model.py:183-186)
// One CTA owns a 128-row block and ALL 512 output columns (one tcgen05
// accumulator of 128 x 512 fp32 = the whole TMEM), so the row reduction of
// the norm needs no cross-CTA exchange: pass 1 adds the TMA-prefetched
// residual, stores x1 (fp32, TMA), accumulates sum(x1^2) per row and writes
// x1 back into TMEM; the two epilogue warps of a lane quadrant combine their
// halves of the row sum; pass 2 re-reads x1 from TMEM and stores h (bf16)
// and inv. Replaces the residual GEMM + rmsnorm_fwd launch pair of the lean /
// full block forward when the pass has >= 100 row blocks (one wave).
#pragma once
#include "gemm.cuh"

namespace mecefo {

constexpr int GN_N = 512;
constexpr int GN_A_BYTES = TC_BM * TC_BK * 2;        // 16 KB
constexpr int GN_B_BYTES = GN_N * TC_BK * 2;         // 64 KB
constexpr int GN_STAGE = GN_A_BYTES + GN_B_BYTES;    // 80 KB
constexpr int GN_STAGES = 2;
constexpr int GN_EPI_BYTES = TC_EPI_WARPS * 2 * TC_STAGE_OUT;  // two 4 KB boxes per epilogue warp
constexpr int GN_SMEM = GN_STAGES * GN_STAGE + GN_EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/ + 1024 /*row sums*/;

struct GnDev {
  int M, K, kblocks;
  float eps;
  const float* gain;  // (512) norm scale
  float* inv;         // (M) out, optional
};

struct GnMaps {
  CUtensorMap a;   // A (M x K bf16, K-major), box 64 x 128
  CUtensorMap b;   // W (512 x K bf16, K-major), box 64 x 256
  CUtensorMap r;   // residual x (M x 512 fp32), box 32 x 32, SW128
  CUtensorMap o;   // x1 out (M x 512 fp32), box 32 x 32, SW128
  CUtensorMap h;   // h out (M x 512 bf16), box 32 x 32, SW64
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_resid_norm_kernel(const __grid_constant__ GnMaps mp, GnDev p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + GN_STAGES * GN_A_BYTES;
  uint8_t* sE = smem + GN_STAGES * GN_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + GN_EPI_BYTES);
  uint64_t* empty = full + GN_STAGES;
  uint64_t* tfull = empty + GN_STAGES;
  uint64_t* rbar = tfull + 1;  // 2 per epilogue warp
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(rbar + 2 * TC_EPI_WARPS);
  float* rowsum = reinterpret_cast<float*>(smem + GN_STAGES * GN_STAGE + GN_EPI_BYTES + 512);  // [2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < GN_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    for (int w = 0; w < 2 * TC_EPI_WARPS; ++w) mbar_init(&rbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  griddep_wait();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int mt = blockIdx.x;  // one 128-row block per CTA

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < p.kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], GN_STAGE);
        const int k0 = kb * TC_BK;
        tma_load_2d(sA + stage * GN_A_BYTES, &mp.a, &full[stage], k0, mt * TC_BM);
        tma_load_2d(sB + stage * GN_B_BYTES, &mp.b, &full[stage], k0, 0);
        tma_load_2d(sB + stage * GN_B_BYTES + 256 * 128, &mp.b, &full[stage], k0, 256);
        if (++stage == GN_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer: two N = 256 products per k-step =====
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < p.kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + stage * GN_A_BYTES);
        const uint32_t b_addr = smem_u32(sB + stage * GN_B_BYTES);
#pragma unroll
        for (int k = 0; k < TC_BK / 16; ++k) {
          const uint64_t ad = make_sdesc(a_addr + k * 32, 16, 1024);
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          tc_mma_bf16(tmem_base, ad, make_sdesc(b_addr + k * 32, 16, 1024), idesc, acc);
          tc_mma_bf16(tmem_base + 256, ad, make_sdesc(b_addr + 256 * 128 + k * 32, 16, 1024), idesc, acc);
        }
        tc_commit(&empty[stage]);
        if (++stage == GN_STAGES) { stage = 0; phase ^= 1; }
      }
      tc_commit(tfull);
    }
  } else if (warp >= 4) {  // ===== epilogue: 8 warps, (lane quadrant, column half) =====
    const int ew = warp - 4, quad = ew & 3, half = ew >> 2;
    uint8_t* box[2] = {sE + ew * 2 * TC_STAGE_OUT, sE + ew * 2 * TC_STAGE_OUT + TC_STAGE_OUT};
    uint32_t rph[2] = {0u, 0u};
    const int r0 = mt * TC_BM + quad * 32;
    const int row = r0 + lane;
    const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16);
    const int c0 = half * 8;  // this warp's 8 chunks of 32 columns
    auto fetch = [&](int i) {  // residual box of chunk c0 + i into box i & 1
      if (lane == 0) {
        mbar_expect_tx(&rbar[2 * ew + (i & 1)], 32 * 32 * 4);
        tma_load_2d(box[i & 1], &mp.r, &rbar[2 * ew + (i & 1)], (c0 + i) * 32, r0);
      }
    };
    fetch(0);
    fetch(1);
    mbar_wait(tfull, 0);
    tc_fence_after();
    float ss = 0.f;
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
      const int col = (c0 + i) * 32;
      float v[32];
      tmem_ld16_nowait(taddr + col, v);
      tmem_ld16_nowait(taddr + col + 16, v + 16);
      tmem_wait_ld();
      mbar_wait(&rbar[2 * ew + (i & 1)], rph[i & 1]);
      rph[i & 1] ^= 1u;
      uint8_t* bx = box[i & 1];
      const uint8_t* rrow = bx + lane * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // + residual (the box's SW128 layout: 16-B unit q of this lane's row)
        const float4 r4 = *reinterpret_cast<const float4*>(rrow + ((q ^ (lane & 7)) << 4));
        v[4 * q] += r4.x; v[4 * q + 1] += r4.y; v[4 * q + 2] += r4.z; v[4 * q + 3] += r4.w;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) ss = fmaf(v[j], v[j], ss);
      __syncwarp();
      stage_write16(bx, v, PREC_F32, 0, lane);
      stage_write16(bx, v + 16, PREC_F32, 1, lane);
      stage_commit(bx, &mp.o, 0, col, r0, lane);  // x1 (fp32)
      tmem_st16(taddr + col, v);                  // x1 back into TMEM for pass 2
      tmem_st16(taddr + col + 16, v + 16);
      if (i + 2 < 8) {
        stage_wait(lane);  // the store just issued has read this box
        fetch(i + 2);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    rowsum[half * 128 + quad * 32 + lane] = ss;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");  // epilogue warps only
    const float tot = rowsum[quad * 32 + lane] + rowsum[128 + quad * 32 + lane];
    const float inv = 1.f / sqrtf(tot / (float)GN_N + p.eps);
    if (half == 0 && p.inv && row < p.M) p.inv[row] = inv;
    // pass 2: h = (x1 * inv) * g (bf16) through the same boxes
    stage_wait(lane);
    int sb = 0;
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
      const int col = (c0 + i) * 32;
      float v[32];
      tmem_ld16_nowait(taddr + col, v);
      tmem_ld16_nowait(taddr + col + 16, v + 16);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(p.gain + col) + q);
        v[4 * q] = (v[4 * q] * inv) * g4.x;
        v[4 * q + 1] = (v[4 * q + 1] * inv) * g4.y;
        v[4 * q + 2] = (v[4 * q + 2] * inv) * g4.z;
        v[4 * q + 3] = (v[4 * q + 3] * inv) * g4.w;
      }
      stage_store32_db(box[0], sb, &mp.h, v, col, r0, lane);  // 2 KB bf16 halves of box 0
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
  }
}

}  // namespace mecefo
