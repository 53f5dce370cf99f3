// Fused FFN recompute + SwiGLU backward on the tensor cores (the MeCeFO
// neighbour-backward hot kernel; approx.py:128-129 -> model.py:214-216,
// 248-253).
//
// For a tile of 128 tokens x 128 FFN columns, ONE kernel accumulates three
// tcgen05 products over the hidden dimension into TMEM:
//     d_act = dy  W_down          (B = W_down read MN-major, no transpose)
//     gate  = h2  W_gate^T        (recomputed)
//     up    = h2  W_up^T          (recomputed)
// and the epilogue emits act = silu(gate)*up, d_gate = d_act*up*silu'(gate)
// and d_up = d_act*silu(gate) through swizzled smem + TMA stores. gate, up and
// d_act never touch HBM, and no epilogue operand is read from
// global memory.
//
// The kernel is bound by shared-memory bandwidth (TMA fills + MMA operand
// reads of narrow-N products). Measured history: 64 pair columns per tile
// with double-buffered TMEM 98-103 us / layer at C1; a 2-CTA cluster variant
// multicasting dy / h2 across column-tile pairs gave no gain (the operands
// are read from smem by the MMAs regardless); 128 pair columns with the TMEM
// ring below 95 us (92.5 us with double-buffered staging); 16 epilogue warps
// (32 columns each, 1 KB boxes, one operand stage fewer) measured 94.7 us.
#pragma once
#include "gemm.cuh"

namespace mecefo {

struct DualDev {
  int M, NP, K;     // tokens, FFN width f, hidden m
  int64_t f_off;    // row offset of W_up inside W_gu (= f)
  int kblocks, tiles_m, tiles_n, num_tiles;
  int has_act;
  int dbg;  // timing experiments only (MECEFO_TIMING_KNOBS builds): 1 = epilogue skips math/stores,
            // 2 = gate|up product does not wait for the previous epilogue (results invalid)
};

// ---------------------------------------------------------------------------
// 128-pair-column variant. Twice the columns per tile halve the A-operand
// (dy, h2) shared-memory traffic per flop — the 64-column kernel is bound by
// shared-memory bandwidth (TMA fills + N=64/128 MMA operand reads). d_act,
// gate and up (3 x 128 fp32 columns) no longer double-buffer in 512 TMEM
// columns, so TMEM is a ring of four 128-column blocks: tile i takes blocks
// 3i, 3i+1, 3i+2 (mod 4). The d_act product of tile i+1 goes to the one block
// tile i does not use and runs while the epilogue drains tile i; its gate|up
// product waits for that epilogue. Stages alternate d-phase (dy + W_down
// slice) and gu-phase (h2 + gate|up rows) k-blocks.
// ---------------------------------------------------------------------------
constexpr int D2_NP = 128;
constexpr int D2_STAGE_BYTES = TC_BM * TC_BK * 2 + 2 * D2_NP * TC_BK * 2;  // 16 KB A + 32 KB B (max of the phases)
constexpr int D2_STAGES = 4;
constexpr int D2_SMEM = D2_STAGES * D2_STAGE_BYTES + TC_EPI_WARPS * TC_STAGE_OUT + 1024 + 256;

__global__ void __launch_bounds__(TC_THREADS, 1)
    swiglu_bwd_dual128_kernel(const __grid_constant__ CUtensorMap tmDy, const __grid_constant__ CUtensorMap tmH2,
                              const __grid_constant__ CUtensorMap tmWd, const __grid_constant__ CUtensorMap tmWgu,
                              const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmDg,
                              const __grid_constant__ CUtensorMap tmDu, DualDev p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sE = smem + D2_STAGES * D2_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + TC_EPI_WARPS * TC_STAGE_OUT);
  uint64_t* empty = full + D2_STAGES;
  uint64_t* tfull = empty + D2_STAGES;  // MMA -> epilogue, one phase per tile
  uint64_t* edone = tfull + 1;          // epilogue has read a tile's TMEM, one phase per tile
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(edone + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < D2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(edone, 32 * TC_EPI_WARPS);
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

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer: per tile, kblocks d-stages then kblocks gu-stages =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int mt = t % p.tiles_m, nt = t / p.tiles_m;
        for (int ph = 0; ph < 2; ++ph) {
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * D2_STAGE_BYTES;
            const int k0 = kb * TC_BK;
            if (ph == 0) {  // dy tile + W_down slice (MN-major, two 64-column boxes)
              mbar_expect_tx(&full[stage], TC_BM * TC_BK * 2 + D2_NP * TC_BK * 2);
              tma_load_2d(st, &tmDy, &full[stage], k0, mt * TC_BM);
              tma_load_2d(st + 16384, &tmWd, &full[stage], nt * D2_NP, k0);
              tma_load_2d(st + 16384 + 8192, &tmWd, &full[stage], nt * D2_NP + 64, k0);
            } else {        // h2 tile + gate rows + up rows (K-major, 128-row boxes)
              mbar_expect_tx(&full[stage], D2_STAGE_BYTES);
              tma_load_2d(st, &tmH2, &full[stage], k0, mt * TC_BM);
              tma_load_2d(st + 16384, &tmWgu, &full[stage], k0, nt * D2_NP);
              tma_load_2d(st + 16384 + 16384, &tmWgu, &full[stage], k0, nt * D2_NP + (int)p.f_off);
            }
            if (++stage == D2_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      constexpr uint32_t id_d = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((128u >> 3) << 17) |
                                ((128u >> 4) << 24);  // A K-major, B MN-major, N = 128
      constexpr uint32_t id_g1 = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t id_g2 = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int seen = 0;  // epilogue completions observed
      int it = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        const uint32_t bD = (3 * it) & 3, bG = (3 * it + 1) & 3, bU = (3 * it + 2) & 3;
        for (int ph = 0; ph < 2; ++ph) {
          // d-phase reuses the block tile it-2 held; gu-phase the blocks of tile it-1
          const int need = (p.dbg & 2) ? -1 : it - 2 + ph;
          while (seen <= need) {
            mbar_wait(edone, seen & 1);
            ++seen;
          }
          tc_fence_after();
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + stage * D2_STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k) {
              const uint32_t acc_on = (kb > 0 || k > 0) ? 1u : 0u;
              const uint64_t ad = make_sdesc(st + k * 32, 16, 1024);
              if (ph == 0) {
                tc_mma_bf16(tmem_base + bD * 128, ad, make_sdesc(st + 16384 + k * 2048, 8192, 1024), id_d, acc_on);
              } else if (bU == bG + 1) {  // gate|up adjacent in TMEM: one N = 256 MMA
                tc_mma_bf16(tmem_base + bG * 128, ad, make_sdesc(st + 16384 + k * 32, 16, 1024), id_g2, acc_on);
              } else {
                tc_mma_bf16(tmem_base + bG * 128, ad, make_sdesc(st + 16384 + k * 32, 16, 1024), id_g1, acc_on);
                tc_mma_bf16(tmem_base + bU * 128, ad, make_sdesc(st + 32768 + k * 32, 16, 1024), id_g1, acc_on);
              }
            }
            tc_commit(&empty[stage]);
            if (++stage == D2_STAGES) { stage = 0; phase ^= 1; }
          }
        }
        tc_commit(tfull);
      }
    }
  } else if (warp >= 4) {  // ===== epilogue: 8 warps, two 32-column chunks each =====
    const int ew = warp - 4, quad = ew & 3, half = ew >> 2;
    uint8_t* stg = sE + ew * TC_STAGE_OUT;
    int sb = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int mt = t % p.tiles_m, nt = t / p.tiles_m;
      const uint32_t bD = (3 * it) & 3, bG = (3 * it + 1) & 3, bU = (3 * it + 2) & 3;
      mbar_wait(tfull, it & 1);
      tc_fence_after();
      const int r0 = mt * TC_BM + quad * 32;
      const uint32_t lanes = tmem_base + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        const int c = half * 2 + cc;
        float d[32], g[32], u[32];
        tmem_ld16_nowait(lanes + bD * 128 + c * 32, d);
        tmem_ld16_nowait(lanes + bD * 128 + c * 32 + 16, d + 16);
        tmem_ld16_nowait(lanes + bG * 128 + c * 32, g);
        tmem_ld16_nowait(lanes + bG * 128 + c * 32 + 16, g + 16);
        tmem_ld16_nowait(lanes + bU * 128 + c * 32, u);
        tmem_ld16_nowait(lanes + bU * 128 + c * 32 + 16, u + 16);
        tmem_wait_ld();
        if (cc == 1) {  // this warp's TMEM reads of the tile are done
          tc_fence_before();
          mbar_arrive(edone);
        }
        const int n0 = nt * D2_NP + c * 32;
        if (n0 < p.NP && !(p.dbg & 1)) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float sg = sigmoid_ieee_f(g[j]);
            const float act = g[j] * sg * u[j];
            const float dg = (d[j] * u[j]) * (sg * (1.f + g[j] * (1.f - sg)));
            const float du = d[j] * (g[j] * sg);
            g[j] = dg;
            u[j] = du;
            d[j] = act;
          }
          // three bf16 boxes through the warp's two 2 KB staging halves (measured 2% faster here)
          if (p.has_act) stage_store32_db(stg, sb, &tmAct, d, n0, r0, lane);
          stage_store32_db(stg, sb, &tmDg, g, n0, r0, lane);
          stage_store32_db(stg, sb, &tmDu, u, n0, r0, lane);
        }
      }
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
