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
  // direct epilogue stores (no smem staging): act (ld f) and [d_gate | d_up] (ld 2f)
  __nv_bfloat16* act;
  __nv_bfloat16* dcat;
  int direct;
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
// 32 fp32 values -> bf16, up to `cnt` columns at p (16-byte vectors when whole).
__device__ __forceinline__ void store_row32_bf16(__nv_bfloat16* p, const float* v, int cnt) {
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  if (cnt == 32 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      reinterpret_cast<uint4*>(p)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < cnt) p[j] = __float2bfloat16_rn(v[j]);
  }
}

// SwiGLU backward of one element (model.py:198-204, 216, 250-253), ~11
// instructions: s = sigmoid(g) by MUFU ex2 + rcp.approx, gs = silu(g),
// (measured: a one-MUFU tanh.approx sigmoid saved 1.1 us of 82 per launch but
// raised the C1 gate/up gradient errors above the bf16-autocast level, 1.27x)
//   act = gs u,  d_up = d gs,  d_gate = d u s (1 + g (1 - s)) = d u (s + gs - gs s).
// In: g = gate, u = up, d = d_act; out: g = d_gate, u = d_up, d = act.
__device__ __forceinline__ void swiglu_bwd_elem(float& g, float& u, float& d) {
  const float s = rcp_approx(1.f + ex2_approx(-1.4426950408889634f * g));
  const float gs = g * s;
  const float du = d * gs;
  const float dg = (d * u) * (s + fmaf(-gs, s, gs));
  d = gs * u;
  g = dg;
  u = du;
}

// A 32 x 32 bf16 box (lane = row, v = its 32 columns) stored through the
// warp's 2 KB staging box with coalesced 16-byte st.global (8 rows x 64 B per
// instruction): no TMA-unit round trip and no completion waits — the box is
// reused after a warp barrier. gp points at (row 0, column 0) of the box,
// ld in elements; rows >= rows_left and columns >= cnt (a multiple of 8) are
// not written.
__device__ __forceinline__ void stage_store32_lsu(uint8_t* box, const float* v, __nv_bfloat16* gp, int64_t ld,
                                                  int rows_left, int cnt, int lane) {
  stage_write16(box, v, PREC_BF16, 0, lane);
  stage_write16(box, v + 16, PREC_BF16, 1, lane);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = k * 32 + lane, row = q >> 2, u = q & 3;
    const uint4 w = *reinterpret_cast<const uint4*>(box + row * 64 + ((u ^ ((row >> 1) & 3)) << 4));
    if (row < rows_left && u * 8 < cnt) *reinterpret_cast<uint4*>(gp + row * ld + u * 8) = w;
  }
  __syncwarp();
}

// 32 fp32 -> 16 bf16x2 words (the packed form an epilogue keeps while it
// loads its next chunk).
__device__ __forceinline__ void pack32_bf16(const float* v, uint32_t* w) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&h);
  }
}
// stage_store32_db for an already packed bf16 32-column row segment.
__device__ __forceinline__ void stage_store32_db_packed(uint8_t* stg, int& sb, const CUtensorMap* map,
                                                        const uint32_t* w, int c0, int r0, int lane) {
  uint8_t* box = stg + sb * 2048;
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
  uint8_t* row = box + lane * 64;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    *reinterpret_cast<uint4*>(row + ((u ^ ((lane >> 1) & 3)) << 4)) =
        make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
  stage_commit(box, map, 0, c0, r0, lane);
  sb ^= 1;
}

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
          for (int j = 0; j < 32; ++j) swiglu_bwd_elem(g[j], u[j], d[j]);
          if (p.direct == 2) {  // coalesced LSU stores through the staging box
            const int64_t f = p.NP;
            const int cnt = min(32, p.NP - n0), rl = p.M - r0;
            if (p.has_act) stage_store32_lsu(stg, d, p.act + (int64_t)r0 * f + n0, f, rl, cnt, lane);
            stage_store32_lsu(stg, g, p.dcat + (int64_t)r0 * 2 * f + n0, 2 * f, rl, cnt, lane);
            stage_store32_lsu(stg, u, p.dcat + (int64_t)r0 * 2 * f + f + n0, 2 * f, rl, cnt, lane);
          } else if (p.direct) {  // each lane's row segment of 32 bf16 straight to global (no smem traffic)
            const int row = r0 + lane;
            if (row < p.M) {
              const int64_t f = p.NP;
              if (p.has_act) store_row32_bf16(p.act + (int64_t)row * f + n0, d, min(32, p.NP - n0));
              store_row32_bf16(p.dcat + (int64_t)row * 2 * f + n0, g, min(32, p.NP - n0));
              store_row32_bf16(p.dcat + (int64_t)row * 2 * f + f + n0, u, min(32, p.NP - n0));
            }
          } else {
            // three bf16 boxes through the warp's two 2 KB staging halves (measured 2% faster here)
            if (p.has_act) stage_store32_db(stg, sb, &tmAct, d, n0, r0, lane);
            stage_store32_db(stg, sb, &tmDg, g, n0, r0, lane);
            stage_store32_db(stg, sb, &tmDu, u, n0, r0, lane);
          }
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

namespace mecefo {

// ---------------------------------------------------------------------------
// CTA-pair (cta_group::2) variant. A cluster of 2 CTAs computes a 256-token x
// 128-pair-column tile with M = 256 tcgen05 MMAs issued by the leader CTA:
// each CTA stages its own 128 rows of dy / h2 (A) but only HALF of the B
// operand — W_down columns [64 crank, 64 crank + 64) of the tile, and gate /
// up rows [64 crank, 64 crank + 64) — which the pair's tensor cores share.
// Per SM that cuts the shared-memory traffic of a k-block (TMA fill + MMA
// operand read) from 64 + 96 KB to 48 + 64 KB; the measured mainloop-only
// time of the single-CTA kernel (70 of 92 us at C1) is bound there.
// TMEM per CTA (its 128 rows): gate|up of the tile in columns [0, 256) as ONE
// N = 256 product — [g 0-63 | u 0-63] from the leader's B half, [g 64-127 |
// u 64-127] from the peer's — and d_act in [256, 384) or [384, 512)
// alternating, so the d_act product of tile i+1 runs under tile i's
// epilogue. Barriers: stage `full` lives in the leader (both CTAs' TMA bytes
// land there), `empty` / `tfull` in both (multicast commits), `edone` in the
// leader (16 epilogue-warp arrivals, 8 of them remote).
// ---------------------------------------------------------------------------
constexpr int D2S_STAGE_BYTES = TC_BM * TC_BK * 2 + D2_NP * TC_BK * 2;  // 16 KB A + 16 KB B half (gu-phase)
// EPW epilogue warps: 8 (two 32-column chunks each, 6 operand stages) or 16
// (one chunk each: a warp loads its chunk's d_act / gate / up from TMEM and
// releases the tile's TMEM right away, so the next tile's gate|up product is
// not held up by the SwiGLU math and stores; 5 operand stages).
template <int EPW>
struct D2S {
  static constexpr int STAGES = EPW == 16 ? 5 : 6;
  static constexpr int THREADS = 128 + 32 * EPW;
  static constexpr int SMEM = STAGES * D2S_STAGE_BYTES + EPW * TC_STAGE_OUT + 1024 + 256;
};

// Release-first epilogue helpers (swiglu_bwd_dual2sm_kernel<8>): a chunk's
// d_act / gate / up (32 columns of one TMEM lane row each) read 8 columns at
// a time and kept as bf16 pairs; then, after the tile's TMEM is released,
// the SwiGLU backward in place and the three staged bf16 stores.
__device__ __forceinline__ void dual_load_chunk_bf16(uint32_t lanes, uint32_t dcol, int c, uint32_t (&w)[48]) {
  const uint32_t gcol = (uint32_t)((c >> 1) * 128 + (c & 1) * 32), ucol = gcol + 64u;
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // 8 columns at a time: 24 fp32 registers in flight
    float d[8], g[8], u[8];
    tmem_ld8_nowait(lanes + dcol + c * 32 + q * 8, d);
    tmem_ld8_nowait(lanes + gcol + q * 8, g);
    tmem_ld8_nowait(lanes + ucol + q * 8, u);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 a2 = __floats2bfloat162_rn(d[2 * j], d[2 * j + 1]);
      __nv_bfloat162 g2 = __floats2bfloat162_rn(g[2 * j], g[2 * j + 1]);
      __nv_bfloat162 u2 = __floats2bfloat162_rn(u[2 * j], u[2 * j + 1]);
      w[q * 4 + j] = *reinterpret_cast<uint32_t*>(&a2);
      w[16 + q * 4 + j] = *reinterpret_cast<uint32_t*>(&g2);
      w[32 + q * 4 + j] = *reinterpret_cast<uint32_t*>(&u2);
    }
  }
}
__device__ __forceinline__ void dual_finish_chunk(uint32_t (&w)[48], uint8_t* stg, int& sb, const CUtensorMap* tmAct,
                                                  const CUtensorMap* tmDg, const CUtensorMap* tmDu, int has_act,
                                                  int n0, int r0, int lane) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {  // word j of d / g / u -> act / d_gate / d_up
    // bf16 -> fp32 by bit placement (no address taken: w stays in registers)
    float d0 = __uint_as_float(w[j] << 16), d1 = __uint_as_float(w[j] & 0xffff0000u);
    float g0 = __uint_as_float(w[16 + j] << 16), g1 = __uint_as_float(w[16 + j] & 0xffff0000u);
    float u0 = __uint_as_float(w[32 + j] << 16), u1 = __uint_as_float(w[32 + j] & 0xffff0000u);
    swiglu_bwd_elem(g0, u0, d0);
    swiglu_bwd_elem(g1, u1, d1);
    __nv_bfloat162 a2 = __floats2bfloat162_rn(d0, d1), g2 = __floats2bfloat162_rn(g0, g1),
                   u2 = __floats2bfloat162_rn(u0, u1);
    w[j] = *reinterpret_cast<uint32_t*>(&a2);
    w[16 + j] = *reinterpret_cast<uint32_t*>(&g2);
    w[32 + j] = *reinterpret_cast<uint32_t*>(&u2);
  }
  if (has_act) stage_store32_db_packed(stg, sb, tmAct, w, n0, r0, lane);
  stage_store32_db_packed(stg, sb, tmDg, w + 16, n0, r0, lane);
  stage_store32_db_packed(stg, sb, tmDu, w + 32, n0, r0, lane);
}

template <int EPW>
__global__ void __launch_bounds__(D2S<EPW>::THREADS, 1)
    swiglu_bwd_dual2sm_kernel(const __grid_constant__ CUtensorMap tmDy, const __grid_constant__ CUtensorMap tmH2,
                              const __grid_constant__ CUtensorMap tmWd, const __grid_constant__ CUtensorMap tmWg,
                              const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmDg,
                              const __grid_constant__ CUtensorMap tmDu, DualDev p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int D2S_STAGES = D2S<EPW>::STAGES;
  uint8_t* sE = smem + D2S_STAGES * D2S_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + EPW * TC_STAGE_OUT);
  uint64_t* empty = full + D2S_STAGES;
  uint64_t* tfull = empty + D2S_STAGES;
  uint64_t* edone = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(edone + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < D2S_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(edone, 2 * EPW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {  // the pair's TMEM, allocated by the same warp of both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote signal
  griddep_wait();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer (both CTAs) =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < p.num_tiles; t += npairs) {
        const int mt = t % p.tiles_m, nt = t / p.tiles_m;
        const int row0 = mt * 2 * TC_BM + (int)crank * TC_BM;
        for (int ph = 0; ph < 2; ++ph) {
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * D2S_STAGE_BYTES;
            const int k0 = kb * TC_BK;
            const bool skipA = (p.dbg & 4) && nt != 0;  // timing experiment: A re-reads elided
            if (ph == 0) {  // dy rows + this CTA's 64 W_down columns (MN-major)
              if (leader) mbar_expect_tx(&full[stage], 2 * ((skipA ? 0 : TC_BM * TC_BK * 2) + 64 * TC_BK * 2));
              if (!skipA) tma_load_2d_2sm(st, &tmDy, &full[stage], k0, row0);
              tma_load_2d_2sm(st + 16384, &tmWd, &full[stage], nt * D2_NP + (int)crank * 64, k0);
            } else {        // h2 rows + this CTA's 64 gate rows and 64 up rows (K-major)
              if (leader) mbar_expect_tx(&full[stage], 2 * D2S_STAGE_BYTES - (skipA ? 2 * TC_BM * TC_BK * 2 : 0));
              if (!skipA) tma_load_2d_2sm(st, &tmH2, &full[stage], k0, row0);
              tma_load_2d_2sm(st + 16384, &tmWg, &full[stage], k0, nt * D2_NP + (int)crank * 64);
              tma_load_2d_2sm(st + 16384 + 8192, &tmWg, &full[stage], k0,
                              (int)p.f_off + nt * D2_NP + (int)crank * 64);
            }
            if (++stage == D2S_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ===== MMA issuer (leader CTA only) =====
      constexpr uint32_t id_d = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((128u >> 3) << 17) |
                                ((256u >> 4) << 24);  // M = 256, N = 128, B MN-major
      constexpr uint32_t id_gu = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int seen = 0;
      int it = 0;
      for (int t = pair; t < p.num_tiles; t += npairs, ++it) {
        const uint32_t dcol = 256u + 128u * (uint32_t)(it & 1);
        for (int ph = 0; ph < 2; ++ph) {
          const int need = (p.dbg & 2) ? -1 : it - 2 + ph;  // d: tile it-2 freed this block; gu: tile it-1
          while (seen <= need) {
            mbar_wait(edone, seen & 1);
            ++seen;
          }
          tc_fence_after();
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + stage * D2S_STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k) {
              const uint32_t acc_on = (kb > 0 || k > 0) ? 1u : 0u;
              const uint64_t ad = make_sdesc(st + k * 32, 16, 1024);
              if (ph == 0)
                tc_mma_bf16_2sm(tmem_base + dcol, ad, make_sdesc(st + 16384 + k * 2048, 8192, 1024), id_d, acc_on);
              else
                tc_mma_bf16_2sm(tmem_base, ad, make_sdesc(st + 16384 + k * 32, 16, 1024), id_gu, acc_on);
            }
            tc_commit_2sm_mc(&empty[stage], 0x3);
            if (++stage == D2S_STAGES) { stage = 0; phase ^= 1; }
          }
        }
        tc_commit_2sm_mc(tfull, 0x3);
      }
    }
  } else if (warp >= 4) {  // ===== epilogue (both CTAs) =====
    const int ew = warp - 4, quad = ew & 3;
    constexpr int CPW = 16 / EPW;  // 32-column chunks per warp (4 per quadrant, EPW / 4 warps per quadrant)
    const int cbase = (ew >> 2) * CPW;
    uint8_t* stg = sE + ew * TC_STAGE_OUT;
    int sb = 0;
    int it = 0;
    for (int t = pair; t < p.num_tiles; t += npairs, ++it) {
      const int mt = t % p.tiles_m, nt = t / p.tiles_m;
      const uint32_t dcol = 256u + 128u * (uint32_t)(it & 1);
      mbar_wait(tfull, it & 1);
      tc_fence_after();
      const int r0 = mt * 2 * TC_BM + (int)crank * TC_BM + quad * 32;
      const uint32_t lanes = tmem_base + ((uint32_t)(quad * 32) << 16);
      if constexpr (CPW == 2) {
#ifndef MECEFO_TIMING_KNOBS
        // Release-first: both chunks' d_act / gate / up are read from TMEM and
        // kept as bf16 pairs (48 words per chunk: the bf16 values a bf16
        // autocast step would hold for these GEMM outputs), the tile's TMEM
        // goes back to the leader's MMA right after the second read, and the
        // SwiGLU backward math and the six staged stores run off the
        // critical path, overlapping the next tile's gate|up product.
        uint32_t w0[48], w1[48];  // per chunk: d words 0-15 | g 16-31 | u 32-47
        dual_load_chunk_bf16(lanes, dcol, cbase, w0);
        dual_load_chunk_bf16(lanes, dcol, cbase + 1, w1);
        tc_fence_before();  // this warp's TMEM reads of the tile are done: release to the leader's MMA
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(edone, 0);
        const int n00 = nt * D2_NP + cbase * 32, n01 = n00 + 32;
        if (n00 < p.NP && r0 < p.M) dual_finish_chunk(w0, stg, sb, &tmAct, &tmDg, &tmDu, p.has_act, n00, r0, lane);
        if (n01 < p.NP && r0 < p.M) dual_finish_chunk(w1, stg, sb, &tmAct, &tmDg, &tmDu, p.has_act, n01, r0, lane);
#else
        // Early release: chunk 0 is loaded, computed and kept PACKED (48
        // words) while chunk 1 is loaded; the tile's TMEM is released right
        // after that second load — before any store — so the next tile's
        // gate|up product waits for two TMEM reads and one SwiGLU pass
        // instead of a whole chunk's three staged stores as well.
        uint32_t pa[16], pg[16], pu[16];
        const int c0 = cbase, n00 = nt * D2_NP + c0 * 32;
        const bool ok0 = n00 < p.NP && r0 < p.M;
        {
          const uint32_t gcol = (uint32_t)((c0 >> 1) * 128 + (c0 & 1) * 32), ucol = gcol + 64u;
          float d[32], g[32], u[32];
          tmem_ld16_nowait(lanes + dcol + c0 * 32, d);
          tmem_ld16_nowait(lanes + dcol + c0 * 32 + 16, d + 16);
          tmem_ld16_nowait(lanes + gcol, g);
          tmem_ld16_nowait(lanes + gcol + 16, g + 16);
          tmem_ld16_nowait(lanes + ucol, u);
          tmem_ld16_nowait(lanes + ucol + 16, u + 16);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) swiglu_bwd_elem(g[j], u[j], d[j]);
          pack32_bf16(d, pa);
          pack32_bf16(g, pg);
          pack32_bf16(u, pu);
        }
        const int c1 = cbase + 1, n01 = nt * D2_NP + c1 * 32;
        const uint32_t gcol = (uint32_t)((c1 >> 1) * 128 + (c1 & 1) * 32), ucol = gcol + 64u;
        float d[32], g[32], u[32];
        tmem_ld16_nowait(lanes + dcol + c1 * 32, d);
        tmem_ld16_nowait(lanes + dcol + c1 * 32 + 16, d + 16);
        tmem_ld16_nowait(lanes + gcol, g);
        tmem_ld16_nowait(lanes + gcol + 16, g + 16);
        tmem_ld16_nowait(lanes + ucol, u);
        tmem_ld16_nowait(lanes + ucol + 16, u + 16);
        tmem_wait_ld();
        tc_fence_before();  // this warp's TMEM reads of the tile are done: release to the leader's MMA
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(edone, 0);
        if (ok0 && !(p.dbg & 1)) {  // (dbg: timing experiments only)
          if (p.has_act) stage_store32_db_packed(stg, sb, &tmAct, pa, n00, r0, lane);
          stage_store32_db_packed(stg, sb, &tmDg, pg, n00, r0, lane);
          stage_store32_db_packed(stg, sb, &tmDu, pu, n00, r0, lane);
        }
        if (n01 < p.NP && r0 < p.M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) swiglu_bwd_elem(g[j], u[j], d[j]);
          if (p.dbg & 1) {  // timing experiments only: keep the math, drop the stores
            float sink = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) sink += d[j] + g[j] + u[j];
            if (sink == 12345.f) p.act[0] = __float2bfloat16_rn(sink);
            continue;
          }
          if (p.has_act) stage_store32_db(stg, sb, &tmAct, d, n01, r0, lane);
          stage_store32_db(stg, sb, &tmDg, g, n01, r0, lane);
          stage_store32_db(stg, sb, &tmDu, u, n01, r0, lane);
        }
#endif
      } else {
#pragma unroll 1
      for (int cc = 0; cc < CPW; ++cc) {
        const int c = cbase + cc;
        const uint32_t gcol = (uint32_t)((c >> 1) * 128 + (c & 1) * 32), ucol = gcol + 64u;
        float d[32], g[32], u[32];
        tmem_ld16_nowait(lanes + dcol + c * 32, d);
        tmem_ld16_nowait(lanes + dcol + c * 32 + 16, d + 16);
        tmem_ld16_nowait(lanes + gcol, g);
        tmem_ld16_nowait(lanes + gcol + 16, g + 16);
        tmem_ld16_nowait(lanes + ucol, u);
        tmem_ld16_nowait(lanes + ucol + 16, u + 16);
        tmem_wait_ld();
        if (cc == CPW - 1) {  // this warp's TMEM reads of the tile are done: release to the leader's MMA
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(edone, 0);
        }
        const int n0 = nt * D2_NP + c * 32;
        if (n0 < p.NP && r0 < p.M && !(p.dbg & 1)) {
#pragma unroll
          for (int j = 0; j < 32; ++j) swiglu_bwd_elem(g[j], u[j], d[j]);
          if (p.direct == 2) {  // coalesced LSU stores through the staging box
            const int64_t f = p.NP;
            const int cnt = min(32, p.NP - n0), rl = p.M - r0;
            if (p.has_act) stage_store32_lsu(stg, d, p.act + (int64_t)r0 * f + n0, f, rl, cnt, lane);
            stage_store32_lsu(stg, g, p.dcat + (int64_t)r0 * 2 * f + n0, 2 * f, rl, cnt, lane);
            stage_store32_lsu(stg, u, p.dcat + (int64_t)r0 * 2 * f + f + n0, 2 * f, rl, cnt, lane);
          } else {
            // three bf16 32x32 boxes through the warp's double-buffered staging (TMA clips rows >= M)
            if (p.has_act) stage_store32_db(stg, sb, &tmAct, d, n0, r0, lane);
            stage_store32_db(stg, sb, &tmDg, g, n0, r0, lane);
            stage_store32_db(stg, sb, &tmDu, u, n0, r0, lane);
          }
        }
      }
      }  // CPW != 2
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the pair is done with TMEM and every remote barrier
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
  }
}

}  // namespace mecefo
