// GEMM engine: C[m, n] = sum_k A(m, k) * B(n, k) with fused epilogues.
//
// Two kernels share one epilogue layer:
//  * gemm_tc_kernel   — bf16 operands on the 5th-gen tensor cores: TMA
//    (SWIZZLE_128B) -> shared-memory ring -> tcgen05.mma (one elected thread)
//    -> double-buffered TMEM accumulator -> 4 epilogue warps (tcgen05.ld).
//    Persistent over output tiles, optional split-K (atomic epilogue).
//    Operands may be K-major or MN-major, which is what lets every
//    contraction in the MeCeFO step (Fprop, Dgrad, the long-K Wgrad and the
//    low-rank d2^T (x V1) V1^T chain) run without transposing activations.
//  * gemm_simt_kernel — fp32 FFMA path used for the fp32 parity mode
//    (tcgen05 has no fp32 MMA).
//
// "Paired" mode computes two accumulators per output column n: rows n and
// n + pair_off of B. It is how the gate/up projections share one GEMM while
// each thread of the epilogue holds matching gate_n and up_n values (SwiGLU
// epilogues), without an interleaved weight copy.
#pragma once
#include "common.cuh"
#include <cuda.h>

namespace mecefo {

enum EpiKind : int {
  EPI_STORE = 0,              // out = alpha*acc (+ beta*out) (+ residual); f32 or bf16 out
  EPI_ATOMIC = 1,             // out += alpha*acc (fp32 atomics; split-K / accumulate)
  EPI_SWIGLU_FWD = 2,         // paired: act = silu(g)*u -> out; optional gate/up -> out2
  EPI_SWIGLU_BWD_RECOMP = 3,  // paired (recomputed g,u) + aux = d_act -> act (out), d_gate/d_up (out2)
  EPI_SWIGLU_BWD_CACHED = 4,  // acc = d_act; aux = cached gate/up -> d_gate/d_up (out2)
};

struct Epilogue {
  int kind;
  void* out;
  int64_t ldo;
  int out_prec;
  float alpha;
  float beta;
  const float* residual;
  int64_t ldr;
  void* out2;
  int64_t ldo2;
  int64_t off2;
  const void* aux;
  int64_t ldaux;
  int64_t offaux;
  int act_prec;
  // RoPE on the q|k columns [0, rope_cols) of a QKV projection (model.py:281-288):
  // interleaved (even, odd) pairs rotated by pos * theta_j, pos = row % rope_T.
  const float* rope_cos;
  const float* rope_sin;
  const float* rope_theta;  // theta_j, j < hd/2 (tcgen05 epilogue computes the angles)
  int rope_T, rope_hd, rope_cols;
};

struct GemmDev {
  int M, N, K;           // N = logical output columns (pair columns in paired mode)
  int paired;            // 0/1
  int64_t pair_off;      // B row offset of the second accumulator (paired)
  int64_t b_diag_off;    // block-diagonal batching: M tile mt reads B N-coordinates + (mt / b_diag_div) * b_diag_off
  int b_diag_div;        // M tiles per diagonal block (>= 1)
  int split;             // number of K splits
  int kb_per_split;      // k-blocks (of 64) per split
  int kblocks;           // total k-blocks
  int tiles_m, tiles_n, num_tiles;
  int tiles_m_cl, num_tiles_cl;  // tiles in units of CTA clusters along M (CL = 1 or 2); x groups
  int split_tiles;               // tiles_m_cl * tiles_n * split (one group)
  int n_fast;                    // tile order: N fastest (A-heavy GEMMs: the N tiles of an A row block run together)
  int b_split;                   // K-major B (single CTA, unpaired) loaded as two BN/2-row boxes
  Epilogue epi;
};

// Tensor maps of one launch. NG > 1: a grouped launch — NG independent
// products of identical shape (e.g. the same low-rank contraction of every
// lean layer), each with its own A, B and slot-0 output; the tile index
// decodes to (group, tile).
template <int NG>
struct alignas(64) TcMaps {
  CUtensorMap a[NG];
  CUtensorMap b[NG];
  CUtensorMap o0[NG];
  CUtensorMap o1, o2;  // paired SwiGLU outputs (NG == 1 only)
  CUtensorMap r;       // fp32 residual boxes (NG == 1 only)
};

// ---------------------------------------------------------------------------
// Epilogue application on 16 consecutive output columns of one row.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void store16(void* base, int64_t idx, const float* v, int cnt, int prec) {
  if (prec == PREC_BF16) {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(base) + idx;
    if (cnt == 16 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      uint4 w[2];
      uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        wp[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      reinterpret_cast<uint4*>(p)[0] = w[0];
      reinterpret_cast<uint4*>(p)[1] = w[1];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < cnt) p[j] = f2bf(v[j]);
    }
  } else {
    float* p = reinterpret_cast<float*>(base) + idx;
    if (cnt == 16 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        reinterpret_cast<float4*>(p)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < cnt) p[j] = v[j];
    }
  }
}

__device__ __forceinline__ void load16(const void* base, int64_t idx, float* v, int cnt, int prec) {
  if (prec == PREC_BF16) {
    const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(base) + idx;
    if (cnt == 16 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      uint4 w[2];
      w[0] = reinterpret_cast<const uint4*>(p)[0];
      w[1] = reinterpret_cast<const uint4*>(p)[1];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(w);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = j < cnt ? bf2f(p[j]) : 0.f;
    }
  } else {
    const float* p = reinterpret_cast<const float*>(base) + idx;
    if (cnt == 16 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4 f = reinterpret_cast<const float4*>(p)[j];
        v[4 * j] = f.x; v[4 * j + 1] = f.y; v[4 * j + 2] = f.z; v[4 * j + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = j < cnt ? p[j] : 0.f;
    }
  }
}

__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Non-paired epilogue: v holds acc for columns n0..n0+cnt-1 of row r.
__device__ __forceinline__ void epi_apply(const Epilogue& e, int r, int n0, int cnt, float* v) {
  if (e.kind == EPI_STORE) {
    const int64_t idx = (int64_t)r * e.ldo + n0;
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] *= e.alpha;
    if (e.rope_cos && n0 < e.rope_cols) {
      const int pos = r % e.rope_T, half = e.rope_hd >> 1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = n0 + 2 * j;
        if (c < e.rope_cols) {
          const int pi = pos * half + ((c % e.rope_hd) >> 1);
          const float cs = e.rope_cos[pi], sn = e.rope_sin[pi];
          const float ev = v[2 * j], od = v[2 * j + 1];
          v[2 * j] = ev * cs - od * sn;
          v[2 * j + 1] = ev * sn + od * cs;
        }
      }
    }
    if (e.beta != 0.f) {
      float o[16];
      load16(e.out, idx, o, cnt, PREC_F32);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] += e.beta * o[j];
    }
    if (e.residual) {
      float o[16];
      load16(e.residual, (int64_t)r * e.ldr + n0, o, cnt, PREC_F32);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] += o[j];
    }
    store16(e.out, idx, v, cnt, e.out_prec);
  } else if (e.kind == EPI_ATOMIC) {
    float* p = reinterpret_cast<float*>(e.out) + (int64_t)r * e.ldo + n0;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < cnt) red_add_f32(p + j, e.alpha * v[j]);
  } else if (e.kind == EPI_SWIGLU_BWD_CACHED) {
    // acc = d_act; aux holds gate (col n) and up (col offaux + n).
    float g[16], u[16], dg[16], du[16];
    load16(e.aux, (int64_t)r * e.ldaux + n0, g, cnt, e.act_prec);
    load16(e.aux, (int64_t)r * e.ldaux + e.offaux + n0, u, cnt, e.act_prec);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float sg = silu_f(g[j]);
      du[j] = v[j] * sg;                       // d_up = d_act * silu(gate)
      dg[j] = (v[j] * u[j]) * silu_grad_f(g[j]);  // d_gate = d_act * up * silu'(gate)
    }
    store16(e.out2, (int64_t)r * e.ldo2 + n0, dg, cnt, e.act_prec);
    store16(e.out2, (int64_t)r * e.ldo2 + e.off2 + n0, du, cnt, e.act_prec);
  }
}

// Paired epilogue: g = acc of B row n, u = acc of B row n + pair_off.
__device__ __forceinline__ void epi_apply_pair(const Epilogue& e, int r, int n0, int cnt, float* g, float* u) {
  float a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = silu_f(g[j]) * u[j];  // model.py:216
  if (e.kind == EPI_SWIGLU_FWD) {
    if (e.out) store16(e.out, (int64_t)r * e.ldo + n0, a, cnt, e.act_prec);
    if (e.out2) {
      store16(e.out2, (int64_t)r * e.ldo2 + n0, g, cnt, e.act_prec);
      store16(e.out2, (int64_t)r * e.ldo2 + e.off2 + n0, u, cnt, e.act_prec);
    }
  } else if (e.kind == EPI_SWIGLU_BWD_RECOMP) {
    float d[16], dg[16], du[16];
    load16(e.aux, (int64_t)r * e.ldaux + n0, d, cnt, e.act_prec);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      du[j] = d[j] * silu_f(g[j]);                 // model.py:252
      dg[j] = (d[j] * u[j]) * silu_grad_f(g[j]);   // model.py:251,253
    }
    if (e.out) store16(e.out, (int64_t)r * e.ldo + n0, a, cnt, e.act_prec);
    store16(e.out2, (int64_t)r * e.ldo2 + n0, dg, cnt, e.act_prec);
    store16(e.out2, (int64_t)r * e.ldo2 + e.off2 + n0, du, cnt, e.act_prec);
  }
}

__device__ __forceinline__ void decode_tile(const GemmDev& p, int t, int& mt, int& nt, int& ks) {
  mt = t % p.tiles_m;
  int rest = t / p.tiles_m;
  nt = rest % p.tiles_n;
  ks = rest / p.tiles_n;
}
// Cluster tile t (pairs of M tiles sharing one B tile) -> this CTA's tile and group.
__device__ __forceinline__ void decode_tile_cl(const GemmDev& p, int t, int crank, int cl, int& mt, int& nt,
                                               int& ks, int& grp) {
  grp = t / p.split_tiles;
  t -= grp * p.split_tiles;
  int mp;
  if (p.n_fast) {  // consecutive tiles share one A row block (read from HBM once, L2 hits for the rest)
    nt = t % p.tiles_n;
    const int rest = t / p.tiles_n;
    mp = rest % p.tiles_m_cl;
    ks = rest / p.tiles_m_cl;
  } else {         // consecutive tiles share one B tile
    mp = t % p.tiles_m_cl;
    const int rest = t / p.tiles_m_cl;
    nt = rest % p.tiles_n;
    ks = rest / p.tiles_n;
  }
  mt = mp * cl + crank;
}

// ---------------------------------------------------------------------------
// tcgen05 / TMA / mbarrier primitives (inline PTX, sm_100a)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// CTA-pair (cta_group::2) primitives: one MMA over M = 256 rows, A rows and
// half of B staged in each CTA of the pair.
__device__ __forceinline__ void tc_mma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// TMA into this CTA's smem, completion bytes counted on the LEADER's barrier
// (the cta-rank bit of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 "version 1" format.
// K-major: 8-row groups 1024 B apart (SBO), rows of 128 B; MN-major: 8-K-row
// groups 1024 B apart (SBO), 64-element MN chunks `lbo` bytes apart.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// ---------------------------------------------------------------------------
// tcgen05 kernel
// ---------------------------------------------------------------------------

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;
constexpr int TC_EPI_WARPS = 8;                        // 2 per TMEM lane quadrant
constexpr int TC_THREADS = 128 + 32 * TC_EPI_WARPS;    // warps 0-3: TMA, MMA, TMEM alloc, spare
constexpr int TC_STAGE_OUT = 4096;                     // per-epilogue-warp staging: 32 rows x 128 B

// CL template value of a CTA pair running ONE cta_group::2 MMA per k-step:
// M = 256 rows per pair tile (128 per CTA, each in its own TMEM), each CTA
// stages its own A rows and HALF of the B tile, so a CTA's operand traffic
// through shared memory per flop drops by a quarter at BN = 256 (A 16 KB +
// B 16 KB per 64-deep k-block instead of 16 + 32 KB) and the ring holds six
// stages instead of four.
constexpr int CL_2SM = 3;

template <int BN, bool TWO = false>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = (TWO ? BN / 2 : BN) * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = TWO ? 6 : ((BN == 256) ? 4 : (BN == 128 ? 6 : 8));
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int EPI_BYTES = TC_EPI_WARPS * TC_STAGE_OUT;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/;
};

// Output slot s of an epilogue: 0 = `out`, 1 = `out2`, 2 = `out2 + off2`.
struct TcOut {
  int used[3];
  int prec[3];
  int reduce[3];  // 1: TMA reduce-add (accumulate / split-K), 0: TMA store
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1, int reduce) {
  if (reduce)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  tmem_ld16(taddr, v);
  tmem_ld16(taddr + 16, v + 16);
}

// Epilogue staging: each epilogue warp owns a 4 KB box holding its 32 rows x
// one 32-column chunk in the TMA swizzle layout of the store map (fp32: 128-B
// rows, SWIZZLE_128B; bf16: 64-B rows, SWIZZLE_64B), written in 16-column
// halves; lane 0 issues the bulk store / reduce-add. (A double-buffered box
// per warp measured 2-4% slower: the extra outstanding bulk stores cost more
// than the read-completion wait they hide.)
__device__ __forceinline__ void stage_wait(int lane) {  // previous store has read the box
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
}
__device__ __forceinline__ void stage_write16(uint8_t* stg, const float* v, int prec, int half, int lane) {
  if (prec == PREC_F32) {
    uint8_t* row = stg + lane * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int u = half * 4 + q;
      *reinterpret_cast<float4*>(row + ((u ^ (lane & 7)) << 4)) =
          make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  } else {
    uint8_t* row = stg + lane * 64;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int u = half * 2 + q;
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * j], v[8 * q + 2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      *reinterpret_cast<uint4*>(row + ((u ^ ((lane >> 1) & 3)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}
__device__ __forceinline__ void stage_commit(uint8_t* stg, const CUtensorMap* map, int reduce, int c0, int r0,
                                             int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) tma_store_2d(map, stg, c0, r0, reduce);
}

__device__ __forceinline__ void stage_store32(uint8_t* stg, const CUtensorMap* map, const float* v, int prec,
                                              int reduce, int c0, int r0, int lane) {
  stage_wait(lane);
  stage_write16(stg, v, prec, 0, lane);
  stage_write16(stg, v + 16, prec, 1, lane);
  stage_commit(stg, map, reduce, c0, r0, lane);
}

// bf16 32-column box (32 rows x 64 B = 2 KB) through one of the two halves
// of the warp's 4 KB staging buffer: only the store before last must have
// read its half.
__device__ __forceinline__ void stage_store32_db(uint8_t* stg, int& sb, const CUtensorMap* map, const float* v,
                                                 int c0, int r0, int lane) {
  uint8_t* box = stg + sb * 2048;
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
  stage_write16(box, v, PREC_BF16, 0, lane);
  stage_write16(box, v + 16, PREC_BF16, 1, lane);
  stage_commit(box, map, 0, c0, r0, lane);
  sb ^= 1;
}

// Epilogue math for output slot `slot` on 16 consecutive output columns n0..
// of row r (tcgen05 path): 0 = out / act, 1 = gate or d_gate, 2 = up or d_up.
__device__ __forceinline__ void epi_slot16(const Epilogue& e, int slot, int r, int n0, int cnt, bool row_ok,
                                           const float* g, const float* u, float* o, bool res_in_smem = false,
                                           const float* rope_pre = nullptr) {
  if (e.kind == EPI_STORE || e.kind == EPI_ATOMIC) {
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = g[j] * e.alpha;
    if (e.rope_cos && n0 < e.rope_cols && row_ok) {
      if (rope_pre && n0 + 16 <= e.rope_cols) {  // this row's (cos, sin) of these 8 frequencies, per tile
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float cs = rope_pre[j], sn = rope_pre[16 + j];
          const float ev = o[2 * j], od = o[2 * j + 1];
          o[2 * j] = ev * cs - od * sn;
          o[2 * j + 1] = ev * sn + od * cs;
        }
        return;
      }
      const int pos = r % e.rope_T, half = e.rope_hd >> 1;
      if ((e.rope_hd & 15) == 0 && n0 + 16 <= e.rope_cols) {
        // The 16-column span lies inside one head: 8 consecutive frequencies.
        // The angles are computed, not looked up — the cos/sin table does
        // not stay L1-resident next to a 224 KB operand ring, and its L2
        // latency was serialising the epilogue. theta_j = 10000^(-2j/hd)
        // (model.py:274); |angle error| <= ~6e-5 rad after Cody-Waite
        // reduction to [-pi, pi], far below the bf16 rounding of q/k.
        if (rope_pre) {  // this row's (cos, sin) of these 8 frequencies, computed once per tile
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float cs = rope_pre[j], sn = rope_pre[16 + j];
            const float ev = o[2 * j], od = o[2 * j + 1];
            o[2 * j] = ev * cs - od * sn;
            o[2 * j + 1] = ev * sn + od * cs;
          }
          return;
        }
        const int j0 = (n0 % e.rope_hd) >> 1;
        const float fpos = (float)pos;
        float th[8];  // 128-B table: stays L1-resident (the cos/sin table did not)
        *reinterpret_cast<float4*>(th) = __ldg(reinterpret_cast<const float4*>(e.rope_theta + j0));
        *reinterpret_cast<float4*>(th + 4) = __ldg(reinterpret_cast<const float4*>(e.rope_theta + j0 + 4));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float ang = fpos * th[j];
          const float kq = rintf(ang * 0.15915494309189535f);
          float rr = fmaf(-kq, 6.28318548202514648f, ang);
          rr = fmaf(kq, 1.7484556e-7f, rr);
          float sn, cs;
          __sincosf(rr, &sn, &cs);
          const float ev = o[2 * j], od = o[2 * j + 1];
          o[2 * j] = ev * cs - od * sn;
          o[2 * j + 1] = ev * sn + od * cs;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = n0 + 2 * j;
          if (c < e.rope_cols) {
            const int pi = pos * half + ((c % e.rope_hd) >> 1);
            const float cs = __ldg(e.rope_cos + pi), sn = __ldg(e.rope_sin + pi);
            const float ev = o[2 * j], od = o[2 * j + 1];
            o[2 * j] = ev * cs - od * sn;
            o[2 * j + 1] = ev * sn + od * cs;
          }
        }
      }
    }
    if (e.residual && !res_in_smem && row_ok && cnt > 0) {
      float t[16];
      load16(e.residual, (int64_t)r * e.ldr + n0, t, min(cnt, 16), PREC_F32);
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] += t[j];
    }
    return;
  }
  if (e.kind == EPI_SWIGLU_BWD_CACHED) {  // g = d_act; aux = cached gate | up
    float gt[16], up[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) { gt[j] = 0.f; up[j] = 0.f; }
    if (row_ok && cnt > 0) {
      load16(e.aux, (int64_t)r * e.ldaux + n0, gt, min(cnt, 16), e.act_prec);
      if (slot == 1) load16(e.aux, (int64_t)r * e.ldaux + e.offaux + n0, up, min(cnt, 16), e.act_prec);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      o[j] = slot == 2 ? g[j] * silu_f(gt[j])                    // d_up   (model.py:252)
                       : (g[j] * up[j]) * silu_grad_f(gt[j]);    // d_gate (model.py:251,253)
    return;
  }
  // paired SwiGLU kinds: g = gate, u = up
  if (slot == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = silu_f(g[j]) * u[j];  // act (model.py:216)
    return;
  }
  if (e.kind == EPI_SWIGLU_FWD) {
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = slot == 1 ? g[j] : u[j];
    return;
  }
  float d[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) d[j] = 0.f;
  if (row_ok && cnt > 0) load16(e.aux, (int64_t)r * e.ldaux + n0, d, min(cnt, 16), e.act_prec);
#pragma unroll
  for (int j = 0; j < 16; ++j)
    o[j] = slot == 2 ? d[j] * silu_f(g[j]) : (d[j] * u[j]) * silu_grad_f(g[j]);
}

template <int BN, bool A_KMAJOR, bool B_KMAJOR, int CL, int NG, bool ROPE = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ TcMaps<NG> mp, GemmDev p, TcOut outs) {
  constexpr bool TWO = CL == CL_2SM;  // CTA pair, cta_group::2 MMA issued by the leader
  constexpr int CLN = TWO ? 2 : CL;   // CTAs per cluster
  static_assert(!TWO || BN == 256, "the pair mode stages B halves of 128 rows");
  using C = TcCfg<BN, TWO>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sE = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(tmem_holder + 2);  // per-epilogue-warp residual-box barriers (x2)
  // fp32 residual epilogues (x + f(x)) with BN >= 128 run the operand ring one
  // stage short and give each epilogue warp a second residual box in the
  // freed stage, so the residual of a chunk is TMA-prefetched while the
  // previous chunk (or the tile's mainloop) is in flight
  const bool res_pf = BN >= 128 && NG == 1 && p.epi.kind == EPI_STORE && p.epi.residual != nullptr &&
                      outs.used[0] && outs.prec[0] == PREC_F32 && !p.paired && !outs.used[1] && !outs.used[2] &&
                      p.kb_per_split <= 12;  // short K only: a long mainloop needs the full ring (measured:
                                             // o_residual K=512 33 -> 29 us, down_residual K=1376 37 -> 39 us)
  const int nst = res_pf ? C::STAGES - 1 : C::STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TWO ? 1 : CL);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], TWO ? 2 * TC_EPI_WARPS : 32 * TC_EPI_WARPS);  // pair: one arrive per warp of both CTAs
    }
    for (int w = 0; w < 2 * TC_EPI_WARPS; ++w) mbar_init(&rbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mp.a[0])) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mp.b[0])) : "memory");
  }
  const int crank = CLN > 1 ? (int)cluster_ctarank() : 0;
  const int cl_id = blockIdx.x / CLN, n_cl = gridDim.x / CLN;
  constexpr uint16_t kMask = (uint16_t)((1u << CLN) - 1);
  if (warp == 2) {
    if constexpr (TWO) {  // the pair's TMEM, allocated by the same warp of both CTAs
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CLN > 1) cluster_sync_all();  // peer barriers initialised before any multicast lands
  griddep_wait();  // predecessor outputs are visible from here on
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cl_id; t < p.num_tiles_cl; t += n_cl) {
        int mt, nt, ks, grp;
        decode_tile_cl(p, t, crank, CLN, mt, nt, ks, grp);
        const CUtensorMap* tmA = &mp.a[NG > 1 ? grp : 0];
        const CUtensorMap* tmB = &mp.b[NG > 1 ? grp : 0];
        // once per tile: this single thread issues every TMA of the k-loop, so
        // nothing per k-block may cost more than a few instructions
        const int boff = p.b_diag_off ? (int)((mt / p.b_diag_div) * p.b_diag_off) : 0;
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.kblocks);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          const int k0 = kb * TC_BK;
          if constexpr (TWO) {
            // both CTAs' bytes complete on the LEADER's barrier (its MMA reads both)
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            if (A_KMAJOR) {
              tma_load_2d_2sm(a, tmA, &full[stage], k0, mt * TC_BM);
            } else {
              tma_load_2d_2sm(a, tmA, &full[stage], mt * TC_BM, k0);
              tma_load_2d_2sm(a + 8192, tmA, &full[stage], mt * TC_BM + 64, k0);
            }
            if (B_KMAJOR) {  // rows [crank * BN/2, +BN/2) of the tile (paired: CTA 0 gate, CTA 1 up)
              const int row = p.paired ? (crank == 0 ? nt * (BN / 2) : nt * (BN / 2) + (int)p.pair_off)
                                       : nt * BN + crank * (BN / 2);
              tma_load_2d_2sm(b, tmB, &full[stage], k0, row);
            } else {         // 64-column chunks [crank * NCH/2, +NCH/2) of the tile
              constexpr int NCH = BN / 64;
#pragma unroll
              for (int c = 0; c < NCH / 2; ++c) {
                const int cc = crank * (NCH / 2) + c;
                const int col = !p.paired ? nt * BN + cc * 64
                                          : (cc < NCH / 2 ? nt * (BN / 2) + cc * 64
                                                          : nt * (BN / 2) + (int)p.pair_off + (cc - NCH / 2) * 64);
                tma_load_2d_2sm(b + c * 8192, tmB, &full[stage], col, k0);
              }
            }
            if (++stage == nst) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          if (A_KMAJOR) {
            tma_load_2d(a, tmA, &full[stage], k0, mt * TC_BM);
          } else {
            tma_load_2d(a, tmA, &full[stage], mt * TC_BM, k0);
            tma_load_2d(a + 8192, tmA, &full[stage], mt * TC_BM + 64, k0);
          }
          if (B_KMAJOR) {
            if (CL > 1) {  // this CTA's half of the B tile, multicast to the pair
              const int row = p.paired ? (crank == 0 ? nt * (BN / 2) : nt * (BN / 2) + (int)p.pair_off)
                                       : nt * BN + crank * (BN / 2);
              tma_load_2d_mc(b + crank * (BN / 2) * 128, tmB, &full[stage], k0, row, kMask);
            } else if (!p.paired && p.b_split) {
              tma_load_2d(b, tmB, &full[stage], k0, nt * BN + boff);
              tma_load_2d(b + (BN / 2) * 128, tmB, &full[stage], k0, nt * BN + boff + BN / 2);
            } else if (!p.paired) {
              tma_load_2d(b, tmB, &full[stage], k0, nt * BN + boff);
            } else {
              tma_load_2d(b, tmB, &full[stage], k0, nt * (BN / 2));
              tma_load_2d(b + (BN / 2) * 128, tmB, &full[stage], k0, nt * (BN / 2) + (int)p.pair_off);
            }
          } else {
            constexpr int NCH = BN / 64;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              if (CL > 1 && c / (NCH / CL) != crank) continue;
              int col;
              if (!p.paired)
                col = nt * BN + c * 64 + boff;
              else
                col = (c < NCH / 2) ? nt * (BN / 2) + c * 64 : nt * (BN / 2) + (int)p.pair_off + (c - NCH / 2) * 64;
              if (CL > 1)
                tma_load_2d_mc(b + c * 8192, tmB, &full[stage], col, k0, kMask);
              else
                tma_load_2d(b + c * 8192, tmB, &full[stage], col, k0);
            }
          }
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && (!TWO || crank == 0)) {
      // ===== MMA issuer (single thread; the pair's leader in TWO mode) =====
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_KMAJOR ? 0u : 1u) << 15) |
                                 ((B_KMAJOR ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)((TWO ? 2 * TC_BM : TC_BM) >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cl_id; t < p.num_tiles_cl; t += n_cl) {
        int mt, nt, ks, grp;
        decode_tile_cl(p, t, crank, CLN, mt, nt, ks, grp);
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.kblocks);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint64_t ad = A_KMAJOR ? make_sdesc(a_addr + k * 32, 16, 1024) : make_sdesc(a_addr + k * 2048, 8192, 1024);
            const uint64_t bd = B_KMAJOR ? make_sdesc(b_addr + k * 32, 16, 1024) : make_sdesc(b_addr + k * 2048, 8192, 1024);
            if constexpr (TWO)
              tc_mma_bf16_2sm(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else
              tc_mma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if (TWO)
            tc_commit_2sm_mc(&empty[stage], 0x3);  // frees the stage in both CTAs
          else if (CL > 1)
            tc_commit_mc(&empty[stage], kMask);  // the stage holds the peer's multicast half too
          else
            tc_commit(&empty[stage]);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        if (TWO)
          tc_commit_2sm_mc(&tfull[acc], 0x3);  // both CTAs' accumulators are ready
        else
          tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===== Epilogue warps: TMEM -> registers -> fused math -> smem -> TMA =====
    const int ew = warp - 4;
    const int quad = ew & 3;        // TMEM lane quadrant == warp % 4
    const int half = ew >> 2;       // which half of the column chunks
    uint8_t* stg = sE + ew * TC_STAGE_OUT;
    // fp32 residual (x + f(x) epilogues): the 32x32 residual box is TMA-loaded
    // into the staging box (same SW128 layout as the fp32 store), added in
    // place, and stored — no per-lane strided global reads in the epilogue
    // (measured: prefetching each lane's row segment into registers one chunk
    // ahead was 13% slower than this)
    const bool res_tma = p.epi.kind == EPI_STORE && p.epi.residual != nullptr && outs.used[0] &&
                         outs.prec[0] == PREC_F32 && !p.paired;
    uint32_t rphase = 0;
    uint32_t pf_phase[2] = {0u, 0u};
    // res_pf: this warp's two residual boxes (the staging box and one in the
    // spare operand stage) and their barriers rbar[ew], rbar[8 + ew]
    uint8_t* pf_box[2] = {stg, ew < 4 ? sA + (C::STAGES - 1) * C::A_BYTES + ew * TC_STAGE_OUT
                                      : sB + (C::STAGES - 1) * C::B_BYTES + (ew - 4) * TC_STAGE_OUT};
    int acc = 0;
    uint32_t acc_phase = 0;
    constexpr int NCHUNK_PLAIN = BN / 32;
    constexpr int NCHUNK_PAIR = BN / 64;
    for (int t = cl_id; t < p.num_tiles_cl; t += n_cl) {
      int mt, nt, ks, grp;
      decode_tile_cl(p, t, crank, CLN, mt, nt, ks, grp);
      const CUtensorMap* tmO0 = &mp.o0[NG > 1 ? grp : 0];
      const int r0 = mt * TC_BM + quad * 32;
      const int nchunks = p.paired ? NCHUNK_PAIR : NCHUNK_PLAIN;
      const int cbase = p.paired ? nt * (BN / 2) : nt * BN;
      if (res_pf) {  // this tile's first two residual boxes, before its accumulator is even ready
        stage_wait(lane);  // every earlier store has read its box
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int cj = half + 2 * j;
            if (cj < nchunks && cbase + cj * 32 < p.N) {
              mbar_expect_tx(&rbar[8 * j + ew], 32 * 32 * 4);
              tma_load_2d(pf_box[j], &mp.r, &rbar[8 * j + ew], cbase + cj * 32, r0);
            }
          }
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = r0 + lane;
      const bool row_ok = row < p.M;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      bool released = false;
      int pf_i = 0;  // this warp's chunk index within the tile
      // hd = 64 RoPE: every chunk this warp handles (c = half + 2k, 32 columns)
      // uses the same 16 frequencies j = 16*half + i, so the row's (cos, sin)
      // are computed once per tile instead of once per head
      // (ROPE instantiation only: the 32 extra registers would spill elsewhere)
      float rcs[ROPE ? 32 : 1];
      const bool rope_pre = ROPE && p.epi.rope_cos && p.epi.rope_hd == 64 && (BN % 64) == 0 && !p.paired &&
                            cbase < p.epi.rope_cols && row_ok;
      if constexpr (ROPE) if (rope_pre) {
        const float fpos = (float)(row % p.epi.rope_T);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float ang = fpos * __ldg(p.epi.rope_theta + half * 16 + i);
          const float kq = rintf(ang * 0.15915494309189535f);
          float rr = fmaf(-kq, 6.28318548202514648f, ang);
          rr = fmaf(kq, 1.7484556e-7f, rr);
          __sincosf(rr, &rcs[16 + i], &rcs[i]);
        }
      }
#pragma unroll 1
      for (int c = half; c < nchunks; c += 2, ++pf_i) {
        const int n0 = cbase + c * 32;
        if (n0 >= p.N) continue;  // warp-uniform
        uint8_t* rbox = res_pf ? pf_box[pf_i & 1] : stg;
        if (res_tma && !res_pf) {
          stage_wait(lane);  // the previous store has read the box
          if (lane == 0) {
            mbar_expect_tx(&rbar[ew], 32 * 32 * 4);
            tma_load_2d(stg, &mp.r, &rbar[ew], n0, r0);
          }
        }
        // all TMEM columns of the chunk in flight before one wait::ld
        float g[32], u[32];
        tmem_ld16_nowait(taddr + c * 32, g);
        tmem_ld16_nowait(taddr + c * 32 + 16, g + 16);
        if (p.paired) {
          tmem_ld16_nowait(taddr + BN / 2 + c * 32, u);
          tmem_ld16_nowait(taddr + BN / 2 + c * 32 + 16, u + 16);
        }
        tmem_wait_ld();
        if (c + 2 >= nchunks || cbase + (c + 2) * 32 >= p.N) {
          // this warp's last chunk is in registers: hand the accumulator
          // back to the MMA warp before the math and stores
          tc_fence_before();
          if constexpr (TWO) {
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
          } else {
            mbar_arrive(&tempty[acc]);
          }
          released = true;
        }
#pragma unroll
        for (int slot = 0; slot < 3; ++slot) {  // unrolled: outs.* indexed statically (no local-memory copy)
          if (!outs.used[slot]) continue;
          const bool rs = slot == 0 && res_tma;
          uint8_t* box = rs ? rbox : stg;
          if (rs && res_pf) {
            mbar_wait(&rbar[8 * (pf_i & 1) + ew], pf_phase[pf_i & 1]);
            pf_phase[pf_i & 1] ^= 1u;
          } else if (rs) {
            mbar_wait(&rbar[ew], rphase);
            rphase ^= 1;
          } else {
            stage_wait(lane);
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float o[16];
            const int n0h = n0 + hh * 16;
            const float* rp = nullptr;
            if constexpr (ROPE) rp = (rope_pre && n0h + 16 <= p.epi.rope_cols) ? rcs + hh * 8 : nullptr;
            epi_slot16(p.epi, slot, row, n0h, p.N - n0h, row_ok, g + hh * 16, u + hh * 16, o, rs, rp);
            if (rs) {  // + residual from the staging box (this lane's row, 16 columns)
              const uint8_t* rrow = box + lane * 128;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4 r4 = *reinterpret_cast<const float4*>(rrow + (((hh * 4 + q) ^ (lane & 7)) << 4));
                o[4 * q] += r4.x; o[4 * q + 1] += r4.y; o[4 * q + 2] += r4.z; o[4 * q + 3] += r4.w;
              }
            }
            stage_write16(box, o, outs.prec[slot], hh, lane);
          }
          stage_commit(box, slot == 0 ? tmO0 : (slot == 1 ? &mp.o1 : &mp.o2), outs.reduce[slot], n0, r0, lane);
        }
        if (res_pf) {  // refill this box with the residual of the warp's chunk after next
          const int cn = c + 4;
          if (cn < nchunks && cbase + cn * 32 < p.N) {
            stage_wait(lane);  // the store just issued has read the box
            if (lane == 0) {
              mbar_expect_tx(&rbar[8 * (pf_i & 1) + ew], 32 * 32 * 4);
              tma_load_2d(rbox, &mp.r, &rbar[8 * (pf_i & 1) + ew], cbase + cn * 32, r0);
            }
          }
        }
      }
      if (!released) {
        tc_fence_before();
        if constexpr (TWO) {
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
        } else {
          mbar_arrive(&tempty[acc]);
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (CLN > 1) cluster_sync_all();  // no CTA leaves while its peer may still multicast into it / signal it
  if (warp == 2) {
    tc_fence_after();
    if constexpr (TWO)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
  }
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (fp32 parity mode; also accepts bf16 operands).
// 64x64 accumulator tile, BK=16, 256 threads, 4x4 per thread.
// ---------------------------------------------------------------------------

struct SimtOperand {
  const void* ptr;
  int64_t ld;
  int kmajor;
  int prec;
};

__global__ void __launch_bounds__(256) gemm_simt_kernel(SimtOperand A, SimtOperand B, GemmDev p) {
  griddep_wait();
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  __shared__ float Cs[64][65];
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  const int mt = blockIdx.x, nt = blockIdx.y, ks = blockIdx.z;
  const int m0 = mt * 64;
  const int kb0 = ks * p.kb_per_split;  // k-blocks of 16 here
  const int kb1 = min(kb0 + p.kb_per_split, p.kblocks);
  float acc[4][4] = {};
  for (int kb = kb0; kb < kb1; ++kb) {
    const int k0 = kb * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      int row, kk;
      if (A.kmajor) { row = e / 16; kk = e % 16; } else { kk = e / 64; row = e % 64; }
      const int gm = m0 + row, gk = k0 + kk;
      float va = 0.f;
      if (gm < p.M && gk < p.K)
        va = load_as_f32(A.ptr, A.kmajor ? (int64_t)gm * A.ld + gk : (int64_t)gk * A.ld + gm, A.prec);
      As[kk][row] = va;
      if (B.kmajor) { row = e / 16; kk = e % 16; } else { kk = e / 64; row = e % 64; }
      int64_t gn;
      bool ok;
      if (!p.paired) {
        gn = (int64_t)nt * 64 + row;
        ok = gn < p.N;
      } else {
        const int pc = nt * 32 + (row & 31);
        ok = pc < p.N;
        gn = pc + ((row >= 32) ? p.pair_off : 0);
      }
      const int gk2 = k0 + kk;
      float vb = 0.f;
      if (ok && gk2 < p.K)
        vb = load_as_f32(B.ptr, B.kmajor ? gn * B.ld + gk2 : (int64_t)gk2 * B.ld + gn, B.prec);
      Bs[kk][row] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Cs[ty * 4 + i][tx * 4 + j] = acc[i][j];
  __syncthreads();
  if (!p.paired) {
    const int row = tid / 4, ch = tid % 4;
    const int gr = m0 + row, n0 = nt * 64 + ch * 16;
    if (gr < p.M && n0 < p.N) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = Cs[row][ch * 16 + j];
      epi_apply(p.epi, gr, n0, min(16, p.N - n0), v);
    }
  } else if (tid < 128) {
    const int row = tid / 2, ch = tid % 2;
    const int gr = m0 + row, n0 = nt * 32 + ch * 16;
    if (gr < p.M && n0 < p.N) {
      float g[16], u[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        g[j] = Cs[row][ch * 16 + j];
        u[j] = Cs[row][32 + ch * 16 + j];
      }
      epi_apply_pair(p.epi, gr, n0, min(16, p.N - n0), g, u);
    }
  }
}

}  // namespace mecefo
