// Host side of the MeCeFO engine: GEMM dispatch (tcgen05 bf16 / fp32 SIMT),
// TMA descriptor cache, block-level orchestration of the lean and exact
// steps, and the C-ABI declared in include/mecefo.h.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>
#include <utility>

#include "../../include/mecefo.h"
#include "host.h"
#include "attention.cuh"
#include "attention_tc.cuh"
#include "attention_bwd_tc.cuh"
#include "gemm_dual.cuh"
#include "gemm_norm.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "subspace.cuh"
#include "ce.cuh"

using namespace mecefo;
using namespace mecefo_host;

// ---------------------------------------------------------------------------
// errors, launch counter, launch profiler (shared with refresh.cu via host.h)
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

// Optional launch profiler: CUDA events around each kernel (or fused
// kernel group) tagged with its algorithmic FLOPs and HBM bytes. Enabled by
// bench.py over its timed region; off by default (zero overhead).
struct ProfRec {
  const char* tag;
  cudaEvent_t a, b;
  double flops, bytes;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t ev() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[next++];
  }
};
Profiler g_prof;
std::mutex g_prof_mu;
}  // namespace

namespace mecefo_host {

int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(MECEFO_ERR_CUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
  return MECEFO_OK;
}

int64_t prof_begin(const char* tag, double flops, double bytes, cudaStream_t s) {
  if (!g_prof.on) return -1;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.recs.push_back(ProfRec{tag, g_prof.ev(), g_prof.ev(), flops, bytes});
  const int64_t idx = (int64_t)g_prof.recs.size() - 1;
  cudaEventRecord(g_prof.recs[idx].a, s);
  return idx;
}

void prof_end(int64_t idx, cudaStream_t s) {
  if (idx < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (idx < (int64_t)g_prof.recs.size()) cudaEventRecord(g_prof.recs[idx].b, s);
}

bool pdl_enabled() {
  static const bool on = getenv("MECEFO_NO_PDL") == nullptr;
  return on;
}

// Dynamic shared memory opt-in per (kernel, device): a process that drives
// several GPUs configures each device's copy of the kernel once.
int ensure_smem(const void* kern, int bytes) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({kern, dev});
  if (it != done.end() && it->second >= bytes) return MECEFO_OK;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[{kern, dev}] = bytes;
  return MECEFO_OK;
}

}  // namespace mecefo_host

namespace {

// Bump allocator over the caller's workspace.
struct Ws {
  uint8_t* base;
  size_t cap, used = 0;
  Ws(void* p, size_t c) : base(reinterpret_cast<uint8_t*>(p)), cap(c) {}
  int take(size_t bytes, void** out) {
    size_t off = (used + 255) & ~size_t(255);
    if (off + bytes > cap)
      return set_err(MECEFO_ERR_CONTRACT, "workspace too small: need %zu more bytes (cap %zu)", off + bytes - cap,
                     cap);
    *out = base + off;
    used = off + bytes;
    return MECEFO_OK;
  }
};

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct TmKey {
  const void* p;
  int64_t inner, outer, ld;
  int box0, box1;
  bool operator==(const TmKey& o) const {
    return p == o.p && inner == o.inner && outer == o.outer && ld == o.ld && box0 == o.box0 && box1 == o.box1;
  }
};
struct TmHash {
  size_t operator()(const TmKey& k) const {
    size_t h = std::hash<const void*>()(k.p);
    auto mix = [&](int64_t v) { h ^= std::hash<int64_t>()(v) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); };
    mix(k.inner); mix(k.outer); mix(k.ld); mix(k.box0); mix(k.box1);
    return h;
  }
};

}  // namespace

struct mecefo_engine {
  mecefo_dims d;
  int prec;
  int ps;  // bytes per compute-precision element
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  // device status word (bits MECEFO_STATUS_*): bad token / bad target /
  // non-finite gradient, set by the kernels, read by the host at iteration
  // boundaries (model.py:463 IndexError, optim.py:55-57 _check_grad)
  int* status = nullptr;
  std::mutex mu;
  std::unordered_map<TmKey, CUtensorMap, TmHash> tmaps;
};

namespace {

int make_tmap(mecefo_engine* e, CUtensorMap* out, const void* p, int64_t inner, int64_t outer, int64_t ld, int box0,
              int box1, int fp32 = 0, int swz = 128) {
  TmKey key{p, inner, outer, ld, box0, box1 + (fp32 << 20) + (swz << 21)};
  {
    std::lock_guard<std::mutex> lk(e->mu);
    auto it = e->tmaps.find(key);
    if (it != e->tmaps.end()) { *out = it->second; return MECEFO_OK; }
  }
  auto enc = get_encode();
  if (!enc) return set_err(MECEFO_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  if ((reinterpret_cast<uintptr_t>(p) & 15) != 0)
    return set_err(MECEFO_ERR_CONTRACT, "bf16 GEMM operand %p is not 16-byte aligned", p);
  const int esz = fp32 ? 4 : 2;
  if ((ld * esz) % 16 != 0)
    return set_err(MECEFO_ERR_CONTRACT, "TMA operand leading dimension %lld x %d B is not a multiple of 16 bytes",
                   (long long)ld, esz);
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esz)};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(out, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(p), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(MECEFO_ERR_CONTRACT, "cuTensorMapEncodeTiled failed (%d) for %lldx%lld ld %lld box %dx%d", (int)r,
                   (long long)inner, (long long)outer, (long long)ld, box0, box1);
  std::lock_guard<std::mutex> lk(e->mu);
  if (e->tmaps.size() > 4096) e->tmaps.clear();
  e->tmaps[key] = *out;
  return MECEFO_OK;
}

struct Op {
  const void* p;
  int64_t ld;
  bool km;
};

struct GemmCall {
  int64_t M = 0, N = 0, K = 0;
  Op a{}, b{};
  bool paired = false;
  int64_t pair_off = 0;
  Epilogue epi{};
  int split = 1;
  const char* tag = "gemm";
  int force_bn = 0;  // tcgen05 tile width override (split-K accumulate GEMMs)
  // block-diagonal batching: M tile mt reads B columns shifted by
  // (mt / b_diag_div) * b_diag_off (independent products sharing one launch;
  // each diagonal block spans b_diag_div whole 128-row tiles)
  int64_t b_diag_off = 0;
  int b_diag_div = 1;
  // grouped launch: `groups` products of this shape, operand/output base
  // pointers per group (ga/gb/go override a.p/b.p/epi.out); same strides
  int groups = 1;
  const void* ga[8] = {};
  const void* gb[8] = {};
  void* go[8] = {};
};
constexpr int kMaxGroups = 8;

Epilogue epi_store(void* out, int64_t ldo, int out_prec, float alpha = 1.f, float beta = 0.f,
                   const float* residual = nullptr, int64_t ldr = 0) {
  Epilogue e{};
  e.kind = EPI_STORE;
  e.out = out; e.ldo = ldo; e.out_prec = out_prec; e.alpha = alpha; e.beta = beta;
  e.residual = residual; e.ldr = ldr;
  return e;
}

template <int BN, bool AK, bool BKM, int CL, int NG, bool ROPE = false>
int launch_tc(mecefo_engine* e, const GemmCall& g, cudaStream_t s) {
  constexpr int CLN = CL == CL_2SM ? 2 : CL;  // CTAs per cluster
  using C = TcCfg<BN, CL == CL_2SM>;
  static_assert(NG == 1 || CL == 1, "grouped launches are single-CTA");
  const int ng = NG > 1 ? g.groups : 1;
  if (ng < 1 || ng > NG) return set_err(MECEFO_ERR_CONSISTENCY, "group count %d outside [1, %d]", ng, NG);
  TcMaps<NG> mp;
  std::memset(&mp, 0, sizeof(mp));
  bool b_split = false;
#ifdef MECEFO_TIMING_KNOBS
  b_split = BN == 256 && BKM && CL == 1 && !g.paired && getenv("MECEFO_B_SPLIT") != nullptr;
#endif
  const int64_t rowsB =
      g.paired ? g.pair_off + g.N : g.N + g.b_diag_off * (((g.M + TC_BM - 1) / TC_BM - 1) / std::max(1, g.b_diag_div));
  for (int q = 0; q < ng; ++q) {
    const void* pa = NG > 1 ? g.ga[q] : g.a.p;
    const void* pb = NG > 1 ? g.gb[q] : g.b.p;
    if (AK) TRY(make_tmap(e, &mp.a[q], pa, g.K, g.M, g.a.ld, 64, TC_BM));
    else TRY(make_tmap(e, &mp.a[q], pa, g.M, g.K, g.a.ld, 64, 64));
    if (BKM) TRY(make_tmap(e, &mp.b[q], pb, g.K, rowsB, g.b.ld, 64, (g.paired || CL > 1 || b_split) ? BN / 2 : BN));
    else TRY(make_tmap(e, &mp.b[q], pb, rowsB, g.K, g.b.ld, 64, 64));
  }
  GemmDev p{};
  p.M = (int)g.M; p.N = (int)g.N; p.K = (int)g.K;
  p.paired = g.paired ? 1 : 0;
  p.pair_off = g.pair_off;
  p.b_diag_off = g.b_diag_off;
  p.b_diag_div = std::max(1, g.b_diag_div);
  p.kblocks = (int)((g.K + TC_BK - 1) / TC_BK);
  int split = std::max(1, std::min(g.split, p.kblocks));
  p.kb_per_split = (p.kblocks + split - 1) / split;
  p.split = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  p.tiles_m = (int)((g.M + TC_BM - 1) / TC_BM);
  const int cols_per_tile = g.paired ? BN / 2 : BN;
  p.tiles_n = (int)((g.N + cols_per_tile - 1) / cols_per_tile);
  p.num_tiles = p.tiles_m * p.tiles_n * p.split * ng;
  p.tiles_m_cl = (p.tiles_m + CLN - 1) / CLN;
  p.split_tiles = p.tiles_m_cl * p.tiles_n * p.split;
  p.num_tiles_cl = p.split_tiles * ng;
  // A-heavy GEMMs with few N tiles (d_h2, the residual GEMMs, head d_xf): N-fastest
  // order so an A row block is streamed from HBM once (measured: d_h2 read
  // 159 MB for a 90 MB A with the M-fastest order)
  p.n_fast = (p.tiles_n >= 2 && p.tiles_n <= 8 && (double)g.M >= 4.0 * (double)g.N * (g.paired ? 2 : 1)) ? 1 : 0;
  p.b_split = b_split ? 1 : 0;
#ifdef MECEFO_TIMING_KNOBS
  if (const char* v = getenv("MECEFO_NFAST_FOR")) {  // "tag=0|1,..."
    const char* hit = g.tag ? strstr(v, g.tag) : nullptr;
    if (hit && hit[strlen(g.tag)] == '=') p.n_fast = atoi(hit + strlen(g.tag) + 1);
  }
#endif
  p.epi = g.epi;
  // output slots -> TMA store / reduce-add maps (32 x 32 boxes, swizzled)
  TcOut outs{};
  const Epilogue& ep = g.epi;
  struct Slot { void* ptr; int64_t ld; int prec; int reduce; };
  Slot slots[3] = {{nullptr, 0, 0, 0}, {nullptr, 0, 0, 0}, {nullptr, 0, 0, 0}};
  const int ps = ep.act_prec == PREC_BF16 ? 2 : 4;
  switch (ep.kind) {
    case EPI_STORE:
      if (ep.beta != 0.f && (ep.beta != 1.f || ep.residual || ep.out_prec != PREC_F32))
        return set_err(MECEFO_ERR_CONTRACT, "tcgen05 epilogue supports beta in {0,1} (fp32 accumulate) only");
      slots[0] = {ep.out, ep.ldo, ep.out_prec, ep.beta != 0.f ? 1 : 0};
      break;
    case EPI_ATOMIC:
      slots[0] = {ep.out, ep.ldo, PREC_F32, 1};
      break;
    case EPI_SWIGLU_FWD:
    case EPI_SWIGLU_BWD_RECOMP:
    case EPI_SWIGLU_BWD_CACHED:
      if (ep.kind != EPI_SWIGLU_BWD_CACHED && ep.out) slots[0] = {ep.out, ep.ldo, ep.act_prec, 0};
      if (ep.out2) {
        slots[1] = {ep.out2, ep.ldo2, ep.act_prec, 0};
        slots[2] = {reinterpret_cast<uint8_t*>(ep.out2) + ep.off2 * ps, ep.ldo2, ep.act_prec, 0};
      }
      break;
    default:
      return set_err(MECEFO_ERR_CONSISTENCY, "unknown epilogue kind %d", ep.kind);
  }
  if (NG > 1 && (slots[1].ptr || slots[2].ptr || ep.residual || ep.rope_cos))
    return set_err(MECEFO_ERR_CONSISTENCY, "grouped launches support plain store / accumulate epilogues only");
  for (int k = 0; k < 3; ++k) {
    if (!slots[k].ptr) continue;
    const int f32 = slots[k].prec == PREC_F32 ? 1 : 0;
    CUtensorMap* dst = k == 0 ? &mp.o0[0] : (k == 1 ? &mp.o1 : &mp.o2);
    for (int q = 0; q < (k == 0 ? ng : 1); ++q)
      TRY(make_tmap(e, dst + q, (k == 0 && NG > 1) ? g.go[q] : slots[k].ptr, g.N, g.M, slots[k].ld, 32, 32, f32,
                    f32 ? 128 : 64));
    outs.used[k] = 1;
    outs.prec[k] = slots[k].prec;
    outs.reduce[k] = slots[k].reduce;
  }
  // fp32 residual boxes (same 32x32 SW128 layout as the fp32 store)
  if (ep.kind == EPI_STORE && ep.residual && outs.used[0] && outs.prec[0] == PREC_F32 && !g.paired)
    TRY(make_tmap(e, &mp.r, ep.residual, g.N, g.M, ep.ldr, 32, 32, 1, 128));
#ifdef MECEFO_TIMING_KNOBS
  {  // timing experiments only (never in a product build): drop outputs / rotation / residual
    if (getenv("MECEFO_DBG_NOEPI")) outs.used[0] = outs.used[1] = outs.used[2] = 0;
    if (getenv("MECEFO_DBG_NOROPE")) p.epi.rope_cos = nullptr;
    if (getenv("MECEFO_DBG_NORES")) p.epi.residual = nullptr;
  }
#endif
  auto kern = gemm_tc_kernel<BN, AK, BKM, CL, NG, ROPE>;
  TRY(ensure_smem((const void*)kern, C::SMEM));
  const int grid = CLN * std::min(p.num_tiles_cl, kNumSMs / CLN);
  if (CLN == 1) {
    CUDA_TRY(pdl_launch(kern, dim3(grid), dim3(TC_THREADS), C::SMEM, s, mp, p, outs));
    return check_launch("gemm_tc_kernel");
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CLN;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mp, p, outs));
  return check_launch("gemm_tc_kernel<cluster>");
}

template <int BN, int CL, int NG = 1>
int dispatch_tc_major(mecefo_engine* e, const GemmCall& g, cudaStream_t s) {
  if (g.a.km && g.b.km) return launch_tc<BN, true, true, CL, NG>(e, g, s);
  if (g.a.km && !g.b.km) return launch_tc<BN, true, false, CL, NG>(e, g, s);
  if (!g.a.km && g.b.km) return launch_tc<BN, false, true, CL, NG>(e, g, s);
  return launch_tc<BN, false, false, CL, NG>(e, g, s);
}

// TMA-multicast CTA pairs along M whenever there are at least two M tiles
// and the B tile splits into halves (BN >= 128).
// Measured: pays off only for very large tile counts (the LM-head GEMMs,
// +10%); neutral-to-negative on the per-layer GEMMs.
bool use_cluster(const GemmCall& g, int BN) {
#ifdef MECEFO_TIMING_KNOBS
  if (getenv("MECEFO_NO_CLUSTER")) return false;
#endif
  if (g.b_diag_off) return false;  // the pair shares ONE B tile
  const int64_t cpt = g.paired ? BN / 2 : BN;
  const int64_t tiles = ((g.M + 127) / 128) * ((g.N + cpt - 1) / cpt);
  // (paired gate|up GEMMs measured 9% slower clustered: excluded)
  int64_t min_tiles = 1024;
#ifdef MECEFO_TIMING_KNOBS
  if (const char* v = getenv("MECEFO_CLUSTER_MIN_TILES")) min_tiles = atoll(v);
#endif
  return BN >= 128 && !g.paired && (g.M + 127) / 128 >= 2 && tiles >= min_tiles;
}

// CTA pairs with ONE cta_group::2 MMA (M = 256 per pair, each CTA stages its
// A rows and half of the B tile): BN = 256 single-group GEMMs with at least
// two M tiles and a long K. Halves the B bytes each CTA moves through shared
// memory, the operand-bandwidth limit of long 128 x 256 mainloops. Measured
// (C1, 16384 tokens): head g_unemb (K 16384) +9 %, d_xf (K 32000) +6 %,
// d_h2 (K 2752) +4 %, exact wgrad_gu +8 %; the K = 512 GEMMs with heavy epilogues (logits, QKV +
// RoPE, gate|up + SwiGLU) lost 5-10 % (shorter tiles: the pair's shared
// accumulator hand-off exposes more of the epilogue), so they stay single.
bool use_2sm(const GemmCall& g, int BN) {
  int64_t min_k = 1024;
#ifdef MECEFO_TIMING_KNOBS
  if (getenv("MECEFO_NO_2SM")) return false;
  if (const char* v = getenv("MECEFO_2SM_MIN_K")) min_k = atoll(v);
#endif
  // (fp32 residual epilogues excluded: down_residual, K 1376, lost 6 %)
  return BN == 256 && !g.b_diag_off && (g.M + 127) / 128 >= 2 && g.K >= min_k && !g.epi.residual;
}

// Tile width for the tcgen05 path. The MMA time of a tile is proportional to
// BN, so the kernel time is ~ waves(BN) * BN with waves = ceil(tiles / 148);
// pick the BN minimising it, and on ties the widest (better L2 arithmetic
// intensity: 128x256 tiles read 85 flop/B, 128x64 only 51).
int choose_bn(const GemmCall& g) {
  if (g.force_bn) return g.force_bn;
#ifdef MECEFO_TIMING_KNOBS
  // timing experiments only: MECEFO_BN_FOR="tag=BN,tag=BN"
  if (const char* v = getenv("MECEFO_BN_FOR")) {
    const char* hit = g.tag ? strstr(v, g.tag) : nullptr;
    if (hit && hit[strlen(g.tag)] == '=') return atoi(hit + strlen(g.tag) + 1);
  }
#endif
  const int64_t nacc = g.paired ? 2 * g.N : g.N;
  const int64_t tm = (g.M + 127) / 128;
  // per-flop penalty of narrower tiles (L2-bound operand traffic), measured
  int best = 64;
  double best_cost = 1e30;
  for (int BN : {256, 128, 64}) {
    if (BN > 64 && nacc <= BN / 2) continue;
    const int64_t cpt = g.paired ? BN / 2 : BN;
    const int64_t tiles = tm * ((g.N + cpt - 1) / cpt) * std::max(1, g.groups);
    const double eff = BN == 256 ? 1.0 : (BN == 128 ? 1.15 : 1.35);
    const double cost = (double)((tiles + kNumSMs - 1) / kNumSMs) * BN * eff;
    if (cost < best_cost * 0.999) { best_cost = cost; best = BN; }
  }
  return best;
}

int tiles_for(const GemmCall& g, int prec) {
  if (prec == PREC_BF16) {
    const int BN = choose_bn(g);
    const int64_t cpt = g.paired ? BN / 2 : BN;
    return (int)(((g.M + 127) / 128) * ((g.N + cpt - 1) / cpt)) * std::max(1, g.groups);
  }
  const int64_t cpt = g.paired ? 32 : 64;
  return (int)(((g.M + 63) / 64) * ((g.N + cpt - 1) / cpt));
}

int run_gemm(mecefo_engine* e, const GemmCall& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return MECEFO_OK;
  const double ncols = (double)(g.paired ? 2 * g.N : g.N);
  const double out_bytes = g.epi.kind == EPI_STORE ? (g.epi.out_prec == PREC_BF16 ? 2.0 : 4.0) * (1 + (g.epi.beta != 0.f) + (g.epi.residual != nullptr))
                         : (g.epi.kind == EPI_ATOMIC ? 8.0 : 3.0 * e->ps);
  const double ngr = (double)std::max(1, g.groups);
  ProfScope prof(g.tag, 2.0 * g.M * ncols * g.K * ngr,
                 ngr * ((double)e->ps * ((double)g.M * g.K + ncols * g.K) + out_bytes * (double)g.M * (double)g.N), s);
  if (g.split > 1 && g.epi.kind != EPI_ATOMIC)
    return set_err(MECEFO_ERR_CONSISTENCY, "split-K requires the atomic epilogue");
  if (g.b_diag_off && (e->prec != PREC_BF16 || g.paired))
    return set_err(MECEFO_ERR_CONSISTENCY, "block-diagonal batching is a tcgen05 (bf16), unpaired mode");
  if (g.groups > 1) {
    if (e->prec != PREC_BF16 || g.paired || g.groups > kMaxGroups)
      return set_err(MECEFO_ERR_CONSISTENCY, "grouped GEMM: bf16, unpaired, <= %d groups", kMaxGroups);
    const int BN = choose_bn(g);
    if (BN == 256) return dispatch_tc_major<256, 1, kMaxGroups>(e, g, s);
    if (BN == 128) return dispatch_tc_major<128, 1, kMaxGroups>(e, g, s);
    return dispatch_tc_major<64, 1, kMaxGroups>(e, g, s);
  }
  if (e->prec == PREC_BF16) {
    if (g.paired && !g.b.km) return set_err(MECEFO_ERR_CONSISTENCY, "paired GEMM needs a K-major B");
    const int BN = choose_bn(g);
    const bool two = use_2sm(g, BN);
    if (g.epi.rope_cos && BN == 256 && g.a.km && g.b.km && !g.paired && (two || !use_cluster(g, BN)))
      return two ? launch_tc<256, true, true, CL_2SM, 1, true>(e, g, s)  // QKV with RoPE (per-tile angle table)
                 : launch_tc<256, true, true, 1, 1, true>(e, g, s);
    if (two) return dispatch_tc_major<256, CL_2SM>(e, g, s);
    const bool cl = use_cluster(g, BN);
    if (BN == 256) return cl ? dispatch_tc_major<256, 2>(e, g, s) : dispatch_tc_major<256, 1>(e, g, s);
    if (BN == 128) return cl ? dispatch_tc_major<128, 2>(e, g, s) : dispatch_tc_major<128, 1>(e, g, s);
    return dispatch_tc_major<64, 1>(e, g, s);
  }
  GemmDev p{};
  p.M = (int)g.M; p.N = (int)g.N; p.K = (int)g.K;
  p.paired = g.paired ? 1 : 0;
  p.pair_off = g.pair_off;
  p.kblocks = (int)((g.K + 15) / 16);
  int split = std::max(1, std::min(g.split, p.kblocks));
  p.kb_per_split = (p.kblocks + split - 1) / split;
  p.split = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  p.tiles_m = (int)((g.M + 63) / 64);
  p.tiles_n = (int)((g.N + (g.paired ? 31 : 63)) / (g.paired ? 32 : 64));
  p.epi = g.epi;
  SimtOperand A{g.a.p, g.a.ld, g.a.km ? 1 : 0, e->prec};
  SimtOperand B{g.b.p, g.b.ld, g.b.km ? 1 : 0, e->prec};
  dim3 grid(p.tiles_m, p.tiles_n, p.split);
  CUDA_TRY(pdl_launch(gemm_simt_kernel, dim3(grid), dim3(256), 0, s, A, B, p));
  return check_launch("gemm_simt_kernel");
}

// out (fp32, ldo) += alpha * A B^T; split-K with atomics when the output has
// too few tiles to fill the GPU (the long-K Wgrad / low-rank contractions).
int gemm_accumulate(mecefo_engine* e, GemmCall g, float* out, int64_t ldo, float alpha, cudaStream_t s) {
  const int kblocks = (int)((g.K + 63) / 64);
  if (e->prec == PREC_BF16 && kblocks >= 8 && ((g.M + 127) / 128) * ((g.N + 255) / 256) < kNumSMs / 2) {
    // long-K, small output: one N tile as wide as the output (each A element
    // read once), split K across the SMs
    g.force_bn = g.N > 128 ? 256 : (g.N > 64 ? 128 : 64);
  }
  const int tiles = tiles_for(g, e->prec);
  if (tiles < 2 * kNumSMs / 3 && kblocks >= 8) {
    Epilogue ep{};
    ep.kind = EPI_ATOMIC; ep.out = out; ep.ldo = ldo; ep.alpha = alpha; ep.out_prec = PREC_F32;
    g.epi = ep;
    // wave-aware split: maximise units / (waves * 148) (a 149th CTA doubles
    // the time of a one-wave launch); ties go to the smaller split
    auto eff = [&](int sp) {
      const double units = (double)tiles * sp;
      return units / (std::ceil(units / kNumSMs) * kNumSMs);
    };
    int best = 1;
    for (int sp = 2; sp <= std::min(32, kblocks / 4); ++sp)
      if (eff(sp) > eff(best) + 0.01) best = sp;
    g.split = best;
    if (e->prec == PREC_F32) g.split = std::max(1, std::min(g.split * 4, (int)((g.K + 15) / 16) / 8));
  } else {
    g.epi = epi_store(out, ldo, PREC_F32, alpha, 1.f);
    g.split = 1;
  }
  return run_gemm(e, g, s);
}

template <int NV>
int launch_rms_fwd(const float* x, const float* g, void* out, float* inv, int64_t rows, int64_t m, int prec,
                   cudaStream_t s) {
  CUDA_TRY(pdl_launch(rmsnorm_fwd_vec_kernel<NV>, dim3((unsigned)((rows + 7) / 8)), dim3(256), 0, s, x, g, out, inv, (int)rows, (int)m, prec));
  return check_launch("rmsnorm_fwd_vec_kernel");
}

int rmsnorm_fwd(mecefo_engine* e, const float* x, const float* g, void* out, float* inv, int64_t rows, int64_t m,
                cudaStream_t s) {
  ProfScope prof("rmsnorm_fwd", 0.0, (double)rows * m * (4 + e->ps) + 4.0 * rows, s);
  if (m % 4 == 0 && m <= 2048) {
    const int nv = (int)((m + 127) / 128);
    if (nv <= 1) return launch_rms_fwd<1>(x, g, out, inv, rows, m, e->prec, s);
    if (nv <= 2) return launch_rms_fwd<2>(x, g, out, inv, rows, m, e->prec, s);
    if (nv <= 4) return launch_rms_fwd<4>(x, g, out, inv, rows, m, e->prec, s);
    if (nv <= 8) return launch_rms_fwd<8>(x, g, out, inv, rows, m, e->prec, s);
    return launch_rms_fwd<16>(x, g, out, inv, rows, m, e->prec, s);
  }
  const int warps = 8;
  CUDA_TRY(pdl_launch(rmsnorm_fwd_kernel, dim3((unsigned)((rows + warps - 1) / warps)), dim3(warps * 32), 0, s, x, g, out, inv, (int)rows, (int)m,
                                                                                    e->prec));
  return check_launch("rmsnorm_fwd_kernel");
}

template <int NV>
int launch_rms_bwd(const float* x, const float* g, const float* inv, const float* d, const float* resid, float* dx,
                   void* dx_lp, int prec, float* partial, int64_t rows, int64_t m, int nblk, int rpb, cudaStream_t s) {
  const int sm = 8 * NV * 32 * 16;
  if (sm > 48 * 1024) TRY(ensure_smem((const void*)rmsnorm_bwd_vec_kernel<NV>, sm));
  CUDA_TRY(pdl_launch(rmsnorm_bwd_vec_kernel<NV>, dim3(nblk), dim3(256), sm, s, x, g, inv, d, resid, dx, dx_lp, prec, partial, (int)rows, (int)m,
                                                   rpb));
  return check_launch("rmsnorm_bwd_vec_kernel");
}

// dx = resid + rmsnorm_bwd(...); grad_scale (+)= alpha * dscale (if non-null).
int rmsnorm_bwd(mecefo_engine* e, Ws& ws, const float* x, const float* g, const float* inv, const float* d,
                const float* resid, float* dx, void* dx_lp, float* grad_scale, float alpha, int64_t rows, int64_t m,
                cudaStream_t s) {
  ProfScope prof("rmsnorm_bwd", 0.0, (double)rows * m * (12 + (resid ? 4 : 0) + 4 + (dx_lp ? e->ps : 0)), s);
  const bool vec = m % 4 == 0 && m <= 2048;
  int nblk, rpb;
  if (vec) {
    nblk = (int)std::min<int64_t>((rows + 7) / 8, 2 * kNumSMs);
    rpb = (int)((rows + nblk - 1) / nblk);
    rpb = (rpb + 7) / 8 * 8;
    nblk = (int)((rows + rpb - 1) / rpb);
  } else {
    rpb = 64;
    nblk = (int)((rows + rpb - 1) / rpb);
  }
  float* partial = nullptr;
  if (grad_scale) TRY(ws.take((size_t)nblk * m * sizeof(float), reinterpret_cast<void**>(&partial)));
  if (vec) {
    const int nv = (int)((m + 127) / 128);
    int rc;
    if (nv <= 1) rc = launch_rms_bwd<1>(x, g, inv, d, resid, dx, dx_lp, e->prec, partial, rows, m, nblk, rpb, s);
    else if (nv <= 2) rc = launch_rms_bwd<2>(x, g, inv, d, resid, dx, dx_lp, e->prec, partial, rows, m, nblk, rpb, s);
    else if (nv <= 4) rc = launch_rms_bwd<4>(x, g, inv, d, resid, dx, dx_lp, e->prec, partial, rows, m, nblk, rpb, s);
    else if (nv <= 8) rc = launch_rms_bwd<8>(x, g, inv, d, resid, dx, dx_lp, e->prec, partial, rows, m, nblk, rpb, s);
    else rc = launch_rms_bwd<16>(x, g, inv, d, resid, dx, dx_lp, e->prec, partial, rows, m, nblk, rpb, s);
    TRY(rc);
  } else {
    const size_t sm = 8 * m * sizeof(float);
    if (sm > 48 * 1024) {
      TRY(ensure_smem((const void*)rmsnorm_bwd_kernel, 200 * 1024));
    }
    CUDA_TRY(pdl_launch(rmsnorm_bwd_kernel, dim3(nblk), dim3(256), sm, s, x, g, inv, d, resid, dx, dx_lp, e->prec, partial, (int)rows, (int)m, rpb));
    TRY(check_launch("rmsnorm_bwd_kernel"));
  }
  if (grad_scale) {
    CUDA_TRY(pdl_launch(colsum_finalize_kernel, dim3((unsigned)((m + 31) / 32)), dim3(256), 0, s, partial, nblk, (int)m, grad_scale, alpha, 1.f));
    TRY(check_launch("colsum_finalize_kernel"));
  }
  return MECEFO_OK;
}

// Which fused recompute kernel runs: 2 = the CTA-pair (cta_group::2) kernel,
// 1 = the single-CTA kernel. MECEFO_DUAL=1 selects the latter.
int dual_variant() {
#ifdef MECEFO_TIMING_KNOBS
  static const int v = getenv("MECEFO_DUAL") ? atoi(getenv("MECEFO_DUAL")) : 2;
  return v == 1 ? 1 : 2;
#else
  return 2;
#endif
}

// Fused d_act / gate / up tcgen05 kernel + SwiGLU backward epilogue (bf16).
int swiglu_bwd_dual(mecefo_engine* e, const void* dy_c, const void* h2, const void* w_down_c, const void* w_gu_c,
                    void* act, void* dcat, int64_t b, cudaStream_t s) {
  const int64_t m = e->d.hidden, f = e->d.ffn;
  ProfScope prof("nbr.fused_recompute_swiglu_bwd", 2.0 * b * f * m * 3.0,
                 2.0 * (2.0 * b * m + 3.0 * f * m) + 2.0 * b * f * (act ? 3 : 2), s);
  CUtensorMap tdy, th2, twd, tact, tdg, tdu;
  TRY(make_tmap(e, &tdy, dy_c, m, b, m, 64, TC_BM));
  TRY(make_tmap(e, &th2, h2, m, b, m, 64, TC_BM));
  TRY(make_tmap(e, &twd, w_down_c, f, m, f, 64, 64));
  std::memset(&tact, 0, sizeof(tact));
  if (act) TRY(make_tmap(e, &tact, act, f, b, f, 32, 32, 0, 64));
  TRY(make_tmap(e, &tdg, dcat, f, b, 2 * f, 32, 32, 0, 64));
  TRY(make_tmap(e, &tdu, reinterpret_cast<uint8_t*>(dcat) + f * 2, f, b, 2 * f, 32, 32, 0, 64));
  // 128-pair-column kernel (TMEM ring; gemm_dual.cuh)
  CUtensorMap twgu128;
  TRY(make_tmap(e, &twgu128, w_gu_c, m, 2 * f, m, 64, 128));
  DualDev p{};
  p.M = (int)b; p.NP = (int)f; p.K = (int)m; p.f_off = f;
  p.kblocks = (int)((m + TC_BK - 1) / TC_BK);
  p.tiles_m = (int)((b + TC_BM - 1) / TC_BM);
  p.tiles_n = (int)((f + D2_NP - 1) / D2_NP);
  p.num_tiles = p.tiles_m * p.tiles_n;
  p.has_act = act ? 1 : 0;
  p.act = reinterpret_cast<__nv_bfloat16*>(act);
  p.dcat = reinterpret_cast<__nv_bfloat16*>(dcat);
  int variant = dual_variant();
#ifdef MECEFO_TIMING_KNOBS
  if (const char* v = getenv("MECEFO_DUAL_DBG")) p.dbg = atoi(v);
  if (const char* v = getenv("MECEFO_DUAL_DIRECT")) p.direct = atoi(v);
#endif
  if (variant == 2) {  // CTA-pair kernel: 256-row tiles, B operand halves per CTA
    CUtensorMap twg64;
    TRY(make_tmap(e, &twg64, w_gu_c, m, 2 * f, m, 64, 64));
    p.tiles_m = (int)((b + 2 * TC_BM - 1) / (2 * TC_BM));
    p.num_tiles = p.tiles_m * p.tiles_n;
    int epw = 8;  // measured: 16 one-chunk warps spill at 96 registers and lose an operand stage (92.5 vs 86 us)
#ifdef MECEFO_TIMING_KNOBS
    if (const char* v = getenv("MECEFO_DUAL_EPW")) epw = atoi(v) == 8 ? 8 : 16;
#endif
    auto kern = epw == 16 ? swiglu_bwd_dual2sm_kernel<16> : swiglu_bwd_dual2sm_kernel<8>;
    const int smem = epw == 16 ? D2S<16>::SMEM : D2S<8>::SMEM;
    TRY(ensure_smem((const void*)kern, smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * std::min(p.num_tiles, kNumSMs / 2)));
    cfg.blockDim = dim3(epw == 16 ? D2S<16>::THREADS : D2S<8>::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tdy, th2, twd, twg64, tact, tdg, tdu, p));
    return check_launch("swiglu_bwd_dual2sm_kernel");
  }
  TRY(ensure_smem((const void*)swiglu_bwd_dual128_kernel, D2_SMEM));
  CUDA_TRY(pdl_launch(swiglu_bwd_dual128_kernel, dim3(std::min(p.num_tiles, kNumSMs)), dim3(TC_THREADS), D2_SMEM, s,
                      tdy, th2, twd, twgu128, tact, tdg, tdu, p));
  return check_launch("swiglu_bwd_dual128_kernel");
}

int cast_to_compute(mecefo_engine* e, const float* src, void* dst, int64_t n, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4096);
  CUDA_TRY(pdl_launch(cast_f32_kernel, dim3((unsigned)std::max<int64_t>(blocks, 1)), dim3(256), 0, s, src, dst, n, e->prec));
  return check_launch("cast_f32_kernel");
}

int attention(mecefo_engine* e, bool backward, AttnDev a, int64_t tokens, cudaStream_t s) {
  const int hd = (int)(e->d.hidden / e->d.heads);
  if (!backward && e->prec == PREC_BF16 && hd == 64 && a.T % 64 == 0 && a.T <= 256) {
    ProfScope prof("attn_fwd_tc", 2.0 * tokens * a.T * a.m, (double)tokens * a.m * e->ps * 4, s);
    CUtensorMap tq;
    TRY(make_tmap(e, &tq, a.qkv, 3 * a.m, tokens, a.ld_qkv, 64, 64));
    AttnTcArgs t{a.ctx, a.ld_ctx, a.lse, a.T, a.H, a.m, a.scale};
    TRY(ensure_smem((const void*)attn_fwd_tc_kernel, ATC_SMEM));
    dim3 grid((unsigned)(tokens / a.T) * a.H, (unsigned)((a.T + 127) / 128));
    CUDA_TRY(pdl_launch(attn_fwd_tc_kernel, dim3(grid), dim3(ATC_THREADS), ATC_SMEM, s, tq, t));
    return check_launch("attn_fwd_tc_kernel");
  }
  if (backward && e->prec == PREC_BF16 && hd == 64 && a.T % 128 == 0 && a.T <= 256) {
    ProfScope prof("attn_bwd_tc", 5.0 * tokens * a.T * a.m, (double)tokens * a.m * e->ps * 9, s);
    CUtensorMap tq, tdo;
    TRY(make_tmap(e, &tq, a.qkv, 3 * a.m, tokens, a.ld_qkv, 64, 64));
    TRY(make_tmap(e, &tdo, a.dctx, a.m, tokens, a.ld_ctx, 64, 64));
    // theta table: stored after the seq_len x (hd/2) cos table (as for the QKV epilogue)
    AttnBwdTcArgs t{a.ctx, a.dctx, a.lse, a.dqkv, e->rope_cos + (size_t)e->d.seq_len * (hd / 2), a.T, a.H, a.m,
                    a.rope, a.scale};
    TRY(ensure_smem((const void*)attn_bwd_tc_kernel, ABT_SMEM));
    const int items = (int)((tokens / a.T) * a.H);
    if (items <= 0) return MECEFO_OK;
    CUDA_TRY(pdl_launch(attn_bwd_tc_kernel, dim3((unsigned)std::min(items, kNumSMs)), dim3(ABT_THREADS), ABT_SMEM, s,
                        tq, tdo, t, items));
    return check_launch("attn_bwd_tc_kernel");
  }
  ProfScope prof(backward ? "attn_bwd" : "attn_fwd", (backward ? 4.0 : 2.0) * tokens * a.T * a.m,
                 (double)tokens * a.m * e->ps * (backward ? 9 : 4), s);
  const int nseq = (int)(tokens / e->d.seq_len);
  dim3 grid(nseq * a.H, (a.T + 63) / 64);
  const size_t per_row = (size_t)(hd + 4) * sizeof(float);
  size_t sm = backward ? std::max<size_t>(2 * a.T * per_row, 2 * a.T * per_row + 2 * a.T * sizeof(float))
                       : 2 * (size_t)a.T * per_row;
  if (sm > 220 * 1024) return set_err(MECEFO_ERR_CONTRACT, "seq_len %d x head_dim %d exceeds the attention smem plan", a.T, hd);
#define ATTN_CASE(D)                                                                                      \
  case D: {                                                                                               \
    if (!backward) {                                                                                      \
      CUDA_TRY(cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
      CUDA_TRY(pdl_launch(attn_fwd_kernel<D>, dim3(grid), dim3(256), sm, s, a));                                                        \
      return check_launch("attn_fwd_kernel");                                                             \
    }                                                                                                     \
    CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dkv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    CUDA_TRY(pdl_launch(attn_bwd_dq_kernel<D>, dim3(grid), dim3(256), sm, s, a));                                                       \
    TRY(check_launch("attn_bwd_dq_kernel"));                                                              \
    CUDA_TRY(pdl_launch(attn_bwd_dkv_kernel<D>, dim3(grid), dim3(256), sm, s, a));                                                      \
    return check_launch("attn_bwd_dkv_kernel");                                                           \
  }
  switch (hd) {
    ATTN_CASE(2)
    ATTN_CASE(4)
    ATTN_CASE(8)
    ATTN_CASE(16)
    ATTN_CASE(32)
    ATTN_CASE(64)
    ATTN_CASE(128)
    default:
      return set_err(MECEFO_ERR_CONTRACT, "unsupported head_dim %d (supported: 2..128, powers of two)", hd);
  }
#undef ATTN_CASE
}

AttnDev attn_args(mecefo_engine* e) {
  AttnDev a{};
  a.T = (int)e->d.seq_len;
  a.H = (int)e->d.heads;
  a.m = (int)e->d.hidden;
  a.rope = e->d.rope;
  a.prec = e->prec;
  a.cosT = e->rope_cos;
  a.sinT = e->rope_sin;
  a.scale = (float)(1.0 / std::sqrt((double)(e->d.hidden / e->d.heads)));
  return a;
}

int check_tokens(mecefo_engine* e, int64_t tokens) {
  if (tokens <= 0 || tokens % e->d.seq_len != 0)
    return set_err(MECEFO_ERR_CONTRACT, "activations of %lld rows do not match seq_len=%lld", (long long)tokens,
                   (long long)e->d.seq_len);
  return MECEFO_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* mecefo_last_error(void) { return g_last_error.c_str(); }
const char* mecefo_version(void) { return "mecefo-b200 0.1 (sm_100a)"; }
int64_t mecefo_launch_count(void) { return g_launches.load(); }

int mecefo_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.on = on != 0;
  g_prof.recs.clear();
  g_prof.next = 0;
  return MECEFO_OK;
}

int64_t mecefo_profile_count(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  return (int64_t)g_prof.recs.size();
}

int mecefo_profile_record(int64_t i, const char** tag, float* ms, double* flops, double* bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (i < 0 || i >= (int64_t)g_prof.recs.size()) return set_err(MECEFO_ERR_CONTRACT, "profile index out of range");
  const ProfRec& r = g_prof.recs[i];
  CUDA_TRY(cudaEventSynchronize(r.b));
  CUDA_TRY(cudaEventElapsedTime(ms, r.a, r.b));
  *tag = r.tag;
  *flops = r.flops;
  *bytes = r.bytes;
  return MECEFO_OK;
}

int mecefo_engine_create(mecefo_engine** out, const mecefo_dims* dims) {
  if (!out || !dims) return set_err(MECEFO_ERR_CONTRACT, "null argument");
  const mecefo_dims& d = *dims;
  if (d.vocab < 1 || d.hidden < 1 || d.heads < 1 || d.ffn < 1 || d.layers < 1 || d.seq_len < 1)
    return set_err(MECEFO_ERR_CONTRACT, "dims must be >= 1");
  if (d.hidden % d.heads != 0) return set_err(MECEFO_ERR_CONTRACT, "hidden must be divisible by heads");
  if (d.rope && (d.hidden / d.heads) % 2 != 0) return set_err(MECEFO_ERR_CONTRACT, "rotary positions need an even head dim");
  if (d.precision != MECEFO_PREC_F32 && d.precision != MECEFO_PREC_BF16)
    return set_err(MECEFO_ERR_CONFIG, "unknown precision %d", d.precision);
  if (d.precision == MECEFO_PREC_BF16 && (d.hidden % 8 != 0 || d.vocab % 8 != 0))
    return set_err(MECEFO_ERR_CONTRACT, "bf16 (TMA) mode needs hidden and vocab to be multiples of 8 (16-byte rows)");
  auto* e = new mecefo_engine();
  e->d = d;
  // FFN width padded to 16-byte rows (LLaMA-1B: f = 5461 -> 5464): zero pad
  // rows of W_gate/W_up and zero pad columns of W_down contribute exactly
  // nothing forward or backward, and their gradients stay zero.
  e->d.ffn = mecefo_padded_ffn(d.ffn);
  e->prec = d.precision;
  e->ps = d.precision == MECEFO_PREC_BF16 ? 2 : 4;
  const int hd = (int)(d.hidden / d.heads);
  const int half = std::max(1, hd / 2);
  // cos table followed by the `half` frequencies theta_j (fp32) that the tcgen05
  // QKV epilogue uses to compute its angles
  std::vector<float> c((size_t)d.seq_len * half + half), sn((size_t)d.seq_len * half);
  for (int j = 0; j < half; ++j) c[(size_t)d.seq_len * half + j] = (float)std::pow(10000.0, -2.0 * j / hd);
  for (int64_t t = 0; t < d.seq_len; ++t)
    for (int j = 0; j < half; ++j) {
      const double theta = std::pow(10000.0, -2.0 * j / hd);  // model.py:274
      const double ang = (double)t * theta;
      c[t * half + j] = (float)std::cos(ang);
      sn[t * half + j] = (float)std::sin(ang);
    }
  cudaError_t ce = cudaMalloc(&e->rope_cos, c.size() * sizeof(float));
  if (ce == cudaSuccess) ce = cudaMalloc(&e->rope_sin, sn.size() * sizeof(float));
  if (ce == cudaSuccess) ce = cudaMemcpy(e->rope_cos, c.data(), c.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(e->rope_sin, sn.data(), sn.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMalloc(&e->status, 16);
  if (ce == cudaSuccess) ce = cudaMemset(e->status, 0, 16);
  if (ce != cudaSuccess) {
    cudaFree(e->rope_cos);
    cudaFree(e->rope_sin);
    cudaFree(e->status);
    delete e;
    return set_err(MECEFO_ERR_CUDA, "engine allocation failed: %s", cudaGetErrorString(ce));
  }
  *out = e;
  return MECEFO_OK;
}

int mecefo_engine_destroy(mecefo_engine* e) {
  if (!e) return MECEFO_OK;
  cudaFree(e->rope_cos);
  cudaFree(e->rope_sin);
  cudaFree(e->status);
  delete e;
  return MECEFO_OK;
}

int64_t mecefo_padded_ffn(int64_t ffn) { return (ffn + 7) / 8 * 8; }

int mecefo_status_device(mecefo_engine* e, int32_t** out) {
  if (!e || !out) return set_err(MECEFO_ERR_CONTRACT, "null argument");
  *out = e->status;
  return MECEFO_OK;
}

int mecefo_status_snapshot(mecefo_engine* e, int32_t* host, void* stream) {
  if (!e || !host) return set_err(MECEFO_ERR_CONTRACT, "null argument");
  CUDA_TRY(cudaMemcpyAsync(host, e->status, 4, cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)));
  return MECEFO_OK;
}

int mecefo_memset_zero(void* p, size_t bytes, void* stream) {
  if (bytes == 0) return MECEFO_OK;
  CUDA_TRY(cudaMemsetAsync(p, 0, bytes, reinterpret_cast<cudaStream_t>(stream)));
  return MECEFO_OK;
}

int mecefo_status_reset(mecefo_engine* e, void* stream) {
  if (!e) return set_err(MECEFO_ERR_CONTRACT, "null engine");
  CUDA_TRY(cudaMemsetAsync(e->status, 0, 16, reinterpret_cast<cudaStream_t>(stream)));
  return MECEFO_OK;
}

size_t mecefo_workspace_bytes(const mecefo_engine* e, int64_t tokens, int32_t rank_pad) {
  const int64_t m = e->d.hidden, f = e->d.ffn, H = e->d.heads, ps = e->ps;
  const int64_t rp = std::max<int32_t>(rank_pad, 16);
  const int64_t per_tok = (6 * m + 4 * f + 3 * rp) * ps + 16 * m + 8 * H + 64;
  const int64_t fixed = 3 * std::max(m, f) * rp * (4 + ps) + 4 * f * rp * (4 + ps) + tokens * 2 * rp * ps +
                        ((tokens + 63) / 64 + 8) * m * 4 * 2 + e->d.vocab * 4 + (4 << 20);
  return (size_t)(tokens * per_tok + fixed);
}

namespace {

// x1 = x + A W^T and h = rmsnorm(x1) * g, inv (gemm_norm.cuh): the fused
// O-projection + norm of one block forward when m = 512 and the pass fills a
// wave of row blocks; returns false when it does not apply.
bool resid_norm_applies(const mecefo_engine* e, int64_t b) {
#ifdef MECEFO_TIMING_KNOBS
  if (getenv("MECEFO_NO_RESID_NORM")) return false;
#endif
  return e->prec == PREC_BF16 && e->d.hidden == GN_N && (b + TC_BM - 1) / TC_BM >= 100;
}

int resid_norm_gemm(mecefo_engine* e, const void* a, int64_t K, const void* w, const float* x, float* x1, void* h,
                    float* inv, const float* gain, int64_t b, cudaStream_t s, const char* tag = "fwd.o_residual_norm") {
  ProfScope prof(tag, 2.0 * b * GN_N * K,
                 2.0 * (b * K + GN_N * K) + 4.0 * 2 * b * GN_N + 2.0 * b * GN_N + 4.0 * b, s);
  GnMaps mp;
  TRY(make_tmap(e, &mp.a, a, K, b, K, 64, TC_BM));
  TRY(make_tmap(e, &mp.b, w, K, GN_N, K, 64, 256));
  TRY(make_tmap(e, &mp.r, x, GN_N, b, GN_N, 32, 32, 1, 128));
  TRY(make_tmap(e, &mp.o, x1, GN_N, b, GN_N, 32, 32, 1, 128));
  TRY(make_tmap(e, &mp.h, h, GN_N, b, GN_N, 32, 32, 0, 64));
  GnDev p{};
  p.M = (int)b; p.K = (int)K; p.kblocks = (int)((K + TC_BK - 1) / TC_BK);
  p.eps = kRmsEps; p.gain = gain; p.inv = inv;
  TRY(ensure_smem((const void*)gemm_resid_norm_kernel, GN_SMEM));
  CUDA_TRY(pdl_launch(gemm_resid_norm_kernel, dim3((unsigned)((b + TC_BM - 1) / TC_BM)), dim3(TC_THREADS), GN_SMEM, s,
                      mp, p));
  return check_launch("gemm_resid_norm_kernel");
}

}  // namespace

namespace {
int forward_block_impl(mecefo_engine* e, const mecefo_layer_weights* lw, mecefo_block_cache* c, float* y,
                       int64_t tokens, int32_t mode, int32_t flags, const float* next_gain, void* next_h1,
                       float* next_inv1, void* wsp, size_t ws_bytes, void* stream);
}  // namespace

int mecefo_forward_block(mecefo_engine* e, const mecefo_layer_weights* lw, mecefo_block_cache* c, float* y, void* y_c,
                         int64_t tokens, int32_t mode, void* wsp, size_t ws_bytes, void* stream) {
  (void)y_c;
  return forward_block_impl(e, lw, c, y, tokens, mode, 0, nullptr, nullptr, nullptr, wsp, ws_bytes, stream);
}

int mecefo_forward_block_chained(mecefo_engine* e, const mecefo_layer_weights* lw, mecefo_block_cache* c, float* y,
                                 int64_t tokens, int32_t mode, int32_t flags, const float* next_norm_gain,
                                 void* next_h1, float* next_inv1, void* wsp, size_t ws_bytes, void* stream) {
  if ((flags & MECEFO_FWD_H1_READY) && (!c->h1 || !c->inv1))
    return set_err(MECEFO_ERR_CONTRACT, "MECEFO_FWD_H1_READY needs cache->h1 and cache->inv1");
  if (next_norm_gain && (!next_h1 || !next_inv1))
    return set_err(MECEFO_ERR_CONTRACT, "next_norm_gain needs next_h1 and next_inv1");
  return forward_block_impl(e, lw, c, y, tokens, mode, flags, next_norm_gain, next_h1, next_inv1, wsp, ws_bytes,
                            stream);
}

namespace {
int forward_block_impl(mecefo_engine* e, const mecefo_layer_weights* lw, mecefo_block_cache* c, float* y,
                       int64_t tokens, int32_t mode, int32_t flags, const float* next_gain, void* next_h1,
                       float* next_inv1, void* wsp, size_t ws_bytes, void* stream) {
  TRY(check_tokens(e, tokens));
  if (mode != MECEFO_CACHE_FULL && mode != MECEFO_CACHE_FFN_INPUT_ONLY)
    return set_err(MECEFO_ERR_CONTRACT, "unknown cache mode %d", mode);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const bool full = mode == MECEFO_CACHE_FULL;
  const int64_t b = tokens, m = e->d.hidden, f = e->d.ffn, H = e->d.heads;
  Ws ws(wsp, ws_bytes);
  void *h1 = c->h1, *qkv = c->qkv, *ctx = c->ctx, *h2 = c->h2, *act = c->act;
  float *inv1 = c->inv1, *lse = c->lse, *inv2 = c->inv2;
  const bool h1_ready = (flags & MECEFO_FWD_H1_READY) != 0;  // the previous block's down kernel wrote them
  if (!h1_ready && (!full || !h1)) TRY(ws.take(b * m * e->ps, &h1));
  if (!h1_ready && (!full || !inv1)) TRY(ws.take(b * 4, reinterpret_cast<void**>(&inv1)));
  if (!full || !qkv) TRY(ws.take(b * 3 * m * e->ps, &qkv));
  if (!full || !ctx) TRY(ws.take(b * m * e->ps, &ctx));
  if (!full) lse = nullptr;
  if (full && !lse) TRY(ws.take(b * H * 4, reinterpret_cast<void**>(&lse)));
  if (!full || !h2) TRY(ws.take(b * m * e->ps, &h2));
  if (!full || !inv2) TRY(ws.take(b * 4, reinterpret_cast<void**>(&inv2)));
  if (!full || !act) TRY(ws.take(b * f * e->ps, &act));

  // h1 = rmsnorm(x) * g_mha; qkv = h1 [Wq;Wk;Wv]^T            (model.py:404, 320-322)
  if (!h1_ready) TRY(rmsnorm_fwd(e, c->x, lw->norm_mha, h1, inv1, b, m, s));
  GemmCall g;
  g.M = b; g.N = 3 * m; g.K = m;
  g.a = {h1, m, true}; g.b = {lw->w_qkv_c, m, true};
  g.epi = epi_store(qkv, 3 * m, e->prec);
  if (e->d.rope) {  // q, k leave the GEMM rotated (model.py:323-326)
    g.epi.rope_cos = e->rope_cos; g.epi.rope_sin = e->rope_sin;
    g.epi.rope_T = (int)e->d.seq_len; g.epi.rope_hd = (int)(m / e->d.heads); g.epi.rope_cols = (int)(2 * m);
    g.epi.rope_theta = e->rope_cos + e->d.seq_len * (g.epi.rope_hd / 2);
  }
  g.tag = "fwd.qkv";
  TRY(run_gemm(e, g, s));
  // causal attention with RoPE -> ctx                         (model.py:323-331)
  AttnDev a = attn_args(e);
  a.qkv = qkv; a.ld_qkv = 3 * m; a.ctx = ctx; a.ld_ctx = m; a.lse = lse;
  TRY(attention(e, false, a, b, s));
  // x1 = x + ctx Wo^T                                          (model.py:332, 406)
  // h2 = rmsnorm(x1) * g_ffn                                   (model.py:213)
  if (resid_norm_applies(e, b)) {
    TRY(resid_norm_gemm(e, ctx, m, lw->w_o_c, c->x, c->x1, h2, inv2, lw->norm_ffn, b, s));
  } else {
    g = GemmCall();
    g.M = b; g.N = m; g.K = m;
    g.a = {ctx, m, true}; g.b = {lw->w_o_c, m, true};
    g.epi = epi_store(c->x1, m, PREC_F32, 1.f, 0.f, c->x, m);
    g.tag = "fwd.o_residual";
    TRY(run_gemm(e, g, s));
    TRY(rmsnorm_fwd(e, c->x1, lw->norm_ffn, h2, inv2, b, m, s));
  }
  // act = silu(h2 Wg^T) * (h2 Wu^T)                            (model.py:214-216)
  g = GemmCall();
  g.M = b; g.N = f; g.K = m;
  g.a = {h2, m, true}; g.b = {lw->w_gu_c, m, true};
  g.paired = true; g.pair_off = f;
  Epilogue ep{};
  ep.kind = EPI_SWIGLU_FWD; ep.out = act; ep.ldo = f; ep.act_prec = e->prec;
  if (full && c->gu) { ep.out2 = c->gu; ep.ldo2 = 2 * f; ep.off2 = f; }
  g.epi = ep;
  g.tag = "fwd.gu_swiglu";
  TRY(run_gemm(e, g, s));
  // y = x1 + act Wd^T                                          (model.py:217, 408)
  // [+ the next block's h1 = rmsnorm(y) * g_mha', inv1'        (model.py:404, 183-186)]
  if (next_gain && resid_norm_applies(e, b) && f % 8 == 0) {
    TRY(resid_norm_gemm(e, act, f, lw->w_down_c, c->x1, y, next_h1, next_inv1, next_gain, b, s,
                        "fwd.down_residual_norm"));
    return MECEFO_OK;
  }
  g = GemmCall();
  g.M = b; g.N = m; g.K = f;
  g.a = {act, f, true}; g.b = {lw->w_down_c, f, true};
  g.epi = epi_store(y, m, PREC_F32, 1.f, 0.f, c->x1, m);
  g.tag = "fwd.down_residual";
  TRY(run_gemm(e, g, s));
  if (next_gain) TRY(rmsnorm_fwd(e, y, next_gain, next_h1, next_inv1, b, m, s));
  return MECEFO_OK;
}
}  // namespace

namespace {

// Low-rank FFN weight gradients (approx.py:24-42, 118-126):
//   grad[kind] += alpha * d2^T (inp2 V1) V1^T   for kind in (gate, up, down).
int lowrank_ffn_wgrads(mecefo_engine* e, Ws& ws, const mecefo_projection* pj, const void* dy_c, const void* h2,
                       const void* act, const void* dcat, const mecefo_layer_grads* gr, int64_t b, cudaStream_t s) {
  const int64_t m = e->d.hidden, f = e->d.ffn, rp = pj->rank_pad;
  const int ps = e->ps;
  if (rp % 16 != 0) return set_err(MECEFO_ERR_CONTRACT, "rank_pad must be a multiple of 16");
  // kind -> (d2, ld_d2, out dim, inp2, in dim, grad pointer)
  struct K { const void* d2; int64_t ldd; int64_t n_out; const void* inp; int64_t n_in; float* grad; };
  const K kinds[3] = {
      {dcat, 2 * f, f, h2, m, gr->gu},
      {dcat ? reinterpret_cast<const uint8_t*>(dcat) + f * ps : nullptr, 2 * f, f, h2, m,
       gr->gu ? gr->gu + f * m : nullptr},
      {dy_c, m, m, act, f, gr->down},
  };
  void* P;
  float* Q;
  void* Qc;
  TRY(ws.take(b * 2 * rp * ps, &P));
  if (e->prec == PREC_BF16 && rp % TC_BM == 0 && kinds[0].grad && kinds[1].grad && pj->v1_gu && pj->v1t_gu &&
      pj->v1[2] && pj->v1t[2]) {
    // Transposed chain (bf16, rank_pad a multiple of the 128-row tile):
    //   [P_g | P_u]   = h2 [V1_g | V1_u]                              (b, 2rp)
    //   [Q_g^T ; Q_u^T] = [P_g | P_u]^T [d_gate | d_up], block-diagonal:
    //                   M tile 0 (P_g^T) meets d_gate, tile 1 (P_u^T) d_up (2rp, f)
    //   [G_g ; G_u]  += alpha blockdiag(Q) [V1_g | V1_u]^T              (2f, m)
    //   down:  Q_d^T = P_d^T dy (rp, m);  G_d += alpha Q_d V1_d^T      (m, f)
    // The long-K contraction runs with the token dim as K and the wide
    // FFN dim as N (256-column tiles), no wasted off-diagonal blocks.
    float* QT;
    void* QTc;
    TRY(ws.take(2 * rp * f * 4, reinterpret_cast<void**>(&QT)));
    TRY(ws.take(2 * rp * 2 * f * ps, &QTc));
    GemmCall g;
    g.M = b; g.N = 2 * rp; g.K = m;
    g.a = {h2, m, true}; g.b = {pj->v1t_gu, m, true};
    g.epi = epi_store(P, 2 * rp, e->prec);
    g.tag = "lowrank.P";
    TRY(run_gemm(e, g, s));
    CUDA_TRY(cudaMemsetAsync(QT, 0, 2 * rp * f * 4, s));
    g = GemmCall();
    g.M = 2 * rp; g.N = f; g.K = b;
    g.a = {P, 2 * rp, false}; g.b = {dcat, 2 * f, false};
    g.b_diag_off = f;
    g.b_diag_div = (int)(rp / TC_BM);  // rows [0, rp) meet d_gate, [rp, 2rp) d_up
    g.tag = "lowrank.Q_gu";
    TRY(gemm_accumulate(e, g, QT, f, 1.f, s));
    {
      const int64_t n = 2 * rp * 2 * f;
      ProfScope prof("lowrank.cast", 0.0, 6.0 * n / 2, s);
      CUDA_TRY(pdl_launch(cast_blockdiag_t_kernel, dim3((unsigned)std::min<int64_t>((n + 255) / 256, 4 * kNumSMs)),
                          dim3(256), 0, s, (const float*)QT, (__nv_bfloat16*)QTc, (int)rp, (int)f, (int64_t)1));
      TRY(check_launch("cast_blockdiag_t_kernel"));
    }
    g = GemmCall();
    g.M = 2 * f; g.N = m; g.K = 2 * rp;
    g.a = {QTc, 2 * f, false}; g.b = {pj->v1_gu, 2 * rp, true};
    g.epi = epi_store(gr->gu, m, PREC_F32, gr->alpha_ffn, 1.f);
    g.tag = "lowrank.up_proj";
    TRY(run_gemm(e, g, s));
    if (!kinds[2].grad) return MECEFO_OK;
    // down: P_d = act V1_d (b, rp) into the P buffer (stream-ordered reuse)
    g = GemmCall();
    g.M = b; g.N = rp; g.K = f;
    g.a = {act, f, true}; g.b = {pj->v1t[2], f, true};
    g.epi = epi_store(P, rp, e->prec);
    g.tag = "lowrank.P_down";
    TRY(run_gemm(e, g, s));
    CUDA_TRY(cudaMemsetAsync(QT, 0, rp * m * 4, s));
    g = GemmCall();
    g.M = rp; g.N = m; g.K = b;
    g.a = {P, rp, false}; g.b = {dy_c, m, false};
    g.tag = "lowrank.Q_down";
    TRY(gemm_accumulate(e, g, QT, m, 1.f, s));
    TRY(cast_to_compute(e, QT, QTc, rp * m, s));
    g = GemmCall();
    g.M = m; g.N = f; g.K = rp;
    g.a = {QTc, m, false}; g.b = {pj->v1[2], rp, true};
    g.epi = epi_store(kinds[2].grad, f, PREC_F32, gr->alpha_ffn, 1.f);
    g.tag = "lowrank.up_proj";
    return run_gemm(e, g, s);
  }
  TRY(ws.take(std::max(m, f) * rp * 4, reinterpret_cast<void**>(&Q)));
  if (e->prec == PREC_BF16) TRY(ws.take(std::max(m, f) * rp * ps, &Qc));
  else Qc = Q;
  for (int k = 0; k < 3; ++k)
    if (kinds[k].grad && (!pj->v1[k] || !pj->v1t[k]))
      return set_err(MECEFO_ERR_CONTRACT, "projection basis %d missing", k);
  // Fully merged gate/up chain (packed bases supplied):
  //   [P_g | P_u]  = h2 [V1_g | V1_u]                         (b, 2rp)
  //   Q            = [d_gate | d_up]^T [P_g | P_u]             (2f, 2rp), split-K
  //   [G_g ; G_u] += alpha blockdiag(Q) [V1_g | V1_u]^T        (2f, m) = the gate|up grad
  if (kinds[0].grad && kinds[1].grad && pj->v1_gu && pj->v1t_gu && e->prec == PREC_BF16) {
    float* Q2;
    void* Q2c;
    TRY(ws.take(2 * f * 2 * rp * 4, reinterpret_cast<void**>(&Q2)));
    TRY(ws.take(2 * f * 2 * rp * ps, &Q2c));
    GemmCall g;
    g.M = b; g.N = 2 * rp; g.K = m;
    g.a = {h2, m, true}; g.b = {pj->v1t_gu, m, true};
    g.epi = epi_store(P, 2 * rp, e->prec);
    g.tag = "lowrank.P";
    TRY(run_gemm(e, g, s));
    CUDA_TRY(cudaMemsetAsync(Q2, 0, 2 * f * 2 * rp * 4, s));
    g = GemmCall();
    g.M = 2 * f; g.N = 2 * rp; g.K = b;
    g.a = {dcat, 2 * f, false}; g.b = {P, 2 * rp, false};
    g.tag = "lowrank.Q";
    TRY(gemm_accumulate(e, g, Q2, 2 * rp, 1.f, s));
    {
      const int64_t n = 4 * f * rp;
      ProfScope prof("lowrank.cast", 0.0, 6.0 * n, s);
      CUDA_TRY(pdl_launch(cast_blockdiag_kernel, dim3((unsigned)std::min<int64_t>((n + 255) / 256, 4 * kNumSMs)),
                          dim3(256), 0, s, (const float*)Q2, Q2c, (int)f, (int)rp, e->prec));
      TRY(check_launch("cast_blockdiag_kernel"));
    }
    g = GemmCall();
    g.M = 2 * f; g.N = m; g.K = 2 * rp;
    g.a = {Q2c, 2 * rp, true}; g.b = {pj->v1_gu, 2 * rp, true};
    g.epi = epi_store(gr->gu, m, PREC_F32, gr->alpha_ffn, 1.f);
    g.tag = "lowrank.up_proj";
    TRY(run_gemm(e, g, s));
    if (!kinds[2].grad) return MECEFO_OK;
    mecefo_projection down_only = *pj;
    mecefo_layer_grads gdown = *gr;
    gdown.gu = nullptr;
    down_only.v1_gu = down_only.v1t_gu = nullptr;
    return lowrank_ffn_wgrads(e, ws, &down_only, dy_c, h2, act, dcat, &gdown, b, s);
  }
  // gate and up share inp2 = h2: when their V1^T are stacked contiguously,
  // one GEMM produces [P_gate | P_up] (b, 2 rp).
  const bool merged = kinds[0].grad && kinds[1].grad &&
                      reinterpret_cast<const uint8_t*>(pj->v1t[1]) ==
                          reinterpret_cast<const uint8_t*>(pj->v1t[0]) + rp * m * ps;
  if (merged) {
    GemmCall g;
    g.M = b; g.N = 2 * rp; g.K = m;
    g.a = {h2, m, true}; g.b = {pj->v1t[0], m, true};
    g.epi = epi_store(P, 2 * rp, e->prec);
    g.tag = "lowrank.P";
    TRY(run_gemm(e, g, s));
  }
  for (int k = 0; k < 3; ++k) {
    const K& kd = kinds[k];
    if (!kd.grad) continue;
    const void* Pk = P;
    int64_t ldp = rp;
    if (merged && k < 2) {
      Pk = reinterpret_cast<const uint8_t*>(P) + k * rp * ps;
      ldp = 2 * rp;
    } else {
      // P = inp2 V1  (b, rp)
      GemmCall g;
      g.M = b; g.N = rp; g.K = kd.n_in;
      g.a = {kd.inp, kd.n_in, true}; g.b = {pj->v1t[k], kd.n_in, true};
      g.epi = epi_store(P, rp, e->prec);
      g.tag = "lowrank.P";
      TRY(run_gemm(e, g, s));
    }
    // Q = d2^T P  (n_out, rp), K = b: the long-K "small contraction"
    CUDA_TRY(cudaMemsetAsync(Q, 0, kd.n_out * rp * 4, s));
    GemmCall g;
    g.M = kd.n_out; g.N = rp; g.K = b;
    g.a = {kd.d2, kd.ldd, false}; g.b = {Pk, ldp, false};
    g.tag = "lowrank.Q";
    TRY(gemm_accumulate(e, g, Q, rp, 1.f, s));
    if (e->prec == PREC_BF16) TRY(cast_to_compute(e, Q, Qc, kd.n_out * rp, s));
    // grad += alpha * Q V1^T  (n_out, n_in), K = rp: the up-projection
    g = GemmCall();
    g.M = kd.n_out; g.N = kd.n_in; g.K = rp;
    g.a = {Qc, rp, true}; g.b = {pj->v1[k], rp, true};
    g.epi = epi_store(kd.grad, kd.n_in, PREC_F32, gr->alpha_ffn, 1.f);
    g.tag = "lowrank.up_proj";
    TRY(run_gemm(e, g, s));
  }
  return MECEFO_OK;
}

}  // namespace

static int neighbor_backward_impl(mecefo_engine* e, const mecefo_layer_weights* lw, const mecefo_block_cache* c,
                                  const float* dy, const void* dy_c, float* dx, void* dx_c,
                                  const mecefo_layer_grads* gr, const mecefo_projection* pj,
                                  const mecefo_ffn_saved* saved, int64_t tokens, void* wsp, size_t ws_bytes,
                                  void* stream);

int mecefo_backward_block_neighbor(mecefo_engine* e, const mecefo_layer_weights* lw, const mecefo_block_cache* c,
                                   const float* dy, const void* dy_c, float* dx, void* dx_c,
                                   const mecefo_layer_grads* gr, const mecefo_projection* pj, int64_t tokens, void* wsp,
                                   size_t ws_bytes, void* stream) {
  return neighbor_backward_impl(e, lw, c, dy, dy_c, dx, dx_c, gr, pj, nullptr, tokens, wsp, ws_bytes, stream);
}

int mecefo_backward_block_neighbor_main(mecefo_engine* e, const mecefo_layer_weights* lw,
                                        const mecefo_block_cache* c, const float* dy, const void* dy_c, float* dx,
                                        void* dx_c, const mecefo_layer_grads* gr, const mecefo_ffn_saved* saved,
                                        int64_t tokens, void* wsp, size_t ws_bytes, void* stream) {
  if (!saved || !saved->h2 || !saved->act || !saved->dcat)
    return set_err(MECEFO_ERR_CONTRACT, "neighbor_main needs caller buffers for h2, act and dcat");
  if (e && e->prec == PREC_BF16 && !dy_c)
    return set_err(MECEFO_ERR_CONTRACT, "neighbor_main needs the compute-precision dy (it is kept for the deferred Wgrads)");
  return neighbor_backward_impl(e, lw, c, dy, dy_c, dx, dx_c, gr, nullptr, saved, tokens, wsp, ws_bytes, stream);
}

static int neighbor_backward_impl(mecefo_engine* e, const mecefo_layer_weights* lw, const mecefo_block_cache* c,
                                  const float* dy, const void* dy_c, float* dx, void* dx_c,
                                  const mecefo_layer_grads* gr, const mecefo_projection* pj,
                                  const mecefo_ffn_saved* saved, int64_t tokens, void* wsp, size_t ws_bytes,
                                  void* stream) {
  TRY(check_tokens(e, tokens));
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, m = e->d.hidden, f = e->d.ffn;
  Ws ws(wsp, ws_bytes);
  mecefo_layer_grads none{};
  if (!gr) gr = &none;
  if (!dy_c || e->prec == PREC_F32) {
    if (e->prec == PREC_F32) dy_c = dy;
    else {
      void* t;
      TRY(ws.take(b * m * e->ps, &t));
      TRY(cast_to_compute(e, dy, t, b * m, s));
      dy_c = t;
    }
  }
  void *h2, *d_act, *act, *dcat;
  float *inv2, *dh;
  if (saved) {  // deferred Wgrads: the FFN intermediates go to caller buffers
    h2 = saved->h2;
    act = saved->act;
    dcat = saved->dcat;
  } else {
    TRY(ws.take(b * m * e->ps, &h2));
    TRY(ws.take(b * f * e->ps, &act));
    TRY(ws.take(b * 2 * f * e->ps, &dcat));
  }
  TRY(ws.take(b * 4, reinterpret_cast<void**>(&inv2)));
  TRY(ws.take(b * f * e->ps, &d_act));
  TRY(ws.take(b * m * 4, reinterpret_cast<void**>(&dh)));
  // recompute h2 = rmsnorm(x1) (approx.py:128 -> model.py:213)
  TRY(rmsnorm_fwd(e, c->x1, lw->norm_ffn, h2, inv2, b, m, s));
  GemmCall g;
  if (e->prec == PREC_BF16) {
    // d_act = dy Wd, gate|up recomputed = h2 [Wg;Wu]^T, both into TMEM of one
    // kernel; its epilogue forms act and the SwiGLU backward (model.py:214-216,
    // 248-253): gate, up and d_act never touch HBM.
    TRY(swiglu_bwd_dual(e, dy_c, h2, lw->w_down_c, lw->w_gu_c, act, dcat, b, s));
  } else {
    // fp32 mode: d_act = dy Wd (model.py:248; Wd is (m, f) = B MN-major), then the
    // recompute GEMM whose epilogue reads d_act.
    g.M = b; g.N = f; g.K = m;
    g.a = {dy_c, m, true}; g.b = {lw->w_down_c, f, false};
    g.epi = epi_store(d_act, f, e->prec);
    g.tag = "nbr.d_act";
    TRY(run_gemm(e, g, s));
    g = GemmCall();
    g.M = b; g.N = f; g.K = m;
    g.a = {h2, m, true}; g.b = {lw->w_gu_c, m, true};
    g.paired = true; g.pair_off = f;
    Epilogue ep{};
    ep.kind = EPI_SWIGLU_BWD_RECOMP; ep.out = act; ep.ldo = f; ep.out2 = dcat; ep.ldo2 = 2 * f; ep.off2 = f;
    ep.aux = d_act; ep.ldaux = f; ep.act_prec = e->prec;
    g.epi = ep;
    g.tag = "nbr.gu_recompute_swiglu_bwd";
    TRY(run_gemm(e, g, s));
  }
  // d_h2 = [d_gate | d_up] [Wg; Wu]  (model.py:258), K = 2f
  g = GemmCall();
  g.M = b; g.N = m; g.K = 2 * f;
  g.a = {dcat, 2 * f, true}; g.b = {lw->w_gu_c, m, false};
  g.epi = epi_store(dh, m, PREC_F32);
  g.tag = "nbr.d_h2";
  TRY(run_gemm(e, g, s));
  // dx = dy + rmsnorm_bwd(x1, ...)   (model.py:259, approx.py:130)
  TRY(rmsnorm_bwd(e, ws, c->x1, lw->norm_ffn, inv2, dh, dy, dx, dx_c, gr->norm_ffn, gr->alpha_ffn, b, m, s));
  // FFN weight gradients
  if (saved) return MECEFO_OK;  // deferred: mecefo_lowrank_wgrads_batched
  if (pj) {
    TRY(lowrank_ffn_wgrads(e, ws, pj, dy_c, h2, act, dcat, gr, b, s));
  } else {
    if (gr->down) {  // g_down = dy^T act (model.py:247)
      g = GemmCall();
      g.M = m; g.N = f; g.K = b;
      g.a = {dy_c, m, false}; g.b = {act, f, false};
      g.tag = "nbr.wgrad_down";
      TRY(gemm_accumulate(e, g, gr->down, f, gr->alpha_ffn, s));
    }
    if (gr->gu) {  // [g_gate; g_up] = [d_gate | d_up]^T h2 (model.py:255-256)
      g = GemmCall();
      g.M = 2 * f; g.N = m; g.K = b;
      g.a = {dcat, 2 * f, false}; g.b = {h2, m, false};
      g.tag = "nbr.wgrad_gu";
      TRY(gemm_accumulate(e, g, gr->gu, m, gr->alpha_ffn, s));
    }
  }
  return MECEFO_OK;
}

int mecefo_backward_block_exact(mecefo_engine* e, const mecefo_layer_weights* lw, const mecefo_block_cache* c,
                                const float* dy, const void* dy_c, float* dx, void* dx_c,
                                const mecefo_layer_grads* gr, int64_t tokens, void* wsp, size_t ws_bytes,
                                void* stream) {
  TRY(check_tokens(e, tokens));
  if (!c->h1 || !c->qkv || !c->ctx || !c->lse || !c->h2 || !c->inv1 || !c->inv2 || !c->gu || !c->act)
    return set_err(MECEFO_ERR_CONTRACT, "exact backward requires a full activation cache");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, m = e->d.hidden, f = e->d.ffn, H = e->d.heads;
  Ws ws(wsp, ws_bytes);
  mecefo_layer_grads none{};
  if (!gr) gr = &none;
  if (!dy_c || e->prec == PREC_F32) {
    if (e->prec == PREC_F32) dy_c = dy;
    else {
      void* t;
      TRY(ws.take(b * m * e->ps, &t));
      TRY(cast_to_compute(e, dy, t, b * m, s));
      dy_c = t;
    }
  }
  void *dcat, *dx1_c, *dctx, *dqkv;
  float *dh, *dx1, *dsum;
  TRY(ws.take(b * 2 * f * e->ps, &dcat));
  TRY(ws.take(b * m * 4, reinterpret_cast<void**>(&dh)));
  TRY(ws.take(b * m * 4, reinterpret_cast<void**>(&dx1)));
  TRY(ws.take(b * m * e->ps, &dx1_c));
  TRY(ws.take(b * m * e->ps, &dctx));
  TRY(ws.take(b * 3 * m * e->ps, &dqkv));
  TRY(ws.take(b * H * 4, reinterpret_cast<void**>(&dsum)));
  // ---- FFN sub-block (model.py:232-261) ----
  GemmCall g;
  if (e->prec == PREC_BF16) {
    TRY(swiglu_bwd_dual(e, dy_c, c->h2, lw->w_down_c, lw->w_gu_c, nullptr, dcat, b, s));
  } else {
    g.M = b; g.N = f; g.K = m;
    g.a = {dy_c, m, true}; g.b = {lw->w_down_c, f, false};
    Epilogue ep{};
    ep.kind = EPI_SWIGLU_BWD_CACHED; ep.out2 = dcat; ep.ldo2 = 2 * f; ep.off2 = f;
    ep.aux = c->gu; ep.ldaux = 2 * f; ep.offaux = f; ep.act_prec = e->prec;
    g.epi = ep;
    g.tag = "exact.d_act_swiglu_bwd";
    TRY(run_gemm(e, g, s));
  }
  g = GemmCall();
  g.M = b; g.N = m; g.K = 2 * f;
  g.a = {dcat, 2 * f, true}; g.b = {lw->w_gu_c, m, false};
  g.epi = epi_store(dh, m, PREC_F32);
  g.tag = "exact.d_h2";
  TRY(run_gemm(e, g, s));
  TRY(rmsnorm_bwd(e, ws, c->x1, lw->norm_ffn, c->inv2, dh, dy, dx1, dx1_c, gr->norm_ffn, gr->alpha_ffn, b, m, s));
  if (gr->down) {
    g = GemmCall();
    g.M = m; g.N = f; g.K = b;
    g.a = {dy_c, m, false}; g.b = {c->act, f, false};
    g.tag = "exact.wgrad_down";
    TRY(gemm_accumulate(e, g, gr->down, f, gr->alpha_ffn, s));
  }
  if (gr->gu) {
    g = GemmCall();
    g.M = 2 * f; g.N = m; g.K = b;
    g.a = {dcat, 2 * f, false}; g.b = {c->h2, m, false};
    g.tag = "exact.wgrad_gu";
    TRY(gemm_accumulate(e, g, gr->gu, m, gr->alpha_ffn, s));
  }
  // ---- attention sub-block (model.py:336-368) ----
  g = GemmCall();  // d_ctx = dx1 Wo
  g.M = b; g.N = m; g.K = m;
  g.a = {dx1_c, m, true}; g.b = {lw->w_o_c, m, false};
  g.epi = epi_store(dctx, m, e->prec);
  g.tag = "exact.d_ctx";
  TRY(run_gemm(e, g, s));
  if (gr->o) {  // g_o = dx1^T ctx
    g = GemmCall();
    g.M = m; g.N = m; g.K = b;
    g.a = {dx1_c, m, false}; g.b = {c->ctx, m, false};
    g.tag = "exact.wgrad_o";
    TRY(gemm_accumulate(e, g, gr->o, m, gr->alpha_mha, s));
  }
  AttnDev a = attn_args(e);
  a.qkv = c->qkv; a.ld_qkv = 3 * m; a.ctx = c->ctx; a.ld_ctx = m; a.dctx = dctx; a.dqkv = dqkv;
  a.lse = c->lse; a.dsum = dsum;
  TRY(attention(e, true, a, b, s));
  g = GemmCall();  // d_h1 = d_qkv [Wq; Wk; Wv], K = 3m
  g.M = b; g.N = m; g.K = 3 * m;
  g.a = {dqkv, 3 * m, true}; g.b = {lw->w_qkv_c, m, false};
  g.epi = epi_store(dh, m, PREC_F32);
  g.tag = "exact.d_h1";
  TRY(run_gemm(e, g, s));
  if (gr->qkv) {  // [g_q; g_k; g_v] = d_qkv^T h1
    g = GemmCall();
    g.M = 3 * m; g.N = m; g.K = b;
    g.a = {dqkv, 3 * m, false}; g.b = {c->h1, m, false};
    g.tag = "exact.wgrad_qkv";
    TRY(gemm_accumulate(e, g, gr->qkv, m, gr->alpha_mha, s));
  }
  // dx = dx1 + rmsnorm_bwd(x, g_mha, inv1, d_h1)   (model.py:433-434)
  TRY(rmsnorm_bwd(e, ws, c->x, lw->norm_mha, c->inv1, dh, dx1, dx, dx_c, gr->norm_mha, gr->alpha_mha, b, m, s));
  return MECEFO_OK;
}

int mecefo_recompute_ffn(mecefo_engine* e, const mecefo_layer_weights* lw, const float* x1, int64_t tokens, void* h2,
                         float* inv2, void* gate, void* up, void* act, float* down, void* wsp, size_t ws_bytes,
                         void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, m = e->d.hidden, f = e->d.ffn;
  Ws ws(wsp, ws_bytes);
  if (!h2) TRY(ws.take(b * m * e->ps, &h2));
  if (!inv2) TRY(ws.take(b * 4, reinterpret_cast<void**>(&inv2)));
  if (!act && down) TRY(ws.take(b * f * e->ps, &act));
  void* gu = nullptr;
  if (gate || up) TRY(ws.take(b * 2 * f * e->ps, &gu));
  TRY(rmsnorm_fwd(e, x1, lw->norm_ffn, h2, inv2, b, m, s));
  GemmCall g;
  g.M = b; g.N = f; g.K = m;
  g.a = {h2, m, true}; g.b = {lw->w_gu_c, m, true};
  g.paired = true; g.pair_off = f;
  Epilogue ep{};
  ep.kind = EPI_SWIGLU_FWD; ep.out = act; ep.ldo = f; ep.out2 = gu; ep.ldo2 = 2 * f; ep.off2 = f; ep.act_prec = e->prec;
  g.epi = ep;
  g.tag = "recompute.gu";
  TRY(run_gemm(e, g, s));
  if (gu) {
    if (gate) CUDA_TRY(cudaMemcpy2DAsync(gate, f * e->ps, gu, 2 * f * e->ps, f * e->ps, b, cudaMemcpyDeviceToDevice, s));
    if (up)
      CUDA_TRY(cudaMemcpy2DAsync(up, f * e->ps, reinterpret_cast<uint8_t*>(gu) + f * e->ps, 2 * f * e->ps, f * e->ps,
                                 b, cudaMemcpyDeviceToDevice, s));
  }
  if (down) {
    g = GemmCall();
    g.M = b; g.N = m; g.K = f;
    g.a = {act, f, true}; g.b = {lw->w_down_c, f, true};
    g.epi = epi_store(down, m, PREC_F32);
    g.tag = "recompute.down";
    TRY(run_gemm(e, g, s));
  }
  return MECEFO_OK;
}

int mecefo_lowrank_wgrad(mecefo_engine* e, const void* g_y, const void* x, const void* v1, float* out, int64_t n_out,
                         int64_t n_in, int64_t batch, int64_t rank, float alpha, void* wsp, size_t ws_bytes,
                         void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (n_out < 1 || n_in < 1 || batch < 1 || rank < 1) return set_err(MECEFO_ERR_CONTRACT, "empty lowrank_wgrad operand");
  Ws ws(wsp, ws_bytes);
  void* P;
  float* Q;
  void* Qc;
  TRY(ws.take(batch * rank * e->ps, &P));
  TRY(ws.take(n_out * rank * 4, reinterpret_cast<void**>(&Q)));
  if (e->prec == PREC_BF16) TRY(ws.take(n_out * rank * e->ps, &Qc));
  else Qc = Q;
  // P = x^T V1 (batch, rank): A(i=b, k=in) = x[k, i] (MN-major), B(n=r, k=in) = v1[k, n] (MN-major)
  GemmCall g;
  g.M = batch; g.N = rank; g.K = n_in;
  g.a = {x, batch, false}; g.b = {v1, rank, false};
  g.epi = epi_store(P, rank, e->prec);
  g.tag = "lowrank_api.P";
  TRY(run_gemm(e, g, s));
  // Q = g_y P (n_out, rank): A = g_y K-major (ld batch), B(n=r, k=b) = P[k, n] MN-major
  CUDA_TRY(cudaMemsetAsync(Q, 0, n_out * rank * 4, s));
  g = GemmCall();
  g.M = n_out; g.N = rank; g.K = batch;
  g.a = {g_y, batch, true}; g.b = {P, rank, false};
  g.tag = "lowrank_api.Q";
  TRY(gemm_accumulate(e, g, Q, rank, 1.f, s));
  if (e->prec == PREC_BF16) TRY(cast_to_compute(e, Q, Qc, n_out * rank, s));
  // out += alpha Q V1^T: B(n=in, k=r) = v1[n, k] K-major
  g = GemmCall();
  g.M = n_out; g.N = n_in; g.K = rank;
  g.a = {Qc, rank, true}; g.b = {v1, rank, true};
  g.epi = epi_store(out, n_in, PREC_F32, alpha, 1.f);
  g.tag = "lowrank_api.up_proj";
  return run_gemm(e, g, s);
}

int mecefo_embedding_forward(mecefo_engine* e, const int64_t* tokens, const float* emb, float* x, int64_t n,
                             void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (n <= 0) return MECEFO_OK;
  CUDA_TRY(pdl_launch(embedding_fwd_kernel, dim3((unsigned)n), dim3(128), 0, s, tokens, emb, x, (int)n, (int)e->d.hidden,
                      (int)e->d.vocab, e->status));
  return check_launch("embedding_fwd_kernel");
}

int mecefo_head_logits(mecefo_engine* e, const float* x_last, const float* final_norm, const void* unemb_c,
                       int64_t tokens, void* xf, float* inv_f, void* logits, void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, m = e->d.hidden, V = e->d.vocab;
  TRY(rmsnorm_fwd(e, x_last, final_norm, xf, inv_f, b, m, s));
  GemmCall g;
  g.M = b; g.N = V; g.K = m;
  g.a = {xf, m, true}; g.b = {unemb_c, m, true};
  g.epi = epi_store(logits, V, e->prec);
  g.tag = "head.logits";
  return run_gemm(e, g, s);
}

int mecefo_cross_entropy_grouped(mecefo_engine* e, void* logits, const int64_t* targets, int64_t tokens,
                                 int64_t group_rows, float* loss, void* wsp, size_t ws_bytes, void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, V = e->d.vocab;
  if (group_rows <= 0 || tokens % group_rows != 0)
    return set_err(MECEFO_ERR_CONTRACT, "%lld rows do not split into groups of %lld", (long long)tokens,
                   (long long)group_rows);
  const float inv_n = 1.f / (float)group_rows;
  Ws ws(wsp, ws_bytes);
  float* rows;
  int* bad = e->status;  // bit MECEFO_STATUS_BAD_TARGET; the row contributes loss 0 and zero dlogits
  TRY(ws.take(b * 4, reinterpret_cast<void**>(&rows)));
  ProfScope prof("cross_entropy", 0.0, 2.0 * b * V * e->ps, s);
  // bf16: a row per CTA staged in shared memory (read once, written once),
  // several CTAs per SM; f16x2 exps (cross_entropy_smem_kernel, ce.cuh).
  // Measured at 16384 x 32000: 0.44 ms vs 0.53 ms for the warp-per-row kernel.
  const size_t rb_al = ((size_t)V * 2 + 127) & ~size_t(127);
  const size_t ce_smem = rb_al + 16 + 8 * 32 + 128;
  if (e->prec == PREC_BF16 && V % 8 == 0 && ce_smem <= 200 * 1024) {
    TRY(ensure_smem((const void*)cross_entropy_smem_kernel<1, 256>, 200 * 1024));
    const int per_sm = std::max(1, (int)((220 * 1024) / (ce_smem + 1024)));
    CUDA_TRY(pdl_launch(cross_entropy_smem_kernel<1, 256>, dim3((unsigned)std::min<int64_t>(b, kNumSMs * per_sm)),
                        dim3(256), ce_smem, s, reinterpret_cast<__nv_bfloat16*>(logits), V, targets, rows, (int)b,
                        (int)V, inv_n, bad));
    TRY(check_launch("cross_entropy_smem_kernel"));
  } else if (e->prec == PREC_BF16 && V % 8 == 0) {
    CUDA_TRY(pdl_launch(cross_entropy_warp_kernel, dim3((unsigned)((b + 7) / 8)), dim3(256), 0, s,
                        reinterpret_cast<__nv_bfloat16*>(logits), V, targets, rows, (int)b, (int)V, inv_n, bad));
    TRY(check_launch("cross_entropy_warp_kernel"));
  } else {
    CUDA_TRY(pdl_launch(cross_entropy_kernel, dim3((unsigned)b), dim3(512), 0, s, logits, V, targets, rows, (int)b,
                        (int)V, inv_n, e->prec, bad));
    TRY(check_launch("cross_entropy_kernel"));
  }
  CUDA_TRY(pdl_launch(mean_kernel, dim3((unsigned)(tokens / group_rows)), dim3(1024), 0, s, rows, (int)group_rows,
                      loss));
  return check_launch("mean_kernel");
}

int mecefo_cross_entropy(mecefo_engine* e, void* logits, const int64_t* targets, int64_t tokens, float* loss,
                         void* wsp, size_t ws_bytes, void* stream) {
  return mecefo_cross_entropy_grouped(e, logits, targets, tokens, tokens, loss, wsp, ws_bytes, stream);
}

int mecefo_head_forward_loss_grouped(mecefo_engine* e, const float* x_last, const float* final_norm,
                                     const void* unemb_c, const int64_t* targets, int64_t tokens, int64_t group_rows,
                                     void* xf, float* inv_f, void* logits, float* loss, void* wsp, size_t ws_bytes,
                                     void* stream) {
  // (Measured: folding softmax statistics into the logits GEMM epilogue made
  // that GEMM epilogue-bound, 1.17 -> 0.57 PFLOP/s; chunking the rows so each
  // chunk's logits stay L2-resident for the CE pass lost 4-13% (small-M
  // GEMMs and an under-occupied CE per chunk). One logits GEMM + one
  // warp-per-row CE pass is faster overall.)
  TRY(mecefo_head_logits(e, x_last, final_norm, unemb_c, tokens, xf, inv_f, logits, stream));
  return mecefo_cross_entropy_grouped(e, logits, targets, tokens, group_rows, loss, wsp, ws_bytes, stream);
}

int mecefo_head_forward_loss(mecefo_engine* e, const float* x_last, const float* final_norm, const void* unemb_c,
                             const int64_t* targets, int64_t tokens, void* xf, float* inv_f, void* logits, float* loss,
                             void* wsp, size_t ws_bytes, void* stream) {
  TRY(mecefo_head_logits(e, x_last, final_norm, unemb_c, tokens, xf, inv_f, logits, stream));
  return mecefo_cross_entropy(e, logits, targets, tokens, loss, wsp, ws_bytes, stream);
}

int mecefo_head_backward(mecefo_engine* e, const float* x_last, const float* final_norm, const float* inv_f,
                         const void* xf, const void* dlogits, const void* unemb_c, float* dx, void* dx_c,
                         float* g_final, float* g_unemb, float alpha, int64_t tokens, void* wsp, size_t ws_bytes,
                         void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, m = e->d.hidden, V = e->d.vocab;
  Ws ws(wsp, ws_bytes);
  float* dxf;
  TRY(ws.take(b * m * 4, reinterpret_cast<void**>(&dxf)));
  if (g_unemb) {  // g_unemb = dlogits^T xf  (model.py:480)
    GemmCall g;
    g.M = V; g.N = m; g.K = b;
    g.a = {dlogits, V, false}; g.b = {xf, m, false};
    g.tag = "head.g_unemb";
    TRY(gemm_accumulate(e, g, g_unemb, m, alpha, s));
  }
  GemmCall g;  // d_xf = dlogits Wun  (model.py:481)
  g.M = b; g.N = m; g.K = V;
  g.a = {dlogits, V, true}; g.b = {unemb_c, m, false};
  g.epi = epi_store(dxf, m, PREC_F32);
  g.tag = "head.d_xf";
  TRY(run_gemm(e, g, s));
  return rmsnorm_bwd(e, ws, x_last, final_norm, inv_f, dxf, nullptr, dx, dx_c, g_final, alpha, b, m, s);
}

int mecefo_embedding_backward(mecefo_engine* e, const int64_t* tokens, const float* dx0, float* g_emb, float alpha,
                              int64_t n, void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (n <= 0) return MECEFO_OK;
  CUDA_TRY(pdl_launch(embedding_bwd_kernel, dim3((unsigned)n), dim3(128), 0, s, tokens, dx0, g_emb, (int)n, (int)e->d.hidden, alpha,
                      (int)e->d.vocab));
  return check_launch("embedding_bwd_kernel");
}

int mecefo_scale_accumulate(const float* src, float* out, int64_t n, float alpha, float beta, void* stream) {
  if (n <= 0) return MECEFO_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 8 * kNumSMs);
  CUDA_TRY(pdl_launch(axpby_kernel, dim3((unsigned)blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), src, out, n, alpha, beta));
  return check_launch("axpby_kernel");
}

int mecefo_cast(mecefo_engine* e, const float* src, void* dst, int64_t n, void* stream) {
  if (n <= 0) return MECEFO_OK;
  return cast_to_compute(e, src, dst, n, reinterpret_cast<cudaStream_t>(stream));
}

int mecefo_cast_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n <= 0) return MECEFO_OK;
  auto s = reinterpret_cast<cudaStream_t>(stream);
  ProfScope prof("grad.cast_bf16", 0.0, 6.0 * n, s);
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 8 * kNumSMs);
  CUDA_TRY(pdl_launch(cast_f32_kernel, dim3((unsigned)blocks), dim3(256), 0, s, src, dst, n, (int)PREC_BF16));
  return check_launch("cast_f32_kernel");
}

int mecefo_widen_bf16(const void* src, float* dst, int64_t n, void* stream) {
  if (n <= 0) return MECEFO_OK;
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return set_err(MECEFO_ERR_CONTRACT, "widen_bf16 needs 16-byte aligned buffers");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  ProfScope prof("grad.widen_bf16", 0.0, 6.0 * n, s);
  const int64_t blocks = std::min<int64_t>((n / 8 + 255) / 256 + 1, 8 * kNumSMs);
  CUDA_TRY(pdl_launch(widen_bf16_kernel, dim3((unsigned)blocks), dim3(256), 0, s,
                      reinterpret_cast<const __nv_bfloat16*>(src), dst, n));
  return check_launch("widen_bf16_kernel");
}

int mecefo_nonfinite(const float* v, int64_t n, int32_t* flag, void* stream) {
  if (n <= 0) return MECEFO_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 8 * kNumSMs);
  CUDA_TRY(pdl_launch(nonfinite_kernel, dim3((unsigned)blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), v, n, flag));
  return check_launch("nonfinite_kernel");
}

int mecefo_adamw_step(mecefo_engine* e, const mecefo_adam_segment* segs, int32_t nseg, int64_t total_numel, float* w,
                      const float* grad, float* m1, float* m2, void* shadow, float beta1, float beta2, float eps,
                      void* stream) {
  if (nseg <= 0) return MECEFO_OK;
  static_assert(sizeof(mecefo_adam_segment) == sizeof(AdamSeg), "segment layout");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  // read g, m, v, w; write m, v, w (+ the compute-precision shadow)
  ProfScope prof("adamw", 0.0, (double)total_numel * (28.0 + (shadow ? (e ? e->ps : 4) : 0)), s);
  const unsigned grid = 8 * kNumSMs;  // grid-stride over the concatenated active segments
  CUDA_TRY(pdl_launch(adamw_kernel, dim3(grid), dim3(256), (nseg + 1) * sizeof(int64_t), s, reinterpret_cast<const AdamSeg*>(segs), nseg, w, grad,
                                                               m1, m2, shadow, e ? e->prec : PREC_F32, beta1, beta2,
                                                               eps, e ? e->status : nullptr));
  return check_launch("adamw_kernel");
}

int mecefo_gemm(mecefo_engine* e, int64_t M, int64_t N, int64_t K, const void* a, int64_t lda, int32_t a_kmajor,
                const void* b, int64_t ldb, int32_t b_kmajor, float* c, int64_t ldc, float alpha, float beta,
                void* stream) {
  GemmCall g;
  g.M = M; g.N = N; g.K = K;
  g.a = {a, lda, a_kmajor != 0}; g.b = {b, ldb, b_kmajor != 0};
  g.epi = epi_store(c, ldc, PREC_F32, alpha, beta);
  return run_gemm(e, g, reinterpret_cast<cudaStream_t>(stream));
}

namespace {
struct SubspacePlan {
  size_t off_b, off_z, off_g, off_m, off_ur, off_th, off_ks, off_jobs, off_scr, total;
  size_t ritz_bytes, chol_bytes;  // per-matrix scratch (smem or global)
  int kmax, rmax;
  bool smem;
};
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int SUB_PHASES = 6;
constexpr int SUB_GRAM_SPLIT = 4;  // split-K of the long-K Gram products (partials summed by their consumers)
constexpr size_t SUB_SMEM_MAX = 220 * 1024;

SubspacePlan subspace_plan(const mecefo_subspace_job* jobs, int count) {
  SubspacePlan p{};
  size_t o = 0, zb = 0, bb = 0;
  p.kmax = 1;
  p.rmax = 1;
  for (int i = 0; i < count; ++i) {
    bb += al256((size_t)jobs[i].cols * jobs[i].cols * 4);
    zb += al256((size_t)jobs[i].cols * jobs[i].k * 4);
    p.kmax = std::max(p.kmax, (int)jobs[i].k);
    p.rmax = std::max(p.rmax, (int)jobs[i].r);
  }
  const size_t kk = (size_t)p.kmax * p.kmax;
  const size_t kl = (size_t)p.kmax * (p.kmax | 1);  // odd row stride (subspace.cuh sub_ld)
  p.chol_bytes = (kl + p.kmax) * 8;
  p.ritz_bytes = kl * 8 + kl * 4;
  p.off_b = o; o += bb;
  p.off_z = o; o += zb;
  p.off_g = o; o += al256(SUB_GRAM_SPLIT * count * kk * 4);
  p.off_m = o; o += al256(count * kk * 4);
  p.off_ur = o; o += al256(count * (size_t)p.kmax * p.rmax * 4);
  p.off_th = o; o += al256(count * (size_t)p.rmax * 4);
  p.off_ks = o; o += al256(2 * count * 4);
  p.off_jobs = o; o += al256(sizeof(SubGemmJob) * count * SUB_PHASES);
  p.smem = std::max(p.chol_bytes, p.ritz_bytes) <= SUB_SMEM_MAX;
  p.off_scr = o; if (!p.smem) o += al256(count * std::max(p.chol_bytes, p.ritz_bytes));
  p.total = o;
  return p;
}

SubGemmJob sub_job(const float* a, int64_t lda, bool a_kmajor, const float* b, int64_t ldb, float* c, int64_t ldc,
                   int M, int N, int K) {
  SubGemmJob j{};
  j.a = a; j.lda = lda; j.a_kmajor = a_kmajor ? 1 : 0;
  j.b = b; j.ldb = ldb; j.c = c; j.ldc = ldc;
  j.M = M; j.N = N; j.K = K;
  j.tiles_n = (N + SG_TN - 1) / SG_TN;
  j.tiles_mn = ((M + SG_TM - 1) / SG_TM) * j.tiles_n;
  j.ksplit = 1;
  j.kchunk = K;
  j.c_split = 0;
  auto al = [](const void* q, int64_t ld) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0 && (ld & 3) == 0; };
  j.vec = al(a, lda) && al(b, ldb) ? 1 : 0;
  return j;
}
}  // namespace

namespace {
bool lowrank_grouped_ok(const mecefo_engine* e, const mecefo_lowrank_job* jobs, int count) {
  if (e->prec != PREC_BF16) return false;
  const int64_t rp = jobs[0].proj ? jobs[0].proj->rank_pad : 0;
  if (rp <= 0 || rp % TC_BM != 0) return false;
  for (int i = 0; i < count; ++i) {
    const mecefo_projection* pj = jobs[i].proj;
    if (!pj || pj->rank_pad != rp || !pj->v1_gu || !pj->v1t_gu || !pj->v1[2] || !pj->v1t[2]) return false;
    if (!jobs[i].grad_gu || !jobs[i].grad_down || !jobs[i].dy_c) return false;
  }
  return true;
}
size_t lowrank_group_bytes(const mecefo_engine* e, int64_t b, int64_t rp) {
  const int64_t m = e->d.hidden, f = e->d.ffn, ps = e->ps;
  auto al = [](int64_t x) { return (size_t)((x + 255) & ~int64_t(255)); };
  return al(b * 2 * rp * ps) + al(2 * rp * f * 4) + al(2 * rp * 2 * f * ps) + al(rp * m * 4) + al(rp * m * ps);
}
}  // namespace

size_t mecefo_lowrank_batched_workspace_bytes(const mecefo_engine* e, int64_t tokens, int32_t rank_pad,
                                             int32_t count) {
  if (!e || tokens < 1 || rank_pad < 1 || count < 1) return 0;
  const int per = std::min<int>(count, kMaxGroups);
  // grouped path: per-group scratch for one chunk; fallback: one neighbour chain
  return std::max(lowrank_group_bytes(e, tokens, rank_pad) * per + 4096,
                  mecefo_workspace_bytes(e, tokens, rank_pad));
}

int mecefo_lowrank_wgrads_batched(mecefo_engine* e, const mecefo_lowrank_job* jobs, int32_t count, int64_t tokens,
                                  void* wsp, size_t ws_bytes, void* stream) {
  TRY(check_tokens(e, tokens));
  if (!jobs || count < 0) return set_err(MECEFO_ERR_CONTRACT, "null job list");
  if (count == 0) return MECEFO_OK;
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t b = tokens, m = e->d.hidden, f = e->d.ffn, ps = e->ps;
  for (int i = 0; i < count; ++i)
    if (!jobs[i].proj || !jobs[i].saved.h2 || !jobs[i].saved.act || !jobs[i].saved.dcat || !jobs[i].dy_c)
      return set_err(MECEFO_ERR_CONTRACT, "lowrank job %d: missing projection, dy or saved intermediates", i);
  if (!lowrank_grouped_ok(e, jobs, count)) {  // general path: one neighbour Wgrad chain per job
    for (int i = 0; i < count; ++i) {
      Ws ws(wsp, ws_bytes);
      mecefo_layer_grads gr{};
      gr.gu = jobs[i].grad_gu;
      gr.down = jobs[i].grad_down;
      gr.alpha_ffn = jobs[i].alpha;
      TRY(lowrank_ffn_wgrads(e, ws, jobs[i].proj, jobs[i].dy_c, jobs[i].saved.h2, jobs[i].saved.act,
                             jobs[i].saved.dcat, &gr, b, s));
    }
    return MECEFO_OK;
  }
  const int64_t rp = jobs[0].proj->rank_pad;
  // Grouped chain (the transposed low-rank path of lowrank_ffn_wgrads, one
  // launch per product for up to 8 lean layers): the per-layer products are
  // too small to fill the GPU alone (88-144 CTAs, 8-22 k-blocks).
  for (int j0 = 0; j0 < count;) {
    int n = 1;
    while (j0 + n < count && n < kMaxGroups && jobs[j0 + n].alpha == jobs[j0].alpha) ++n;
    const mecefo_lowrank_job* J = jobs + j0;
    const float alpha = J[0].alpha;
    Ws ws(wsp, ws_bytes);
    void* P;
    float *QT, *QTd;
    void *QTc, *QTdc;
    TRY(ws.take(n * b * 2 * rp * ps, &P));
    TRY(ws.take(n * 2 * rp * f * 4, reinterpret_cast<void**>(&QT)));
    TRY(ws.take(n * 2 * rp * 2 * f * ps, &QTc));
    TRY(ws.take(n * rp * m * 4, reinterpret_cast<void**>(&QTd)));
    TRY(ws.take(n * rp * m * ps, &QTdc));
    auto Pq = [&](int q) { return reinterpret_cast<uint8_t*>(P) + (size_t)q * b * 2 * rp * ps; };
    GemmCall g;
    // [P_g | P_u] = h2 [V1_g | V1_u]
    g.M = b; g.N = 2 * rp; g.K = m;
    g.a = {J[0].saved.h2, m, true}; g.b = {J[0].proj->v1t_gu, m, true};
    g.epi = epi_store(Pq(0), 2 * rp, e->prec);
    g.groups = n;
    for (int q = 0; q < n; ++q) { g.ga[q] = J[q].saved.h2; g.gb[q] = J[q].proj->v1t_gu; g.go[q] = Pq(q); }
    g.tag = "lowrank.P";
    TRY(run_gemm(e, g, s));
    // [Q_g^T ; Q_u^T] = [P_g | P_u]^T [d_gate | d_up], block-diagonal
    CUDA_TRY(cudaMemsetAsync(QT, 0, n * 2 * rp * f * 4, s));
    g = GemmCall();
    g.M = 2 * rp; g.N = f; g.K = b;
    g.a = {Pq(0), 2 * rp, false}; g.b = {J[0].saved.dcat, 2 * f, false};
    g.b_diag_off = f;
    g.b_diag_div = (int)(rp / TC_BM);  // rows [0, rp) meet d_gate, [rp, 2rp) d_up
    g.groups = n;
    for (int q = 0; q < n; ++q) { g.ga[q] = Pq(q); g.gb[q] = J[q].saved.dcat; g.go[q] = QT + (size_t)q * 2 * rp * f; }
    g.tag = "lowrank.Q";
    TRY(gemm_accumulate(e, g, QT, f, 1.f, s));
    {
      const int64_t nel = (int64_t)n * 2 * rp * 2 * f;
      ProfScope prof("lowrank.cast", 0.0, 6.0 * nel / 2, s);
      CUDA_TRY(pdl_launch(cast_blockdiag_t_kernel, dim3((unsigned)std::min<int64_t>((nel + 255) / 256, 8 * kNumSMs)),
                          dim3(256), 0, s, (const float*)QT, (__nv_bfloat16*)QTc, (int)rp, (int)f, (int64_t)n));
      TRY(check_launch("cast_blockdiag_t_kernel"));
    }
    // [G_g ; G_u] += alpha blockdiag(Q) [V1_g | V1_u]^T
    g = GemmCall();
    g.M = 2 * f; g.N = m; g.K = 2 * rp;
    g.a = {QTc, 2 * f, false}; g.b = {J[0].proj->v1_gu, 2 * rp, true};
    g.epi = epi_store(J[0].grad_gu, m, PREC_F32, alpha, 1.f);
    g.groups = n;
    for (int q = 0; q < n; ++q) {
      g.ga[q] = reinterpret_cast<uint8_t*>(QTc) + (size_t)q * 2 * rp * 2 * f * ps;
      g.gb[q] = J[q].proj->v1_gu;
      g.go[q] = J[q].grad_gu;
    }
    g.tag = "lowrank.up_proj";
    TRY(run_gemm(e, g, s));
    // down: P_d = act V1_d (into the P buffers), Q_d^T = P_d^T dy, G_d += alpha Q_d V1_d^T
    g = GemmCall();
    g.M = b; g.N = rp; g.K = f;
    g.a = {J[0].saved.act, f, true}; g.b = {J[0].proj->v1t[2], f, true};
    g.epi = epi_store(Pq(0), rp, e->prec);
    g.groups = n;
    for (int q = 0; q < n; ++q) { g.ga[q] = J[q].saved.act; g.gb[q] = J[q].proj->v1t[2]; g.go[q] = Pq(q); }
    g.tag = "lowrank.P";
    TRY(run_gemm(e, g, s));
    CUDA_TRY(cudaMemsetAsync(QTd, 0, n * rp * m * 4, s));
    g = GemmCall();
    g.M = rp; g.N = m; g.K = b;
    g.a = {Pq(0), rp, false}; g.b = {J[0].dy_c, m, false};
    g.groups = n;
    for (int q = 0; q < n; ++q) { g.ga[q] = Pq(q); g.gb[q] = J[q].dy_c; g.go[q] = QTd + (size_t)q * rp * m; }
    g.tag = "lowrank.Q";
    TRY(gemm_accumulate(e, g, QTd, m, 1.f, s));
    TRY(cast_to_compute(e, QTd, QTdc, n * rp * m, s));
    g = GemmCall();
    g.M = m; g.N = f; g.K = rp;
    g.a = {QTdc, m, false}; g.b = {J[0].proj->v1[2], rp, true};
    g.epi = epi_store(J[0].grad_down, f, PREC_F32, alpha, 1.f);
    g.groups = n;
    for (int q = 0; q < n; ++q) {
      g.ga[q] = reinterpret_cast<uint8_t*>(QTdc) + (size_t)q * rp * m * ps;
      g.gb[q] = J[q].proj->v1[2];
      g.go[q] = J[q].grad_down;
    }
    g.tag = "lowrank.up_proj";
    TRY(run_gemm(e, g, s));
    j0 += n;
  }
  return MECEFO_OK;
}

size_t mecefo_subspace_workspace_bytes(const mecefo_subspace_job* jobs, int32_t count) {
  if (!jobs || count < 1) return 0;
  return subspace_plan(jobs, count).total;
}

int mecefo_subspace_iteration_batched(mecefo_engine* e, const mecefo_subspace_job* jobs, int32_t count,
                                      int32_t iterations, void* workspace, size_t workspace_bytes, void* stream) {
  if (!e) return set_err(MECEFO_ERR_CONTRACT, "null engine");
  if (!jobs || count < 1) return set_err(MECEFO_ERR_CONTRACT, "subspace iteration needs >= 1 job");
  if (iterations < 1) return set_err(MECEFO_ERR_CONTRACT, "iterations must be >= 1, got %d", iterations);
  for (int i = 0; i < count; ++i) {
    const mecefo_subspace_job& j = jobs[i];
    if (!j.w || !j.v || !j.v1) return set_err(MECEFO_ERR_CONTRACT, "job %d: null pointer", i);
    if (j.rows < 1 || j.cols < 1 || j.ldw < j.cols)
      return set_err(MECEFO_ERR_CONTRACT, "job %d: bad shape %lldx%lld ld %lld", i, (long long)j.rows,
                     (long long)j.cols, (long long)j.ldw);
    if (j.r < 1 || j.k < j.r || j.k > j.cols || j.k > 512)
      return set_err(MECEFO_ERR_CONTRACT, "job %d: need 1 <= r=%d <= k=%d <= min(cols=%lld, 512)", i, j.r, j.k,
                     (long long)j.cols);
    if (j.cols > 46340 || j.rows > (int64_t)1 << 30) return set_err(MECEFO_ERR_CONTRACT, "job %d: too large", i);
  }
  const SubspacePlan p = subspace_plan(jobs, count);
  if (!workspace || workspace_bytes < p.total)
    return set_err(MECEFO_ERR_CONTRACT, "subspace workspace too small: %zu < %zu", workspace_bytes, p.total);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  const int kmax = p.kmax, rmax = p.rmax;
  const size_t kk = (size_t)kmax * kmax;
  float* G = reinterpret_cast<float*>(ws + p.off_g);
  float* Mm = reinterpret_cast<float*>(ws + p.off_m);
  float* Ur = reinterpret_cast<float*>(ws + p.off_ur);
  float* Th = reinterpret_cast<float*>(ws + p.off_th);
  // phases: 0 B = W^T W, 1 Z = B V, 2 G = Z^T Z, 3 V = Z M, 4 S = V^T Z (into G), 5 V1 = V Ur
  std::vector<SubGemmJob> hj((size_t)count * SUB_PHASES);
  std::vector<int> hk(2 * count);
  int tiles[SUB_PHASES] = {};
  size_t ob = p.off_b, oz = p.off_z;
  for (int i = 0; i < count; ++i) {
    const mecefo_subspace_job& j = jobs[i];
    const int n = (int)j.cols, k = j.k, r = j.r, rows = (int)j.rows;
    float* B = reinterpret_cast<float*>(ws + ob); ob += al256((size_t)n * n * 4);
    float* Z = reinterpret_cast<float*>(ws + oz); oz += al256((size_t)n * k * 4);
    float* g = G + i * kk;
    float* m = Mm + i * kk;
    SubGemmJob ph[SUB_PHASES] = {
        sub_job(j.w, j.ldw, false, j.w, j.ldw, B, n, n, n, rows),
        sub_job(B, n, true, j.v, k, Z, k, n, k, n),
        sub_job(Z, k, false, Z, k, g, kmax, k, k, n),
        sub_job(Z, k, true, m, kmax, j.v, k, n, k, k),
        sub_job(j.v, k, false, Z, k, g, kmax, k, k, n),
        sub_job(j.v, k, true, Ur + (size_t)i * kmax * rmax, r, j.v1, r, n, r, k),
    };
    for (int q : {2, 4}) {  // Gram products: K = cols >> k
      ph[q].ksplit = SUB_GRAM_SPLIT;
      ph[q].kchunk = ((n + SUB_GRAM_SPLIT - 1) / SUB_GRAM_SPLIT + SG_TK - 1) / SG_TK * SG_TK;
      ph[q].c_split = (int64_t)count * kk;
    }
    for (int q = 0; q < SUB_PHASES; ++q) {
      ph[q].tile0 = tiles[q];
      tiles[q] += ph[q].tiles_mn * ph[q].ksplit;
      hj[(size_t)q * count + i] = ph[q];
    }
    hk[i] = k;
    hk[count + i] = r;
  }
  SubGemmJob* dj = reinterpret_cast<SubGemmJob*>(ws + p.off_jobs);
  int* dk = reinterpret_cast<int*>(ws + p.off_ks);
  // pageable sources: the copies are staged before these calls return
  CUDA_TRY(cudaMemcpyAsync(dj, hj.data(), hj.size() * sizeof(SubGemmJob), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dk, hk.data(), hk.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  TRY(ensure_smem((const void*)subspace_chol_inv_kernel, (int)SUB_SMEM_MAX));
  TRY(ensure_smem((const void*)subspace_ritz_kernel, (int)SUB_SMEM_MAX));
  void* scratch = p.smem ? nullptr : ws + p.off_scr;
  const size_t scr_stride = std::max(p.chol_bytes, p.ritz_bytes);
  static const char* const phase_tag[SUB_PHASES] = {"subspace.gram_w", "subspace.bv", "subspace.gram_z",
                                                     "subspace.zm", "subspace.vtz", "subspace.rotate"};
  auto gemm_phase = [&](int q) -> int {
    ProfScope ps(phase_tag[q], 0.0, 0.0, s);
    subspace_gemm_kernel<<<tiles[q], SG_THREADS, 0, s>>>(dj + (size_t)q * count, count);
    return check_launch("subspace_gemm_kernel");
  };
  TRY(gemm_phase(0));
  for (int it = 0; it < iterations; ++it) {
    TRY(gemm_phase(1));
    TRY(gemm_phase(2));
    {
      ProfScope ps("subspace.chol", 0.0, 0.0, s);
      // the global-scratch layout uses the same per-matrix stride as the Ritz step
      subspace_chol_inv_kernel<<<count, SUB_SMALL_THREADS, p.smem ? p.chol_bytes : 0, s>>>(
          G, Mm, dk, kmax, static_cast<double*>(scratch), p.smem ? 1 : 0, scr_stride / 8, SUB_GRAM_SPLIT,
          (size_t)count * kk);
      TRY(check_launch("subspace_chol_inv_kernel"));
    }
    TRY(gemm_phase(3));
  }
  TRY(gemm_phase(1));
  TRY(gemm_phase(4));
  {
    ProfScope ps("subspace.ritz", 0.0, 0.0, s);
    subspace_ritz_kernel<<<count, SUB_SMALL_THREADS, p.smem ? p.ritz_bytes : 0, s>>>(G, Ur, Th, dk, dk + count, kmax, rmax, scratch,
                                                                     scr_stride, p.smem ? 1 : 0, SUB_GRAM_SPLIT,
                                                                     (size_t)count * kk);
    TRY(check_launch("subspace_ritz_kernel"));
  }
  TRY(gemm_phase(5));
  for (int i = 0; i < count; ++i)
    if (jobs[i].theta)
      CUDA_TRY(cudaMemcpyAsync(jobs[i].theta, Th + (size_t)i * rmax, jobs[i].r * 4, cudaMemcpyDeviceToDevice, s));
  return MECEFO_OK;
}

}  // extern "C"
