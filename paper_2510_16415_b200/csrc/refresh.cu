// Converged projection refresh: host orchestration and C-ABI
// (include/mecefo.h: mecefo_refresh_converged). Each job is one
// top_r_right_singular_vectors call (linalg.py:97-142); a refresh batches
// every due (layer, kind) of a rank (approx.py:66-87), and all matrices
// advance together, one launch per phase.
//
// The computed object and the stopping rule are the reference's: the top-r
// invariant subspace of B = W^T W, returned when every kept Ritz pair has
//   ||B v_j - theta_j v_j|| <= tol * theta_0        (linalg.py:131-135)
// in float64; otherwise MECEFO_ERR_SVD_NOCONV (SvdConvergenceError). The
// iteration that gets there is cheaper than the reference's one
// B-product-per-step block power method:
//   * Chebyshev filtering: between two Rayleigh-Ritz steps the block is
//     multiplied by T_d((B - c)/e), the degree-d Chebyshev polynomial that
//     damps [0, theta_{k-1}] and amplifies the wanted end — the
//     (lambda_r / lambda_k)^d power-method contraction becomes ~exp(-2 d
//     sqrt(gap)); d is chosen so T_d(x_max) <= 1e6 (well-conditioned CholQR);
//   * a wider block (k = r + oversample, oversample >= 4 chosen by the
//     caller) — only span(V[:, :r]) is returned, as in the reference;
//   * when W is wide (rows < cols, e.g. the down projection, m x f) the
//     iteration runs on the smaller C = W W^T (rows x rows) from the start
//     block W V0 (the image of the reference's start block) and maps back,
//     V = W^T U diag(theta)^-1/2; the reference's residual is then checked in
//     the original space on B = W^T W itself;
//   * one B-product per Rayleigh-Ritz step (B V comes out of the Ritz
//     rotation of B Q), float64 DMMA tensor-core GEMMs, Jacobi-preconditioned
//     CholeskyQR2, a device Jacobi eigensolver for the k x k Ritz problem.
// `products` counts block products with B (or C) against the caller's
// max_iterations budget (the reference spends one per iteration).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "host.h"
#include "refresh.cuh"

using namespace mecefo;
using namespace mecefo::rf;
using namespace mecefo_host;

namespace {

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kSlots = 96;  // device job-array slots per outer iteration
// Chebyshev amplification ceiling T_d(x_max) per filtered step:
// clamp(kChebScale / residual, kChebMin, kChebMax); overridable for experiments
// through MECEFO_CHEB="min,max,scale".
double kChebMin = 1e8, kChebMax = 1e12, kChebScale = 1e4;
#ifdef MECEFO_TIMING_KNOBS  // experiments only (libmecefo_timing.so)
struct ChebEnv {
  ChebEnv() {
    if (const char* v = getenv("MECEFO_CHEB")) sscanf(v, "%lf,%lf,%lf", &kChebMin, &kChebMax, &kChebScale);
  }
} g_cheb_env;
#endif
constexpr size_t kSmemLimit = 227 * 1024;

struct RfPlan {
  int dual = 0;
  int64_t n = 0;  // Gram dimension
  int k = 0, r = 0;
  size_t off = 0;  // this job's region in the workspace
  size_t bytes = 0;
  // region layout (doubles)
  double *G, *Q, *Wq, *GV, *V, *Xa, *Xb, *S, *Mk, *Uk, *scr, *Vs, *BVs, *P;
  int done = 0;
  int products = 0;
  int rr_steps = 0;
  double resid = INFINITY, tol_inner = 0.0;
  std::vector<double> theta;
};

int64_t n_of(const mecefo_refresh_job& j, int* dual) {
  *dual = (j.cols > j.rows && j.k <= j.rows) ? 1 : 0;
  return *dual ? j.rows : j.cols;
}

size_t scratch_doubles(int k) { return (size_t)k * k + (size_t)k * (k | 1) + 2 * (size_t)k; }

void layout(RfPlan& p, const mecefo_refresh_job& j, char* base) {
  p.n = n_of(j, &p.dual);
  p.k = j.k;
  p.r = j.r;
  const size_t n = p.n, k = p.k, r = p.r;
  size_t o = 0;
  auto take = [&](size_t doubles) {
    double* q = base ? reinterpret_cast<double*>(base + p.off + o) : nullptr;
    o = al256(o + doubles * 8);
    return q;
  };
  p.G = take(n * n);
  p.Q = take(n * k);
  p.Wq = take(n * k);
  p.GV = take(n * k);
  p.V = take(n * k);
  p.Xa = take(n * k);
  p.Xb = take(n * k);
  p.S = take(k * k);
  p.Mk = take(k * k);
  p.Uk = take(k * k);
  p.scr = take(scratch_doubles(p.k));
  if (p.dual) {
    p.Vs = take((size_t)j.cols * r);
    p.BVs = take((size_t)j.cols * r);
    p.P = take((size_t)j.rows * r);
  } else {
    p.Vs = p.BVs = p.P = nullptr;
  }
  p.bytes = o;
}

struct Ctx {
  cudaStream_t s;
  char* arena;        // kSlots x slot_bytes
  size_t slot_bytes;
  int slot = 0;
  double* summary;    // per job: [theta (kmax), resid]
  int kmax;
  int64_t launches = 0;
  void* next_slot(size_t bytes, int* rc) {
    if (slot >= kSlots || bytes > slot_bytes) {
      *rc = set_err(MECEFO_ERR_CONSISTENCY, "refresh job-array arena exhausted");
      return nullptr;
    }
    return arena + (size_t)(slot++) * slot_bytes;
  }
};

int launch_dgemm(Ctx& cx, std::vector<DJob>& jobs, const char* tag) {
  if (jobs.empty()) return MECEFO_OK;
  int tiles = 0;
  double flops = 0.0;
  for (auto& j : jobs) {
    j.tiles_n = (j.N + DG_BN - 1) / DG_BN;
    j.tiles_mn = ((j.M + DG_BM - 1) / DG_BM) * j.tiles_n;
    if (j.ksplit < 1) j.ksplit = 1;
    j.kchunk = ((j.K + j.ksplit - 1) / j.ksplit + DG_BK - 1) / DG_BK * DG_BK;
    j.ksplit = (j.K + j.kchunk - 1) / j.kchunk;
    j.tile0 = tiles;
    tiles += j.tiles_mn * j.ksplit;
    flops += 2.0 * j.M * j.N * j.K;
  }
  int rc = MECEFO_OK;
  void* d = cx.next_slot(jobs.size() * sizeof(DJob), &rc);
  TRY(rc);
  CUDA_TRY(cudaMemcpyAsync(d, jobs.data(), jobs.size() * sizeof(DJob), cudaMemcpyHostToDevice, cx.s));
  ProfScope prof(tag, flops, 0.0, cx.s);
  dgemm_batched_kernel<<<tiles, DG_THREADS, 0, cx.s>>>(reinterpret_cast<const DJob*>(d), (int)jobs.size());
  return check_launch("dgemm_batched_kernel");
}

// Gram-type products (k x k output, long K): split K across the SMs when the
// output tiles alone cannot fill the GPU; the outputs are zeroed first.
int launch_dgemm_split(Ctx& cx, std::vector<DJob>& jobs, const char* tag) {
  int tiles = 0;
  for (auto& j : jobs) tiles += ((j.M + DG_BM - 1) / DG_BM) * ((j.N + DG_BN - 1) / DG_BN);
  const int want = tiles >= kNumSMs ? 1 : (kNumSMs + tiles - 1) / std::max(1, tiles);
  for (auto& j : jobs) {
    const int sp = std::max(1, std::min(want, j.K / (4 * DG_BK)));
    j.ksplit = sp;
    if (sp > 1) {
      if (j.cin || j.din) return set_err(MECEFO_ERR_CONSISTENCY, "split-K GEMM cannot fuse beta/gamma terms");
      CUDA_TRY(cudaMemsetAsync(j.c, 0, (size_t)j.M * j.ldc * sizeof(double), cx.s));
    }
  }
  return launch_dgemm(cx, jobs, tag);
}

}  // namespace

extern "C" {

size_t mecefo_refresh_workspace_bytes(const mecefo_refresh_job* jobs, int32_t count) {
  if (!jobs || count < 1) return 0;
  size_t total = 0;
  int kmax = 1;
  for (int i = 0; i < count; ++i) {
    RfPlan p;
    p.off = total;
    layout(p, jobs[i], nullptr);
    total = al256(total + p.bytes);
    kmax = std::max(kmax, jobs[i].k);
  }
  const size_t slot = al256(2 * (size_t)count * std::max(sizeof(DJob), std::max(sizeof(SmallJob), sizeof(ResJob) + sizeof(CopyJob) + sizeof(AxJob))));
  total += kSlots * slot;
  total += al256((size_t)count * (kmax + 2) * sizeof(double));
  return total + 1024;
}

}  // extern "C"

namespace {

int run_small(Ctx& cx, const void* kern, std::vector<SmallJob>& js, size_t smem) {
  if (js.empty()) return MECEFO_OK;
  int rc = MECEFO_OK;
  void* d = cx.next_slot(js.size() * sizeof(SmallJob), &rc);
  TRY(rc);
  CUDA_TRY(cudaMemcpyAsync(d, js.data(), js.size() * sizeof(SmallJob), cudaMemcpyHostToDevice, cx.s));
  if (smem > 0) TRY(ensure_smem(kern, (int)smem));
  ProfScope prof(kern == (const void*)cholqr_kernel ? "refresh.cholqr" : "refresh.jacobi", 0.0, 0.0, cx.s);
  void* args[] = {&d};
  CUDA_TRY(cudaLaunchKernel(kern, dim3((unsigned)js.size()), dim3(RF_SMALL_THREADS), args, smem, cx.s));
  return check_launch(kern == (const void*)cholqr_kernel ? "cholqr_kernel" : "jacobi_eig_kernel");
}

// CholeskyQR2 of Z (n x k, per plan) into Qout, via tmp; Z, tmp, Qout distinct.
int qr2(Ctx& cx, std::vector<RfPlan*>& ps, std::vector<double*>& Z, std::vector<double*>& tmp,
        std::vector<double*>& Qout) {
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<DJob> g;
    for (size_t i = 0; i < ps.size(); ++i) {
      RfPlan& p = *ps[i];
      double* src = pass == 0 ? Z[i] : tmp[i];
      DJob j{};
      j.a = src; j.lda = p.k; j.a_kmajor = 0;  // A(m, t) = Z[t, m]
      j.b = src; j.ldb = p.k; j.b_kmajor = 0;  // B(t, n) = Z[t, n]
      j.c = p.S; j.ldc = p.k; j.alpha = 1.0;
      j.M = p.k; j.N = p.k; j.K = (int)p.n;
      g.push_back(j);
    }
    TRY(launch_dgemm_split(cx, g, "refresh.qr_gram"));
    std::vector<SmallJob> sj;
    size_t smem = 0;
    for (auto* pp : ps) {
      const size_t need = ((size_t)pp->k * (pp->k | 1) + 2 * (size_t)pp->k) * 8;
      const int use = need <= kSmemLimit - 1024 ? 1 : 0;
      if (use) smem = std::max(smem, need);
      sj.push_back(SmallJob{pp->S, pp->Mk, nullptr, pp->scr, pp->k, use, 0.0, nullptr});
    }
    TRY(run_small(cx, (const void*)cholqr_kernel, sj, smem));
    std::vector<DJob> m;
    for (size_t i = 0; i < ps.size(); ++i) {
      RfPlan& p = *ps[i];
      DJob j{};
      j.a = pass == 0 ? Z[i] : tmp[i]; j.lda = p.k; j.a_kmajor = 1;
      j.b = p.Mk; j.ldb = p.k;
      j.c = pass == 0 ? tmp[i] : Qout[i]; j.ldc = p.k; j.alpha = 1.0;
      j.M = (int)p.n; j.N = p.k; j.K = p.k;
      m.push_back(j);
    }
    TRY(launch_dgemm(cx, m, "refresh.qr_apply"));
  }
  return MECEFO_OK;
}

// Rayleigh-Ritz on the orthonormal block Q: Wq = G Q (one G-product),
// S = Q^T Wq, S = U diag(theta) U^T, V = Q U, GV = Wq U, residual.
int rayleigh_ritz(Ctx& cx, std::vector<RfPlan*>& ps, std::vector<int>& idx) {
  std::vector<DJob> a, b, c;
  for (auto* pp : ps) {
    RfPlan& p = *pp;
    DJob j{};
    j.a = p.G; j.lda = p.n; j.a_kmajor = 1;
    j.b = p.Q; j.ldb = p.k;
    j.c = p.Wq; j.ldc = p.k; j.alpha = 1.0;
    j.M = (int)p.n; j.N = p.k; j.K = (int)p.n;
    a.push_back(j);
    p.products += 1;
    p.rr_steps += 1;
    DJob s{};
    s.a = p.Q; s.lda = p.k; s.a_kmajor = 0;
    s.b = p.Wq; s.ldb = p.k;
    s.c = p.S; s.ldc = p.k; s.alpha = 1.0;
    s.M = p.k; s.N = p.k; s.K = (int)p.n;
    b.push_back(s);
  }
  TRY(launch_dgemm(cx, a, "refresh.bq"));
  TRY(launch_dgemm_split(cx, b, "refresh.qtbq"));
  std::vector<SmallJob> sj;
  size_t smem = 0;
  for (size_t i = 0; i < ps.size(); ++i) {
    RfPlan& p = *ps[i];
    const size_t need = (((size_t)p.k * (p.k + 1) / 2 + 1) / 2 * 2 + (size_t)p.k * p.k) * 8;
    const int use = need <= kSmemLimit - 14 * 1024 ? 1 : 0;
    if (use) smem = std::max(smem, need);
    // Jacobi accuracy follows the outer residual: early Ritz steps need only
    // a rough rotation (Frobenius off-mass 1e-8 x the residual, squared)
    const double rel = std::min(1e-6, std::max(1e-15, 1e-4 * p.resid));
    double* th = cx.summary + (size_t)idx[i] * (cx.kmax + 2);
    sj.push_back(SmallJob{p.S, p.Uk, th, p.scr, p.k, use, rel * rel, th + cx.kmax + 1});
  }
  TRY(run_small(cx, (const void*)jacobi_eig_kernel, sj, smem));
  for (auto* pp : ps) {
    RfPlan& p = *pp;
    DJob v{};
    v.a = p.Q; v.lda = p.k; v.a_kmajor = 1;
    v.b = p.Uk; v.ldb = p.k;
    v.c = p.V; v.ldc = p.k; v.alpha = 1.0;
    v.M = (int)p.n; v.N = p.k; v.K = p.k;
    c.push_back(v);
    DJob w = v;
    w.a = p.Wq;
    w.c = p.GV;
    c.push_back(w);
  }
  TRY(launch_dgemm(cx, c, "refresh.rotate"));
  std::vector<ResJob> rj;
  for (size_t i = 0; i < ps.size(); ++i) {
    RfPlan& p = *ps[i];
    double* th = cx.summary + (size_t)idx[i] * (cx.kmax + 2);
    rj.push_back(ResJob{p.V, p.GV, th, th + cx.kmax, (int)p.n, p.k, p.r});
  }
  int rc = MECEFO_OK;
  void* d = cx.next_slot(rj.size() * sizeof(ResJob), &rc);
  TRY(rc);
  CUDA_TRY(cudaMemcpyAsync(d, rj.data(), rj.size() * sizeof(ResJob), cudaMemcpyHostToDevice, cx.s));
  ProfScope prof("refresh.residual", 0.0, 0.0, cx.s);
  residual_kernel<<<(unsigned)rj.size(), 1024, 0, cx.s>>>(reinterpret_cast<const ResJob*>(d));
  return check_launch("residual_kernel");
}

int axpby(Ctx& cx, std::vector<AxJob>& js) {
  if (js.empty()) return MECEFO_OK;
  int64_t total = 0;
  for (auto& j : js) {
    j.off = total;
    total += j.n;
  }
  int rc = MECEFO_OK;
  void* d = cx.next_slot(js.size() * sizeof(AxJob), &rc);
  TRY(rc);
  CUDA_TRY(cudaMemcpyAsync(d, js.data(), js.size() * sizeof(AxJob), cudaMemcpyHostToDevice, cx.s));
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 8 * kNumSMs);
  ProfScope prof("refresh.axpby", 0.0, 0.0, cx.s);
  axpby_f64_kernel<<<(unsigned)blocks, 256, 0, cx.s>>>(reinterpret_cast<const AxJob*>(d), (int)js.size(), total);
  return check_launch("axpby_f64_kernel");
}

int extract(Ctx& cx, std::vector<CopyJob>& js) {
  if (js.empty()) return MECEFO_OK;
  int64_t total = 0;
  for (auto& j : js) {
    j.off = total;
    total += (int64_t)j.rows * j.cols;
  }
  int rc = MECEFO_OK;
  void* d = cx.next_slot(js.size() * sizeof(CopyJob), &rc);
  TRY(rc);
  CUDA_TRY(cudaMemcpyAsync(d, js.data(), js.size() * sizeof(CopyJob), cudaMemcpyHostToDevice, cx.s));
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 8 * kNumSMs);
  extract_cols_kernel<<<(unsigned)blocks, 256, 0, cx.s>>>(reinterpret_cast<const CopyJob*>(d), (int)js.size(), total);
  return check_launch("extract_cols_kernel");
}

}  // namespace

extern "C" {

int mecefo_refresh_converged(mecefo_engine* e, mecefo_refresh_job* jobs, int32_t count, double tol,
                             int32_t max_products, void* workspace, size_t workspace_bytes, void* stream) {
  (void)e;
  if (!jobs || count < 1) return set_err(MECEFO_ERR_CONTRACT, "refresh needs >= 1 job");
  if (!(tol > 0.0)) return set_err(MECEFO_ERR_CONTRACT, "tolerance must be > 0");
  if (max_products < 1) return set_err(MECEFO_ERR_CONTRACT, "max_iterations must be >= 1");
  for (int i = 0; i < count; ++i) {
    const mecefo_refresh_job& j = jobs[i];
    if (!j.w || !j.v0 || !j.v1) return set_err(MECEFO_ERR_CONTRACT, "job %d: null pointer", i);
    if (j.rows < 1 || j.cols < 1 || j.ldw < j.cols)
      return set_err(MECEFO_ERR_CONTRACT, "job %d: bad shape %lldx%lld ld %lld", i, (long long)j.rows,
                     (long long)j.cols, (long long)j.ldw);
    if (j.r < 1 || j.r > j.cols) return set_err(MECEFO_ERR_CONTRACT, "rank %d exceeds the column count of (%lld, %lld)",
                                                 j.r, (long long)j.rows, (long long)j.cols);
    if (j.k < j.r || j.k > j.cols || j.k > 1024)
      return set_err(MECEFO_ERR_CONTRACT, "job %d: need r=%d <= k=%d <= min(cols=%lld, 1024)", i, j.r, j.k,
                     (long long)j.cols);
    if (j.cols > 46340 || j.rows > 46340) return set_err(MECEFO_ERR_CONTRACT, "job %d: matrix too large", i);
  }
  const size_t need = mecefo_refresh_workspace_bytes(jobs, count);
  if (!workspace || workspace_bytes < need)
    return set_err(MECEFO_ERR_CONTRACT, "refresh workspace too small: %zu < %zu", workspace_bytes, need);
  char* base = static_cast<char*>(workspace);
  base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + 255) & ~uintptr_t(255));
  std::vector<RfPlan> plans(count);
  size_t off = 0;
  int kmax = 1;
  for (int i = 0; i < count; ++i) {
    plans[i].off = off;
    layout(plans[i], jobs[i], base);
    off = al256(off + plans[i].bytes);
    kmax = std::max(kmax, jobs[i].k);
  }
  Ctx cx;
  cx.s = reinterpret_cast<cudaStream_t>(stream);
  cx.slot_bytes = al256(2 * (size_t)count * std::max(sizeof(DJob), std::max(sizeof(SmallJob), sizeof(ResJob) + sizeof(CopyJob) + sizeof(AxJob))));
  cx.arena = base + off;
  off += kSlots * cx.slot_bytes;
  cx.summary = reinterpret_cast<double*>(base + off);
  cx.kmax = kmax;
  std::vector<double> summary((size_t)count * (kmax + 2));
  CUDA_TRY(cudaMemsetAsync(cx.summary, 0, summary.size() * 8, cx.s));
  for (int i = 0; i < count; ++i) plans[i].tol_inner = plans[i].dual ? tol / 16.0 : tol;

  // ---- B = W^T W (primal) or C = W W^T (dual), from the fp32 weights
  {
    std::vector<DJob> g;
    for (int i = 0; i < count; ++i) {
      const mecefo_refresh_job& jb = jobs[i];
      RfPlan& p = plans[i];
      DJob j{};
      j.a = jb.w; j.lda = jb.ldw; j.a_f32 = 1;
      j.b = jb.w; j.ldb = jb.ldw; j.b_f32 = 1;
      if (p.dual) {  // C(i, j) = sum_t W[i, t] W[j, t]
        j.a_kmajor = 1; j.b_kmajor = 1;
        j.M = j.N = (int)jb.rows; j.K = (int)jb.cols;
      } else {       // B(i, j) = sum_t W[t, i] W[t, j]
        j.a_kmajor = 0; j.b_kmajor = 0;
        j.M = j.N = (int)jb.cols; j.K = (int)jb.rows;
      }
      j.c = p.G; j.ldc = p.n; j.alpha = 1.0;
      g.push_back(j);
    }
    TRY(launch_dgemm_split(cx, g, "refresh.gram"));
  }
  // ---- start block: Q0 = V0 (primal, orthonormal from the host QR,
  // linalg.py:117) or qr(W V0) (dual: the image of the same start block)
  std::vector<RfPlan*> all;
  std::vector<int> all_idx;
  for (int i = 0; i < count; ++i) {
    all.push_back(&plans[i]);
    all_idx.push_back(i);
  }
  {
    std::vector<DJob> st;
    std::vector<RfPlan*> dps;
    std::vector<double*> Z, T, Qo;
    for (int i = 0; i < count; ++i) {
      RfPlan& p = plans[i];
      const mecefo_refresh_job& jb = jobs[i];
      if (!p.dual) {
        CUDA_TRY(cudaMemcpyAsync(p.Q, jb.v0, (size_t)p.n * p.k * 8, cudaMemcpyDeviceToDevice, cx.s));
        continue;
      }
      DJob j{};
      j.a = jb.w; j.lda = jb.ldw; j.a_f32 = 1; j.a_kmajor = 1;
      j.b = jb.v0; j.ldb = p.k;
      j.c = p.Xa; j.ldc = p.k; j.alpha = 1.0;
      j.M = (int)jb.rows; j.N = p.k; j.K = (int)jb.cols;
      st.push_back(j);
      dps.push_back(&p);
      Z.push_back(p.Xa);
      T.push_back(p.Xb);
      Qo.push_back(p.Q);
    }
    TRY(launch_dgemm(cx, st, "refresh.start"));
    if (!dps.empty()) TRY(qr2(cx, dps, Z, T, Qo));
  }
  TRY(rayleigh_ritz(cx, all, all_idx));

  int rc_final = MECEFO_OK;
  double worst = 0.0;
  for (;;) {
    CUDA_TRY(cudaMemcpyAsync(summary.data(), cx.summary, summary.size() * 8, cudaMemcpyDeviceToHost, cx.s));
    CUDA_TRY(cudaStreamSynchronize(cx.s));
    cx.slot = 0;
    std::vector<RfPlan*> act;
    std::vector<int> act_idx;
    for (int i = 0; i < count; ++i) {
      RfPlan& p = plans[i];
      if (p.done) continue;
      const double* th = summary.data() + (size_t)i * (kmax + 2);
      p.resid = th[kmax];
      p.theta.assign(th, th + p.k);
      if (!(th[0] > 0.0)) {  // B == 0 (linalg.py:112-114): first r standard basis vectors
        std::vector<float> eye((size_t)jobs[i].cols * p.r, 0.f);
        for (int c = 0; c < p.r; ++c) eye[(size_t)c * p.r + c] = 1.f;
        CUDA_TRY(cudaMemcpyAsync(jobs[i].v1, eye.data(), eye.size() * 4, cudaMemcpyHostToDevice, cx.s));
        CUDA_TRY(cudaStreamSynchronize(cx.s));
        if (jobs[i].v1_f64) {
          std::vector<double> e64(eye.begin(), eye.end());
          CUDA_TRY(cudaMemcpy(jobs[i].v1_f64, e64.data(), e64.size() * 8, cudaMemcpyHostToDevice));
        }
        if (jobs[i].theta) CUDA_TRY(cudaMemsetAsync(jobs[i].theta, 0, (size_t)p.r * 8, cx.s));
        p.done = 1;
        p.resid = 0.0;
        continue;
      }
      if (p.resid <= p.tol_inner) {
        p.done = 2;  // finalize below
        continue;
      }
      if (p.products >= max_products) {
        p.done = 3;
        continue;
      }
      act.push_back(&p);
      act_idx.push_back(i);
    }
    // ---- finalize converged jobs
    std::vector<int> fin_jobs;
    for (int i = 0; i < count; ++i)
      if (plans[i].done == 2) fin_jobs.push_back(i);
    if (!fin_jobs.empty()) {
      std::vector<CopyJob> cj;
      std::vector<DJob> m1, m2, m3;
      std::vector<int> duals;
      for (int i : fin_jobs) {
        RfPlan& p = plans[i];
        const mecefo_refresh_job& jb = jobs[i];
        if (!p.dual) {
          cj.push_back(CopyJob{jb.v1, p.V, p.r, p.k, jb.v1_f64, nullptr, (int)p.n, p.r, 0});
          continue;
        }
        // V = W^T U_r diag(theta_r)^-1/2 (cols x r); B V = W^T (W V) for the reference residual
        DJob j{};
        j.a = jb.w; j.lda = jb.ldw; j.a_f32 = 1; j.a_kmajor = 0;  // A(m, t) = W[t, m]
        j.b = p.V; j.ldb = p.k;
        j.c = p.BVs; j.ldc = p.r; j.alpha = 1.0;
        j.M = (int)jb.cols; j.N = p.r; j.K = (int)jb.rows;
        m1.push_back(j);
        duals.push_back(i);
      }
      TRY(launch_dgemm(cx, m1, "refresh.map"));
      // per-column scale theta^-1/2 (host computes the scale vector into Mk's first row)
      for (int i : duals) {
        RfPlan& p = plans[i];
        std::vector<double> sc(p.r);
        for (int c = 0; c < p.r; ++c) sc[c] = p.theta[c] > 0.0 ? 1.0 / std::sqrt(p.theta[c]) : 0.0;
        CUDA_TRY(cudaMemcpyAsync(p.Mk, sc.data(), p.r * 8, cudaMemcpyHostToDevice, cx.s));
        CUDA_TRY(cudaStreamSynchronize(cx.s));
        cj.push_back(CopyJob{nullptr, p.BVs, p.r, p.r, p.Vs, p.Mk, (int)jobs[i].cols, p.r, 0});
      }
      TRY(extract(cx, cj));
      // theta out for primal jobs and duals
      for (int i : fin_jobs)
        if (jobs[i].theta)
          CUDA_TRY(cudaMemcpyAsync(jobs[i].theta, cx.summary + (size_t)i * (kmax + 2), (size_t)plans[i].r * 8,
                                   cudaMemcpyDeviceToDevice, cx.s));
      if (!duals.empty()) {
        for (int i : duals) {
          RfPlan& p = plans[i];
          const mecefo_refresh_job& jb = jobs[i];
          DJob j{};
          j.a = jb.w; j.lda = jb.ldw; j.a_f32 = 1; j.a_kmajor = 1;  // P = W V
          j.b = p.Vs; j.ldb = p.r;
          j.c = p.P; j.ldc = p.r; j.alpha = 1.0;
          j.M = (int)jb.rows; j.N = p.r; j.K = (int)jb.cols;
          m2.push_back(j);
          DJob k2{};
          k2.a = jb.w; k2.lda = jb.ldw; k2.a_f32 = 1; k2.a_kmajor = 0;  // B V = W^T P
          k2.b = p.P; k2.ldb = p.r;
          k2.c = p.BVs; k2.ldc = p.r; k2.alpha = 1.0;
          k2.M = (int)jb.cols; k2.N = p.r; k2.K = (int)jb.rows;
          m3.push_back(k2);
        }
        TRY(launch_dgemm(cx, m2, "refresh.check_wv"));
        TRY(launch_dgemm(cx, m3, "refresh.check_wtwv"));
        std::vector<ResJob> rj;
        std::vector<double> resd(duals.size());
        for (size_t q = 0; q < duals.size(); ++q) {
          RfPlan& p = plans[duals[q]];
          rj.push_back(ResJob{p.Vs, p.BVs, cx.summary + (size_t)duals[q] * (kmax + 2), plans[duals[q]].S, (int)jobs[duals[q]].cols,
                              p.r, p.r});
        }
        int rc = MECEFO_OK;
        void* d = cx.next_slot(rj.size() * sizeof(ResJob), &rc);
        TRY(rc);
        CUDA_TRY(cudaMemcpyAsync(d, rj.data(), rj.size() * sizeof(ResJob), cudaMemcpyHostToDevice, cx.s));
        residual_kernel<<<(unsigned)rj.size(), 1024, 0, cx.s>>>(reinterpret_cast<const ResJob*>(d));
        TRY(check_launch("residual_kernel"));
        for (size_t q = 0; q < duals.size(); ++q)
          CUDA_TRY(cudaMemcpyAsync(&resd[q], plans[duals[q]].S, 8, cudaMemcpyDeviceToHost, cx.s));
        CUDA_TRY(cudaStreamSynchronize(cx.s));
        std::vector<CopyJob> out;
        for (size_t q = 0; q < duals.size(); ++q) {
          RfPlan& p = plans[duals[q]];
          p.resid = resd[q];
          if (resd[q] <= tol) {
            out.push_back(CopyJob{jobs[duals[q]].v1, p.Vs, p.r, p.r, jobs[duals[q]].v1_f64, nullptr,
                                  (int)jobs[duals[q]].cols, p.r, 0});
          } else if (p.products < max_products) {  // tighten the inner tolerance and keep iterating
            p.tol_inner *= 0.125;
            p.done = 0;
            act.push_back(&p);
            act_idx.push_back(duals[q]);
          } else {
            p.done = 3;
          }
        }
        TRY(extract(cx, out));
      }
      for (int i : fin_jobs)
        if (plans[i].done == 2) plans[i].done = 1;
    }
    if (act.empty()) break;
    // ---- one Chebyshev-filtered step for every active job
    std::vector<int> deg(act.size());
    std::vector<double> cc(act.size()), ee(act.size());
    int dmax = 1;
    for (size_t q = 0; q < act.size(); ++q) {
      RfPlan& p = *act[q];
      const double t0 = p.theta[0], tk = p.theta[p.k - 1];
      const double a = std::max(tk, 1e-12 * t0);  // damp [0, theta_{k-1}]
      cc[q] = 0.5 * a;
      ee[q] = 0.5 * a;
      const double xmax = (1.05 * t0 - cc[q]) / ee[q];
      int d = 1;
      // amplification ceiling T_d(x_max): 1e6 while the block is rough, up to
      // 1e10 as the Ritz vectors converge (their contamination x the ratio
      // stays far below the columns' own signal)
      const double lim = std::max(kChebMin, std::min(kChebMax, kChebScale / std::max(p.resid, 1e-30)));
      if (xmax > 1.0 + 1e-12 && p.k < p.n) d = (int)std::floor(std::acosh(lim) / std::acosh(xmax));
      if (p.k >= p.n) d = 1;
      d = std::max(1, std::min(d, 24));
      d = std::min(d, std::max(1, max_products - p.products - 1));
      deg[q] = d;
      dmax = std::max(dmax, d);
    }
    // X1 = (G V - c V) / e
    std::vector<double*> Xprev(act.size()), Xcur(act.size()), Xfree(act.size());
    {
      std::vector<AxJob> ax;
      for (size_t q = 0; q < act.size(); ++q) {
        RfPlan& p = *act[q];
        ax.push_back(AxJob{p.Xa, p.GV, p.V, 1.0 / ee[q], -cc[q] / ee[q], (int64_t)p.n * p.k, 0});
        Xprev[q] = p.V;
        Xcur[q] = p.Xa;
        Xfree[q] = p.Xb;
      }
      TRY(axpby(cx, ax));
    }
    for (int s = 1; s < dmax; ++s) {  // X_{s+1} = 2/e (G X_s) - 2c/e X_s - X_{s-1}
      std::vector<DJob> g;
      for (size_t q = 0; q < act.size(); ++q) {
        if (deg[q] <= s) continue;
        RfPlan& p = *act[q];
        DJob j{};
        j.a = p.G; j.lda = p.n; j.a_kmajor = 1;
        j.b = Xcur[q]; j.ldb = p.k;
        j.c = Xfree[q]; j.ldc = p.k;
        j.alpha = 2.0 / ee[q];
        j.cin = Xcur[q]; j.ldcin = p.k; j.beta = -2.0 * cc[q] / ee[q];
        j.din = Xprev[q]; j.lddin = p.k; j.gamma = -1.0;
        j.M = (int)p.n; j.N = p.k; j.K = (int)p.n;
        g.push_back(j);
        p.products += 1;
        double* nf = Xprev[q];
        Xprev[q] = Xcur[q];
        Xcur[q] = Xfree[q];
        Xfree[q] = nf;
      }
      TRY(launch_dgemm(cx, g, "refresh.chebyshev"));
    }
    // QR of the filtered block into Q (temp: the free buffer), then Rayleigh-Ritz
    std::vector<double*> Z(act.size()), T(act.size()), Qo(act.size());
    for (size_t q = 0; q < act.size(); ++q) {
      Z[q] = Xcur[q];
      T[q] = Xfree[q];
      Qo[q] = act[q]->Q;
    }
    TRY(qr2(cx, act, Z, T, Qo));
    TRY(rayleigh_ritz(cx, act, act_idx));
  }
  for (int i = 0; i < count; ++i) {
    jobs[i].residual = plans[i].resid;
    jobs[i].products = plans[i].products;
    jobs[i].rr_steps = plans[i].rr_steps;
    jobs[i].jacobi_sweeps = (int32_t)summary[(size_t)i * (kmax + 2) + kmax + 1];
    jobs[i].converged = plans[i].done == 1 ? 1 : 0;
    if (plans[i].done != 1) {
      worst = std::max(worst, plans[i].resid);
      rc_final = MECEFO_ERR_SVD_NOCONV;
    }
  }
  if (rc_final != MECEFO_OK)
    return set_err(MECEFO_ERR_SVD_NOCONV,
                   "subspace iteration did not converge within %d iterations (last residual %.3e)", max_products,
                   worst);
  CUDA_TRY(cudaStreamSynchronize(cx.s));
  return MECEFO_OK;
}

}  // extern "C"
