// Batched block power iteration for the projection refresh (approx.py:66-87
// over every due (layer, kind), each running linalg.py:97-142).
//
// All matrices of one refresh advance together, so every phase of an
// iteration is ONE launch over the union of their tiles:
//   B = W^T W                      (once)
//   repeat: Z = B V ; G = Z^T Z ; M = chol(G)^{-T} ; V = Z M   (CholeskyQR)
//   S = V^T B V ; S = U diag(theta) U^T (Jacobi) ; V1 = V U[:, top r]
// The GEMMs are fp32 FFMA (the basis is a subspace estimate; fp32 keeps
// the Gram matrices usable for the Cholesky). The k x k Cholesky, the
// triangular inverse and the Rayleigh-Ritz eigensolve run in fp64, one CTA
// per matrix, so a whole refresh never round-trips through the host.
#pragma once
#include "common.cuh"

namespace mecefo {

struct SubGemmJob {
  const float* a;  // A(m, kk) = a_kmajor ? a[m * lda + kk] : a[kk * lda + m]
  int64_t lda;
  const float* b;  // B(kk, n) = b[kk * ldb + n]
  int64_t ldb;
  float* c;        // C(m, n) = c[m * ldc + n] (+ split * c_split for split-K partials)
  int64_t ldc;
  int64_t c_split;
  int M, N, K;
  int a_kmajor;
  int tiles_n, tiles_mn;
  int tile0;       // first global tile of this job
  int vec;         // 16-byte aligned operands: float4 loads
  int ksplit, kchunk;
};

constexpr int SG_TM = 64, SG_TN = 64, SG_TK = 16, SG_THREADS = 256;

__device__ __forceinline__ float4 sg_load4(const float* p, int64_t idx, bool ok4, int valid) {
  if (ok4 && valid >= 4) return *reinterpret_cast<const float4*>(p + idx);
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid > 0) r.x = p[idx];
  if (valid > 1) r.y = p[idx + 1];
  if (valid > 2) r.z = p[idx + 2];
  if (valid > 3) r.w = p[idx + 3];
  return r;
}

// C = A B for a list of jobs; blockIdx.x indexes the union of all jobs'
// (split, tile) pairs. 64 x 64 tiles, 4 x 4 outputs per thread, register
// prefetch of the next k-slice + double-buffered shared memory: one barrier
// per 16-wide k-step.
__global__ void __launch_bounds__(SG_THREADS) subspace_gemm_kernel(const SubGemmJob* __restrict__ jobs, int njobs) {
  __shared__ __align__(16) float As[2][SG_TK][SG_TM + 4];
  __shared__ __align__(16) float Bs[2][SG_TK][SG_TN + 4];
  int lo = 0, hi = njobs - 1;  // last job with tile0 <= blockIdx.x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const SubGemmJob j = jobs[lo];
  const int t = blockIdx.x - j.tile0;
  const int split = t / j.tiles_mn, tt = t % j.tiles_mn;
  const int m0 = (tt / j.tiles_n) * SG_TM, n0 = (tt % j.tiles_n) * SG_TN;
  const int kbeg = split * j.kchunk, kend = min(j.K, kbeg + j.kchunk);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const bool v4 = j.vec != 0;
  // per-thread load coordinates
  const int ak_r = tid >> 2, ak_k = (tid & 3) * 4;   // A K-major: row, k
  const int am_k = tid >> 4, am_r = (tid & 15) * 4;  // A M-major: k, row
  const int b_k = tid >> 4, b_c = (tid & 15) * 4;    // B: k, col
  float4 ra, rb;
  auto load = [&](int k0) {
    ra = make_float4(0.f, 0.f, 0.f, 0.f);
    rb = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j.a_kmajor) {
      if (m0 + ak_r < j.M) ra = sg_load4(j.a, (int64_t)(m0 + ak_r) * j.lda + k0 + ak_k, v4, kend - k0 - ak_k);
    } else if (k0 + am_k < kend) {
      ra = sg_load4(j.a, (int64_t)(k0 + am_k) * j.lda + m0 + am_r, v4, j.M - m0 - am_r);
    }
    if (k0 + b_k < kend) rb = sg_load4(j.b, (int64_t)(k0 + b_k) * j.ldb + n0 + b_c, v4, j.N - n0 - b_c);
  };
  auto store = [&](int buf) {
    if (j.a_kmajor) {
      As[buf][ak_k][ak_r] = ra.x; As[buf][ak_k + 1][ak_r] = ra.y;
      As[buf][ak_k + 2][ak_r] = ra.z; As[buf][ak_k + 3][ak_r] = ra.w;
    } else {
      *reinterpret_cast<float4*>(&As[buf][am_k][am_r]) = ra;
    }
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_c]) = rb;
  };
  float acc[4][4] = {};
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  int buf = 0;
  for (int k0 = kbeg; k0 < kend; k0 += SG_TK) {
    const bool more = k0 + SG_TK < kend;
    if (more) load(k0 + SG_TK);
#pragma unroll
    for (int kk = 0; kk < SG_TK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  float* C = j.c + (int64_t)split * j.c_split;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= j.M) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gn = n0 + tx * 4 + q;
      if (gn < j.N) C[(int64_t)gm * j.ldc + gn] = acc[i][q];
    }
  }
}

// Row stride (in elements) of the k x k fp64/fp32 work matrices: odd, so
// the column accesses of one warp (consecutive rows) hit distinct banks.
__device__ __forceinline__ int sub_ld(int k) { return k | 1; }

__device__ __forceinline__ double sub_block_sum(double v, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid < 32) {
    double x = tid < (nt >> 5) ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (tid == 0) red[0] = x;
  }
  __syncthreads();
  return red[0];
}

constexpr int SUB_SMALL_THREADS = 1024;

// M = L^{-T} with L L^T = sym(G) (fp64), one CTA per matrix. G and M are
// kmax x kmax (ld kmax); only the leading k x k block is used and M's
// padding is written as zero. `A` (k x ld doubles + k) is dynamic shared
// memory when it fits, else the global scratch slice (scratch_stride
// doubles per matrix).
__global__ void __launch_bounds__(SUB_SMALL_THREADS) subspace_chol_inv_kernel(
    const float* __restrict__ G, float* __restrict__ Mo, const int* __restrict__ ks, int kmax,
    double* __restrict__ scratch, int use_smem, size_t scratch_stride, int nsplit, size_t split_stride) {
  extern __shared__ double sm_d[];
  __shared__ double red[32];
  const int job = blockIdx.x, k = ks[job], ld = sub_ld(k), tid = threadIdx.x, nt = blockDim.x;
  double* A = use_smem ? sm_d : scratch + (size_t)job * scratch_stride;
  double* dinv = A + (size_t)k * ld;
  const float* g = G + (size_t)job * kmax * kmax;
  float* m = Mo + (size_t)job * kmax * kmax;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  double tr = 0.0;
  for (int i = warp; i < k; i += nw)  // symmetrised sum of the split-K partials
    for (int l = lane; l < k; l += 32) {
      double v = 0.0;
      for (int sp = 0; sp < nsplit; ++sp)
        v += (double)g[sp * split_stride + (size_t)i * kmax + l] + (double)g[sp * split_stride + (size_t)l * kmax + i];
      v *= 0.5;
      A[i * ld + l] = v;
      if (i == l) tr += v;
    }
  const double trace = sub_block_sum(tr, red);
  // pivot floor: a (numerically) rank-deficient block stays factorable
  const double floor_ = trace > 0.0 ? 1e-12 * trace / k : 1.0;
  for (int jj = 0; jj < k; ++jj) {
    double d = A[jj * ld + jj];
    d = sqrt(d > floor_ ? d : floor_);
    const double id = 1.0 / d;
    // column jj below the pivot; the pivot itself is rewritten after the
    // barrier that follows every thread's read of it
    for (int i = jj + 1 + tid; i < k; i += nt) A[i * ld + jj] *= id;
    __syncthreads();
    if (tid == 0) A[jj * ld + jj] = d;
    for (int i = jj + 1 + warp; i < k; i += nw) {  // trailing lower triangle, a warp per row
      const double lij = A[i * ld + jj];
      for (int l = jj + 1 + lane; l <= i; l += 32) A[i * ld + l] -= lij * A[l * ld + jj];
    }
    __syncthreads();
  }
  for (int i = tid; i < k; i += nt) dinv[i] = 1.0 / A[i * ld + i];
  __syncthreads();
  // X = L^{-1} by forward substitution: a quad of lanes owns column c and
  // splits each dot product; X[i][c] (i > c) lives in the free upper
  // triangle at A[c][i], X[c][c] in dinv.
  // Warp-uniform loops (the quad shuffles need every lane present): a warp
  // owns columns [cb, cb + 8), the i loop starts at the warp's first column.
  const int quad = tid & 3;
  for (int cb = (tid >> 5) * 8; cb < k; cb += (nt >> 5) * 8) {
    const int c = cb + (lane >> 2);
    const bool valid = c < k;
    const double xc = valid ? dinv[c] : 0.0;
    for (int i = cb + 1; i < k; ++i) {
      const bool act = valid && i > c;
      double s = 0.0;
      if (act)
        for (int q = c + 1 + quad; q < i; q += 4) s += A[i * ld + q] * A[c * ld + q];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (act && quad == 0) A[c * ld + i] = -(A[i * ld + c] * xc + s) * dinv[i];
      __syncwarp();
    }
  }
  __syncthreads();
  // M = X^T: M[c][i] = X[i][c] (upper triangular)
  for (int e = tid; e < kmax * kmax; e += nt) {
    const int c = e / kmax, i = e % kmax;
    float v = 0.f;
    if (c < k && i < k && i >= c) v = (float)(i == c ? dinv[c] : A[c * ld + i]);
    m[e] = v;
  }
}

// Rayleigh-Ritz on the device (linalg.py:124-129): eigen-decomposition of
// S = V^T B V (k x k) by parallel cyclic Jacobi — round-robin ordering, k/2
// disjoint rotations per round, fp64 S, fp32 eigenvector accumulator — then
// the eigenvectors of the r largest eigenvalues, in descending order, as the
// columns of Ur (k x r, ld r). One CTA per matrix; S (ld kmax) is read from
// the Gram buffer. The work matrices live in dynamic shared memory when they
// fit, else in the global scratch slice (same layout).
__global__ void __launch_bounds__(SUB_SMALL_THREADS) subspace_ritz_kernel(
    const float* __restrict__ Sg, float* __restrict__ Ur, float* __restrict__ theta_out, const int* __restrict__ ks,
    const int* __restrict__ rs, int kmax, int rmax, void* __restrict__ scratch, size_t scratch_stride, int use_smem,
    int nsplit, size_t split_stride) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  __shared__ double red[32];
  __shared__ int rot_p[256], rot_q[256];
  __shared__ double rot_c[256], rot_s[256];
  const int job = blockIdx.x, k = ks[job], r = rs[job], ld = sub_ld(k), tid = threadIdx.x, nt = blockDim.x;
  unsigned char* base = use_smem ? sm_raw : static_cast<unsigned char*>(scratch) + (size_t)job * scratch_stride;
  double* S = reinterpret_cast<double*>(base);
  float* U = reinterpret_cast<float*>(base + (size_t)k * ld * 8);
  const float* sg = Sg + (size_t)job * kmax * kmax;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int i = warp; i < k; i += nw)
    for (int l = lane; l < k; l += 32) {
      double v = 0.0;
      for (int sp = 0; sp < nsplit; ++sp)
        v += (double)sg[sp * split_stride + (size_t)i * kmax + l] + (double)sg[sp * split_stride + (size_t)l * kmax + i];
      S[i * ld + l] = 0.5 * v;
      U[i * ld + l] = i == l ? 1.f : 0.f;
    }
  const int kp = (k + 1) & ~1;  // players (one dummy when k is odd)
  const int npair = kp / 2;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = warp; i < k; i += nw)
      for (int l = lane; l < k; l += 32) {
        const double v = S[i * ld + l] * S[i * ld + l];
        tot += v;
        if (i != l) off += v;
      }
    off = sub_block_sum(off, red);
    tot = sub_block_sum(tot, red);
    if (off <= 1e-18 * tot || tot == 0.0) break;  // off-diagonal < 1e-9 relative (Frobenius)
    for (int rd = 0; rd < kp - 1; ++rd) {
      for (int i = tid; i < npair; i += nt) {  // pair i of this round (circle method)
        int a, b;
        if (i == 0) { a = 0; b = rd + 1; }
        else { a = ((i + rd) % (kp - 1)) + 1; b = ((kp - 1 - i + rd) % (kp - 1)) + 1; }
        double c = 1.0, sn = 0.0;
        const int p = min(a, b), q = max(a, b);
        if (q < k) {
          const double apq = S[p * ld + q];
          // negligible against the diagonal: no rotation (quadratic
          // convergence leaves most pairs here in the last sweep)
          if (fabs(apq) > 1e-300 && fabs(apq) > 1e-15 * sqrt(fabs(S[p * ld + p] * S[q * ld + q]))) {
            const double tau = (S[q * ld + q] - S[p * ld + p]) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            sn = t * c;
          }
        }
        rot_p[i] = p; rot_q[i] = q; rot_c[i] = c; rot_s[i] = sn;
      }
      __syncthreads();
      // S <- S J (columns p, q of every row); U <- U J
      for (int i = warp; i < npair; i += nw) {  // a warp per rotation, lanes over rows
        const int p = rot_p[i], q = rot_q[i];
        const double sn = rot_s[i];
        if (q >= k || sn == 0.0) continue;
        const double c = rot_c[i];
        for (int row = lane; row < k; row += 32) {
          const double xp = S[row * ld + p], xq = S[row * ld + q];
          S[row * ld + p] = c * xp - sn * xq;
          S[row * ld + q] = sn * xp + c * xq;
          const float up = U[row * ld + p], uq = U[row * ld + q];
          U[row * ld + p] = (float)(c * up - sn * uq);
          U[row * ld + q] = (float)(sn * up + c * uq);
        }
      }
      __syncthreads();
      // S <- J^T S (rows p, q)
      for (int i = warp; i < npair; i += nw) {  // lanes over columns
        const int p = rot_p[i], q = rot_q[i];
        const double sn = rot_s[i];
        if (q >= k || sn == 0.0) continue;
        const double c = rot_c[i];
        for (int col = lane; col < k; col += 32) {
          const double xp = S[p * ld + col], xq = S[q * ld + col];
          S[p * ld + col] = c * xp - sn * xq;
          S[q * ld + col] = sn * xp + c * xq;
        }
      }
      __syncthreads();
    }
  }
  // descending order of the eigenvalues diag(S); ties broken by index
  float* ur = Ur + (size_t)job * kmax * rmax;
  for (int i = tid; i < k; i += nt) {
    const double ti = S[i * ld + i];
    int pos = 0;
    for (int j = 0; j < k; ++j) {
      const double tj = S[j * ld + j];
      pos += (tj > ti) || (tj == ti && j < i);
    }
    if (pos < r) {
      for (int row = 0; row < k; ++row) ur[(size_t)row * r + pos] = U[row * ld + i];
      if (theta_out) theta_out[(size_t)job * rmax + pos] = (float)ti;
    }
  }
}

}  // namespace mecefo
