// Converged projection refresh on the device (approx.py:66-87 over every
// due (layer, kind); each matrix is linalg.py:97-142): float64 throughout so
// the reference's stopping rule, residual <= tol * theta_max with tol = 1e-9
// (harness.py:367), is attainable.
//
// Kernels (all batched over the matrices of one refresh, one launch per phase):
//   dgemm_batched_kernel    C = alpha op(A) B + beta Cin + gamma Din (fp64
//                           DMMA m8n8k4 tensor-core tiles; fp32 or fp64
//                           operands; optional split-K with fp64 atomics)
//   cholqr_kernel           M = D^-1/2 L^-T with L L^T = D^-1/2 (Z^T Z) D^-1/2
//                           (Jacobi-preconditioned CholeskyQR: Z M is
//                           orthonormal), one CTA per matrix
//   jacobi_eig_kernel       S = U diag(theta) U^T by parallel cyclic Jacobi,
//                           fp64 S and U, eigenpairs sorted descending
//   residual_kernel         max_j<r ||B v_j - theta_j v_j|| / theta_0
//                           (linalg.py:131-135)
//   axpby_kernel_f64        Chebyshev first step X1 = a X + b Y
#pragma once
#include "common.cuh"

namespace mecefo {
namespace rf {

struct DJob {
  const void* a;  // A(m, k) = a_kmajor ? a[m * lda + k] : a[k * lda + m]
  int64_t lda;
  const void* b;  // B(k, n) = b_kmajor ? b[n * ldb + k] : b[k * ldb + n]
  int64_t ldb;
  double* c;      // C(m, n) = c[m * ldc + n]
  int64_t ldc;
  const double* cin;  // + beta * Cin(m, n) (ld ldcin), optional
  int64_t ldcin;
  const double* din;  // + gamma * Din(m, n) (ld lddin), optional
  int64_t lddin;
  double alpha, beta, gamma;
  int M, N, K;
  int a_kmajor, b_kmajor, a_f32, b_f32;
  int tiles_n, tiles_mn, tile0;
  int ksplit, kchunk;  // ksplit > 1: c += alpha * partial via atomicAdd (c pre-zeroed)
};

constexpr int DG_BM = 64, DG_BN = 64, DG_BK = 16, DG_THREADS = 128, DG_LD = DG_BM + 8;

__device__ __forceinline__ double ld_elem(const void* p, int64_t i, int f32) {
  return f32 ? (double)reinterpret_cast<const float*>(p)[i] : reinterpret_cast<const double*>(p)[i];
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 64 x 64 output tile per CTA, 4 warps of 32 x 32 (4 x 4 DMMA 8x8 tiles),
// k-slices of 16 staged through registers into double-buffered shared memory
// (stored m/n-fastest: conflict-free; fragment reads hit 16 distinct 8-byte
// banks twice — the 2-wavefront minimum for 32 doubles).
__global__ void __launch_bounds__(DG_THREADS) dgemm_batched_kernel(const DJob* __restrict__ jobs, int njobs) {
  __shared__ __align__(16) double As[2][DG_BK][DG_LD];
  __shared__ __align__(16) double Bs[2][DG_BK][DG_LD];
  int lo = 0, hi = njobs - 1;  // last job with tile0 <= blockIdx.x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const DJob& j = jobs[lo];
  const int t = blockIdx.x - j.tile0;
  const int split = t / j.tiles_mn, tt = t % j.tiles_mn;
  const int m0 = (tt / j.tiles_n) * DG_BM, n0 = (tt % j.tiles_n) * DG_BN;
  const int kbeg = split * j.kchunk, kend = min(j.K, kbeg + j.kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int M = j.M, N = j.N;
  const void* A = j.a;
  const void* B = j.b;
  const int64_t lda = j.lda, ldb = j.ldb;
  const int akm = j.a_kmajor, bkm = j.b_kmajor, af = j.a_f32, bf = j.b_f32;
  double ra[8], rb[8];
  // element e = q * 128 + tid of the 16 x 64 slice: row (k) = e / 64, col (m or n) = e % 64
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = q * DG_THREADS + tid, kk = e >> 6, mm = e & 63;
      const int gk = k0 + kk, gm = m0 + mm, gn = n0 + mm;
      ra[q] = (gk < kend && gm < M) ? ld_elem(A, akm ? (int64_t)gm * lda + gk : (int64_t)gk * lda + gm, af) : 0.0;
      rb[q] = (gk < kend && gn < N) ? ld_elem(B, bkm ? (int64_t)gn * ldb + gk : (int64_t)gk * ldb + gn, bf) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = q * DG_THREADS + tid, kk = e >> 6, mm = e & 63;
      As[buf][kk][mm] = ra[q];
      Bs[buf][kk][mm] = rb[q];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  int buf = 0;
  const int fr = lane & 3, fc = lane >> 2;
  for (int k0 = kbeg; k0 < kend; k0 += DG_BK) {
    const bool more = k0 + DG_BK < kend;
    if (more) load(k0 + DG_BK);
#pragma unroll
    for (int ks = 0; ks < DG_BK; ks += 4) {
      double af4[4], bf4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af4[i] = As[buf][ks + fr][wm + i * 8 + fc];
#pragma unroll
      for (int q = 0; q < 4; ++q) bf4[q] = Bs[buf][ks + fr][wn + q * 8 + fc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma(acc[i][q][0], acc[i][q][1], af4[i], bf4[q]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  // epilogue: thread holds C[row][col0 .. col0 + 1] of every 8x8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + wm + i * 8 + fc;
    if (gm >= M) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn + q * 8 + 2 * fr + h;
        if (gn >= N) continue;
        double v = j.alpha * acc[i][q][h];
        double* dst = j.c + (int64_t)gm * j.ldc + gn;
        if (j.ksplit > 1) {
          atomicAdd(dst, v);
        } else {
          if (j.cin) v += j.beta * j.cin[(int64_t)gm * j.ldcin + gn];
          if (j.din) v += j.gamma * j.din[(int64_t)gm * j.lddin + gn];
          *dst = v;
        }
      }
    }
  }
}

// Per-matrix descriptor of the small (k x k) phases.
struct SmallJob {
  double* g;      // k x k (ld k): Gram / Rayleigh quotient input
  double* m;      // k x k (ld k): output (CholeskyQR M, or eigenvectors U sorted)
  double* theta;  // k: eigenvalues, descending (jacobi only)
  double* scratch;  // global fallback for the work matrices
  int k;
  int use_smem;
  double tol2;      // jacobi: stop when off-diagonal mass <= tol2 * total (Frobenius^2)
  double* stat;     // jacobi (optional): += sweeps run
};

__device__ __forceinline__ double blk_sum_d(double v, double* red) {
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

constexpr int RF_SMALL_THREADS = 1024;

// Jacobi-preconditioned CholeskyQR: with D = diag(G), factor
// D^-1/2 G D^-1/2 = L L^T and return M = D^-1/2 L^-T, so Z M has orthonormal
// columns (Z^T Z = G). The filtered blocks have near-orthogonal columns of
// very different norms; the diagonal scaling keeps the factorisation well
// conditioned. One CTA per matrix; work matrix ld = k | 1 (odd: column walks
// of a warp hit distinct banks).
__global__ void __launch_bounds__(RF_SMALL_THREADS) cholqr_kernel(const SmallJob* __restrict__ jobs) {
  extern __shared__ double rf_smem[];
  const SmallJob jb = jobs[blockIdx.x];
  const int k = jb.k, ld = k | 1, tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  double* A = jb.use_smem ? rf_smem : jb.scratch;
  double* dsc = A + (size_t)k * ld;  // D^-1/2
  double* dinv = dsc + k;            // 1 / L_ii
  for (int i = tid; i < k; i += nt) {
    const double d = 0.5 * (jb.g[(size_t)i * k + i] + jb.g[(size_t)i * k + i]);
    dsc[i] = d > 0.0 ? 1.0 / sqrt(d) : 0.0;
  }
  __syncthreads();
  for (int i = warp; i < k; i += nw)
    for (int l = lane; l < k; l += 32)
      A[i * ld + l] = 0.5 * (jb.g[(size_t)i * k + l] + jb.g[(size_t)l * k + i]) * dsc[i] * dsc[l];
  __syncthreads();
  const double floor_ = 1e-30;  // scaled diagonal is ~1; a null column stays factorable
  for (int jj = 0; jj < k; ++jj) {
    double d = A[jj * ld + jj];
    d = sqrt(d > floor_ ? d : floor_);
    const double id = 1.0 / d;
    for (int i = jj + 1 + tid; i < k; i += nt) A[i * ld + jj] *= id;
    __syncthreads();
    if (tid == 0) A[jj * ld + jj] = d;
    for (int i = jj + 1 + warp; i < k; i += nw) {
      const double lij = A[i * ld + jj];
      for (int l = jj + 1 + lane; l <= i; l += 32) A[i * ld + l] -= lij * A[l * ld + jj];
    }
    __syncthreads();
  }
  for (int i = tid; i < k; i += nt) dinv[i] = 1.0 / A[i * ld + i];
  __syncthreads();
  // X = L^{-1} by forward substitution; X[i][c] (i > c) stored at A[c][i]
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
  // M = D^-1/2 X^T: M[r][c] = dsc[r] * X[c][r] (upper triangular)
  for (int e = tid; e < k * k; e += nt) {
    const int r = e / k, c = e % k;
    double v = 0.0;
    if (c >= r) v = dsc[r] * (c == r ? dinv[r] : A[r * ld + c]);
    jb.m[e] = v;
  }
}

// Rayleigh-Ritz eigensolve (linalg.py:124-129): S = U diag(theta) U^T by
// parallel cyclic Jacobi (round-robin pairs, k/2 disjoint rotations per
// round), fp64 S and U; sweeps until the off-diagonal mass is below 1e-30 of
// the total (relative 1e-15, Frobenius). Output: theta descending and U's
// columns in that order (jb.m, k x k, ld k).
// S is kept as its packed upper triangle and the accumulated rotation
// transposed (Ut: rotations update two contiguous rows), both in shared
// memory when 8 (k(k+1)/2 + k^2) bytes fit (k <= 132), else in the global
// scratch. One round = rotation parameters, then every (rotation, rotation)
// 2x2 block of S updated as J1^T B J2 by one thread (a single pass, no
// row/column phases) and the Ut rows rotated.
__device__ __forceinline__ int tri_off(int i, int k) { return i * k - (i * (i - 1)) / 2; }
__device__ __forceinline__ int tri_idx(int i, int j, int k) {  // symmetric access
  return i <= j ? tri_off(i, k) + (j - i) : tri_off(j, k) + (i - j);
}

__global__ void __launch_bounds__(RF_SMALL_THREADS) jacobi_eig_kernel(const SmallJob* __restrict__ jobs) {
  extern __shared__ double rf_smem[];
  __shared__ double red[32];
  __shared__ int rot_p[512], rot_q[512];  // k <= 1024
  __shared__ double rot_c[512], rot_s[512];
  const SmallJob jb = jobs[blockIdx.x];
  const int k = jb.k, tid = threadIdx.x, nt = blockDim.x;
  const int ntri = k * (k + 1) / 2;
  double* S = jb.use_smem ? rf_smem : jb.scratch;
  double* Ut = S + ((ntri + 1) & ~1);  // k x k, ld k: Ut[c][row] = U[row][c]
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, l = e % k;
    if (i <= l) S[tri_off(i, k) + (l - i)] = 0.5 * (jb.g[(size_t)i * k + l] + jb.g[(size_t)l * k + i]);
    Ut[e] = i == l ? 1.0 : 0.0;
  }
  __syncthreads();
  const int kp = (k + 1) & ~1;
  const int npair = kp / 2;
  const int nblk = npair * (npair + 1) / 2;
  // this thread's fixed work items of every round (rotation slots are
  // positional, so the (i1, i2) block and (rotation, column) maps never change)
  constexpr int MAXB = 3, MAXU = 9;
  const bool fast = nblk <= MAXB * nt && npair * k <= MAXU * nt;
  int bi1[MAXB], bi2[MAXB], ui[MAXU], uc[MAXU];
  if (fast) {
#pragma unroll
    for (int t = 0; t < MAXB; ++t) {
      const int bi = tid + t * nt;
      bi1[t] = -1;
      if (bi < nblk) {
        int i1 = (int)((2.0 * npair + 1.0 - sqrt((2.0 * npair + 1.0) * (2.0 * npair + 1.0) - 8.0 * bi)) * 0.5);
        while (i1 > 0 && tri_off(i1, npair) > bi) --i1;
        while (i1 + 1 < npair && tri_off(i1 + 1, npair) <= bi) ++i1;
        bi1[t] = i1;
        bi2[t] = i1 + (bi - tri_off(i1, npair));
      }
    }
#pragma unroll
    for (int t = 0; t < MAXU; ++t) {
      const int e = tid + t * nt;
      ui[t] = e < npair * k ? e / k : -1;
      uc[t] = e < npair * k ? e % k : 0;
    }
  }
  auto block = [&](int i1, int i2) {
    const double s1 = rot_s[i1], s2 = rot_s[i2];
    if (s1 == 0.0 && s2 == 0.0) return;
    const double c1 = rot_c[i1], c2 = rot_c[i2];
    const int p1 = rot_p[i1], q1 = rot_q[i1], p2 = rot_p[i2], q2 = rot_q[i2];
    if (i1 == i2) {  // diagonal block (p, q): becomes diag(app', aqq')
      const int ip = tri_off(p1, k), iq = tri_off(q1, k), ipq = ip + (q1 - p1);
      const double app = S[ip], aqq = S[iq], apq = S[ipq];
      S[ip] = c1 * c1 * app - 2.0 * c1 * s1 * apq + s1 * s1 * aqq;
      S[iq] = s1 * s1 * app + 2.0 * c1 * s1 * apq + c1 * c1 * aqq;
      S[ipq] = 0.0;
      return;
    }
    const bool hq1 = q1 < k, hq2 = q2 < k;
    const int e00 = tri_idx(p1, p2, k);
    const int e01 = hq2 ? tri_idx(p1, q2, k) : 0;
    const int e10 = hq1 ? tri_idx(q1, p2, k) : 0;
    const int e11 = (hq1 && hq2) ? tri_idx(q1, q2, k) : 0;
    const double b00 = S[e00], b01 = hq2 ? S[e01] : 0.0, b10 = hq1 ? S[e10] : 0.0,
                 b11 = (hq1 && hq2) ? S[e11] : 0.0;
    const double x00 = b00 * c2 - b01 * s2, x01 = b00 * s2 + b01 * c2;  // X = B J2
    const double x10 = b10 * c2 - b11 * s2, x11 = b10 * s2 + b11 * c2;
    S[e00] = c1 * x00 - s1 * x10;  // J1^T X
    if (hq2) S[e01] = c1 * x01 - s1 * x11;
    if (hq1) S[e10] = s1 * x00 + c1 * x10;
    if (hq1 && hq2) S[e11] = s1 * x01 + c1 * x11;
  };
  auto urot = [&](int i, int col) {
    const double sn = rot_s[i];
    if (sn == 0.0) return;
    const double c = rot_c[i];
    double* up = Ut + (size_t)rot_p[i] * k + col;
    double* uq = Ut + (size_t)rot_q[i] * k + col;
    const double a0 = *up, b0 = *uq;
    *up = c * a0 - sn * b0;
    *uq = sn * a0 + c * b0;
  };
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = tid >> 5; i < k; i += nt >> 5) {  // a warp per packed row
      const double* row = S + tri_off(i, k);
      for (int l = (tid & 31); l < k - i; l += 32) {
        const double v = row[l] * row[l];
        tot += l == 0 ? v : 2.0 * v;
        if (l) off += 2.0 * v;
      }
    }
    off = blk_sum_d(off, red);
    tot = blk_sum_d(tot, red);
    if (off <= jb.tol2 * tot || tot == 0.0) {
      if (tid == 0 && jb.stat) *jb.stat += sweep;
      break;
    }
    // threshold Jacobi: a pair whose a_pq^2 is below tol2 * total / k^2 is
    // not rotated (all such pairs together hold less than the stopping mass),
    // so the nearly diagonal Ritz blocks of later iterations cost few rotations
    const double thr2 = jb.tol2 * tot / ((double)k * (double)k);
    for (int rd = 0; rd < kp - 1; ++rd) {
      for (int i = tid; i < npair; i += nt) {
        int a, b;
        if (i == 0) { a = 0; b = rd + 1; }
        else { a = ((i + rd) % (kp - 1)) + 1; b = ((kp - 1 - i + rd) % (kp - 1)) + 1; }
        double c = 1.0, sn = 0.0;
        const int p = min(a, b), q = max(a, b);
        if (q < k) {
          const double apq = S[tri_off(p, k) + (q - p)];
          const double app = S[tri_off(p, k)], aqq = S[tri_off(q, k)];
          if (apq * apq > thr2 && fabs(apq) > 1e-17 * sqrt(fabs(app * aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            sn = t * c;
          }
        }
        rot_p[i] = p; rot_q[i] = q; rot_c[i] = c; rot_s[i] = sn;
      }
      __syncthreads();
      if (fast) {
#pragma unroll
        for (int t = 0; t < MAXB; ++t)
          if (bi1[t] >= 0) block(bi1[t], bi2[t]);
#pragma unroll
        for (int t = 0; t < MAXU; ++t)
          if (ui[t] >= 0) urot(ui[t], uc[t]);
      } else {
        for (int bi = tid; bi < nblk; bi += nt) {
          int i1 = (int)((2.0 * npair + 1.0 - sqrt((2.0 * npair + 1.0) * (2.0 * npair + 1.0) - 8.0 * bi)) * 0.5);
          while (i1 > 0 && tri_off(i1, npair) > bi) --i1;
          while (i1 + 1 < npair && tri_off(i1 + 1, npair) <= bi) ++i1;
          block(i1, i1 + (bi - tri_off(i1, npair)));
        }
        for (int e = tid; e < npair * k; e += nt) urot(e / k, e % k);
      }
      __syncthreads();
    }
  }
  // descending order; eigenvector i = column i of U = row i of Ut
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  __syncthreads();
  for (int i = warp; i < k; i += nw) {
    const double ti = S[tri_off(i, k)];
    int pos = 0;
    for (int jx = 0; jx < k; ++jx) {
      const double tj = S[tri_off(jx, k)];
      pos += (tj > ti) || (tj == ti && jx < i);
    }
    if (lane == 0) jb.theta[pos] = ti;
    for (int row = lane; row < k; row += 32) jb.m[(size_t)row * k + pos] = Ut[(size_t)i * k + row];
  }
}

struct ResJob {
  const double* v;   // n x k (ld k): Ritz vectors
  const double* bv;  // n x k (ld k): B v
  const double* theta;
  double* out;       // residual (relative to theta_0)
  int n, k, r;
};

// linalg.py:131-135: max_j<r ||B v_j - theta_j v_j||_2 / max(theta_0, tiny).
// One CTA per matrix; a warp per column, lanes over rows.
__global__ void __launch_bounds__(1024) residual_kernel(const ResJob* __restrict__ jobs) {
  __shared__ double red[32];
  const ResJob jb = jobs[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double worst = 0.0;
  for (int c = warp; c < jb.r; c += nw) {
    const double th = jb.theta[c];
    double s = 0.0;
    for (int i = lane; i < jb.n; i += 32) {
      const double d = jb.bv[(size_t)i * jb.k + c] - th * jb.v[(size_t)i * jb.k + c];
      s += d * d;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    worst = fmax(worst, s);
  }
  if (lane == 0) red[warp] = worst;
  __syncthreads();
  if (threadIdx.x == 0) {
    double w = 0.0;
    for (int i = 0; i < nw; ++i) w = fmax(w, red[i]);
    const double t0 = jb.theta[0];
    *jb.out = sqrt(w) / fmax(t0, 2.2250738585072014e-308);
  }
}

struct AxJob {
  double* out;
  const double* x;
  const double* y;
  double a, b;
  int64_t n;
  int64_t off;  // first element of this job in the launch's virtual range
};

// out = a x + b y (Chebyshev first step, column extraction); grid-stride over
// the concatenated jobs.
__global__ void axpby_f64_kernel(const AxJob* __restrict__ jobs, int njobs, int64_t total) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].off <= v) lo = mid; else hi = mid - 1;
    }
    const AxJob& j = jobs[lo];
    const int64_t i = v - j.off;
    j.out[i] = j.a * j.x[i] + (j.y ? j.b * j.y[i] : 0.0);
  }
}

struct CopyJob {
  float* dst;        // rows x cols (ld ldd) fp32
  const double* src; // rows x ? (ld lds) fp64
  int64_t ldd, lds;
  double* dst64;     // optional fp64 copy (ld ldd)
  const double* scale;  // optional per-column scale (cols)
  int rows, cols;
  int64_t off;
};

// Column block extraction with optional per-column scaling, fp64 -> fp32 (+fp64).
__global__ void extract_cols_kernel(const CopyJob* __restrict__ jobs, int njobs, int64_t total) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].off <= v) lo = mid; else hi = mid - 1;
    }
    const CopyJob& j = jobs[lo];
    const int64_t i = v - j.off;
    const int r = (int)(i / j.cols), c = (int)(i % j.cols);
    double x = j.src[(int64_t)r * j.lds + c];
    if (j.scale) x *= j.scale[c];
    if (j.dst) j.dst[(int64_t)r * j.ldd + c] = (float)x;
    if (j.dst64) j.dst64[(int64_t)r * j.ldd + c] = x;
  }
}

}  // namespace rf
}  // namespace mecefo
