// EAMC construction by k-means on device: the reference's
// Lloyd iterations with seeded k-means++ (sketches.py:62-139) over sketch
// vectors in HBM.
//
//  * moeb_row_sqnorms: (x * x).sum(axis=1) with numpy's pairwise summation
//    (blocks of <= 128 with 8 accumulators, halving splits rounded to
//    multiples of 8, identity 0 first) -- bit-identical to the reference.
//  * moeb_sqdist_argmin: squared distances max((|x|^2 - 2 x.c) + |c|^2, 0)
//    (_squared_distances, sketches.py:62-69) for all (vector, centroid)
//    pairs as an fp64 register-tiled GEMM (64 x 64 tiles, 4 x 4 per thread,
//    K staged through shared memory) with the argmin fused into the
//    epilogue: per vector the first minimal centroid and its distance; the
//    n x k matrix is never materialised. The dot products use a different
//    summation order than the reference's BLAS (ulp-level differences).
//  * moeb_sqdist_update: k-means++ step, d2 = minimum(d2, dist(x, c)) for one
//    new centroid (warp per vector, coalesced).
//  * moeb_cluster_means: members.mean(axis=0) per cluster with the members
//    in index order and numpy's axis-0 accumulation order (sequential), then
//    one division by the count -- bit-identical given the same assignments.
#include "common.cuh"

namespace {

// numpy pairwise_sum of x*x over a[0..n) with stride 1 (numpy/_core/src/
// umath/loops_utils.h.src): n < 8 sequential; n <= 128 eight accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; otherwise the
// two halves split at n/2 rounded down to a multiple of 8. Products and sums
// are separately rounded (no FMA contraction), as numpy's x * x then sum.
__device__ double pairwise_sq_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, __dmul_rn(a[i], a[i]));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(a[j], a[j]);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(a[i + j], a[i + j]));
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn(a[i], a[i]));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sq_sum(a, n2) + pairwise_sq_sum(a + n2, n - n2);
}

__global__ void k_row_sqnorms(const double* X, int64_t n, int64_t D, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = 0.0 + pairwise_sq_sum(X + i * D, D);  // reduce starts from the identity
}

constexpr int TB = 64;   // tile rows (vectors) and columns (centroids)
constexpr int TK = 16;   // K chunk
constexpr int kThr = 256;

// Per CTA: 64 vectors x all centroids (loop over centroid tiles), running
// first-min per vector held in shared memory.
__global__ void __launch_bounds__(kThr) k_sqdist_argmin(const double* __restrict__ X,
                                                        const double* __restrict__ xn,
                                                        const double* __restrict__ C,
                                                        const double* __restrict__ cn, int64_t n,
                                                        int k, int64_t D, int64_t* out_idx,
                                                        double* out_d2) {
  __shared__ double As[TK][TB + 1];
  __shared__ double Bs[TK][TB + 1];
  __shared__ double best_v[TB][16];
  __shared__ int best_i[TB][16];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;  // 16 x 16 threads, 4 x 4 each
  const int64_t row0 = (int64_t)blockIdx.x * TB;
  double bv[4];
  int bi[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    bv[a] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    bi[a] = 0;
  }
  for (int c0 = 0; c0 < k; c0 += TB) {
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int64_t k0 = 0; k0 < D; k0 += TK) {
      // load 64 x 16 of X and of C (transposed into [k][row])
      for (int e = tid; e < TB * TK; e += kThr) {
        const int r = e / TK, kk = e % TK;
        const int64_t gr = row0 + r, gk = k0 + kk;
        As[kk][r] = (gr < n && gk < D) ? X[gr * D + gk] : 0.0;
        const int64_t gc = c0 + r;
        Bs[kk][r] = (gc < k && gk < D) ? C[gc * D + gk] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        double av[4], bw[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][tr + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bw[b] = Bs[kk][tc + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(2.0 * av[a], bw[b], acc[a][b]);
      }
      __syncthreads();
    }
    // epilogue: distances of this tile, first-min per row (columns ascending)
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t gr = row0 + tr + 16 * a;
      const double x2 = gr < n ? xn[gr] : 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int gc = c0 + tc + 16 * b;
        if (gc < k) {
          double d = (x2 - acc[a][b]) + cn[gc];
          d = d > 0.0 ? d : 0.0;  // np.maximum(sq, 0.0)
          if (d < bv[a] || (d == bv[a] && gc < bi[a])) {
            bv[a] = d;
            bi[a] = gc;
          }
        }
      }
    }
  }
  // combine the 16 column-threads of each row: min value, lowest index
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    best_v[tr + 16 * a][tc] = bv[a];
    best_i[tr + 16 * a][tc] = bi[a];
  }
  __syncthreads();
  if (tid < TB) {
    const int64_t gr = row0 + tid;
    double v = best_v[tid][0];
    int ix = best_i[tid][0];
    for (int c = 1; c < 16; ++c) {
      const double w = best_v[tid][c];
      const int j = best_i[tid][c];
      if (w < v || (w == v && j < ix)) {
        v = w;
        ix = j;
      }
    }
    if (gr < n) {
      out_idx[gr] = ix;
      if (out_d2) out_d2[gr] = v;
    }
  }
}

// d2[i] = minimum(d2[i], max((xn[i] - 2 x_i . c) + cn, 0)); warp per vector.
__global__ void k_sqdist_update(const double* __restrict__ X, const double* __restrict__ xn,
                                const double* __restrict__ c, const double* cn_ptr, int64_t n,
                                int64_t D, int init, double* d2) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const double* x = X + w * D;
  double s = 0.0;
  for (int64_t j = lane; j < D; j += 32) s = fma(2.0 * x[j], c[j], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    double d = (xn[w] - s) + *cn_ptr;
    d = d > 0.0 ? d : 0.0;
    if (init) d2[w] = d;
    else d2[w] = d < d2[w] ? d : d2[w];  // np.minimum (no NaNs here)
  }
}

// cent[j][d] = sum_{m in members(j), index order} X[m][d] / count(j);
// clusters without members keep their centroid (sketches.py:131-134).
__global__ void k_cluster_means(const double* __restrict__ X, const int64_t* __restrict__ members,
                                const int64_t* __restrict__ offs, int k, int64_t D,
                                double* cent) {
  const int j = blockIdx.y;
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k || d >= D) return;
  const int64_t a = offs[j], b = offs[j + 1];
  if (b == a) return;
  double s = 0.0;
  for (int64_t m = a; m < b; ++m) s += X[members[m] * D + d];
  cent[(int64_t)j * D + d] = s / (double)(b - a);
}

}  // namespace

extern "C" {

int moeb_row_sqnorms(const double* X, int64_t n, int64_t D, double* out, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(n >= 0 && D >= 1 && (n == 0 || (X && out)), "bad argument");
  if (n == 0) return MOEB_OK;
  k_row_sqnorms<<<(unsigned)((n + 127) / 128), 128, 0, moeb::as_stream(stream)>>>(X, n, D, out);
  return moeb::check_launch("k_row_sqnorms");
}

int moeb_sqdist_argmin(const double* X, const double* xn, const double* C, const double* cn,
                       int64_t n, int k, int64_t D, int64_t* out_idx, double* out_d2,
                       void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(n >= 0 && k >= 1 && D >= 1, "bad shape");
  MOEB_REQUIRE(n == 0 || (X && xn && C && cn && out_idx), "null argument");
  if (n == 0) return MOEB_OK;
  k_sqdist_argmin<<<(unsigned)((n + TB - 1) / TB), kThr, 0, moeb::as_stream(stream)>>>(
      X, xn, C, cn, n, k, D, out_idx, out_d2);
  return moeb::check_launch("k_sqdist_argmin");
}

int moeb_sqdist_update(const double* X, const double* xn, const double* c, const double* cn,
                       int64_t n, int64_t D, int init, double* d2, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(n >= 0 && D >= 1 && (n == 0 || (X && xn && c && cn && d2)), "bad argument");
  if (n == 0) return MOEB_OK;
  const int64_t threads = n * 32;
  k_sqdist_update<<<(unsigned)((threads + 255) / 256), 256, 0, moeb::as_stream(stream)>>>(
      X, xn, c, cn, n, D, init, d2);
  return moeb::check_launch("k_sqdist_update");
}

int moeb_cluster_means(const double* X, const int64_t* members, const int64_t* offs, int k,
                       int64_t D, double* centroids, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(X && members && offs && centroids && k >= 1 && D >= 1, "bad argument");
  const dim3 grid((unsigned)((D + 127) / 128), (unsigned)k);
  k_cluster_means<<<grid, 128, 0, moeb::as_stream(stream)>>>(X, members, offs, k, D, centroids);
  return moeb::check_launch("k_cluster_means");
}

}  // extern "C"
