// cmc.cu — N2: construction of the CMC factors L1^m, L2^m on the GPU
// (eq:l1l2).
//
// For every non-text modality m:
//   A_m = X_m S_m^-1 (the f32 smoothed activations the path computes)
//   G = A_m^T A_m: exact int8-slice Gram on the tensor cores (gram.cu), then in f64:
//   eig G = P Lambda P^T (cuSOLVER Dsyevd; MASQ_CMC_EIG=1, else the Cholesky route below)
//   Lambda' = max(Lambda, 0) + eps_rel * lambda_max (reading Q27)
//   dW = S_m W - Q(S_t W) (exact in f64, this file's kernel, from the text codes and scales)
//   M = T dW = diag(sqrt Lambda') P^T dW      (Dgemm + row scaling)
//   C = M M^T (Dsyrk) -> eig: the top-r eigenvectors are the left singular vectors U_r of M and
//   the eigenvalues its squared singular values (only the leading r are needed)
//   L2 = U_r^T M = Sigma_r V_r^T,  L1 = T^-1 U_r = P diag(1/sqrt Lambda') U_r
//   resid (optional) = ||A_m (dW - L1 L2)||_F^2 = <E, G E>, E = dW - L1 L2 (Dsymm + reduction).
// When n < d the same optimum comes from the n x n side: eig(dW^T G' dW) = V Sigma^2 V^T,
// L2 = Sigma_r V_r^T, L1 = dW V_r Sigma_r^-1 (T^-1 M = dW, so no d x d factorisation is needed).
// Default route for n >= d: G' = Lc Lc^T (Cholesky), T = Lc^T (any T with T^T T = G' gives the
// same L1 L2), M = Lc^T dW, U_r from eig(M M^T), L2 = U_r^T M, L1 = Lc^-T U_r.
// Two phases so that token-sharded runs can SUM the Grams between them:
// launch_cmc_gram (per shard / batch, accumulating) and launch_cmc_from_gram.
// cuBLAS / cuSOLVER are plain library linear algebra here (GEMM, SYRK, symmetric eigensolver);
// they are loaded with dlopen on first use so that libmasq.so itself has no link dependency on
// them (a box without them fails this call with MASQ_ERR_UNSUPPORTED, nothing else).
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_bf16.h>
#include <dlfcn.h>

#include <cstdlib>

#include <mutex>

#include "internal.h"

namespace masq {
namespace {

struct LinAlg {
  bool tried = false, ok = false;
  decltype(&cublasCreate_v2) create = nullptr;
  decltype(&cublasSetStream_v2) set_stream = nullptr;
  decltype(&cublasDgemm_v2) dgemm = nullptr;
  decltype(&cublasDsyrk_v2) dsyrk = nullptr;
  decltype(&cublasDsymm_v2) dsymm = nullptr;
  decltype(&cusolverDnCreate) sv_create = nullptr;
  decltype(&cusolverDnSetStream) sv_set_stream = nullptr;
  decltype(&cusolverDnDsyevd_bufferSize) syevd_size = nullptr;
  decltype(&cusolverDnDsyevd) syevd = nullptr;
  decltype(&cusolverDnDpotrf_bufferSize) potrf_size = nullptr;
  decltype(&cusolverDnDpotrf) potrf = nullptr;
  decltype(&cublasDtrmm_v2) dtrmm = nullptr;
  decltype(&cublasDtrsm_v2) dtrsm = nullptr;
  decltype(&cublasDsymv_v2) dsymv = nullptr;
  cublasHandle_t hb[64] = {};
  cusolverDnHandle_t hs[64] = {};
};

std::mutex g_la_mu;
LinAlg g_la;

void* open_first(const char* const* names) {
  for (int i = 0; names[i]; ++i)
    if (void* h = dlopen(names[i], RTLD_NOW | RTLD_GLOBAL)) return h;
  return nullptr;
}

// returns the loaded table with this device's handles bound to st, or nullptr
LinAlg* linalg(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_la_mu);
  LinAlg& L = g_la;
  if (!L.tried) {
    L.tried = true;
    static const char* const kBlas[] = {"libcublas.so.12", "libcublas.so", "/usr/local/cuda/lib64/libcublas.so.12",
                                        nullptr};
    static const char* const kSolver[] = {"libcusolver.so.11", "libcusolver.so",
                                          "/usr/local/cuda/lib64/libcusolver.so.11", nullptr};
    void* hb = open_first(kBlas);
    void* hs = open_first(kSolver);
    if (hb && hs) {
      L.create = reinterpret_cast<decltype(L.create)>(dlsym(hb, "cublasCreate_v2"));
      L.set_stream = reinterpret_cast<decltype(L.set_stream)>(dlsym(hb, "cublasSetStream_v2"));
      L.dgemm = reinterpret_cast<decltype(L.dgemm)>(dlsym(hb, "cublasDgemm_v2"));
      L.dsyrk = reinterpret_cast<decltype(L.dsyrk)>(dlsym(hb, "cublasDsyrk_v2"));
      L.dsymm = reinterpret_cast<decltype(L.dsymm)>(dlsym(hb, "cublasDsymm_v2"));
      L.sv_create = reinterpret_cast<decltype(L.sv_create)>(dlsym(hs, "cusolverDnCreate"));
      L.sv_set_stream = reinterpret_cast<decltype(L.sv_set_stream)>(dlsym(hs, "cusolverDnSetStream"));
      L.syevd_size = reinterpret_cast<decltype(L.syevd_size)>(dlsym(hs, "cusolverDnDsyevd_bufferSize"));
      L.syevd = reinterpret_cast<decltype(L.syevd)>(dlsym(hs, "cusolverDnDsyevd"));
      L.potrf_size = reinterpret_cast<decltype(L.potrf_size)>(dlsym(hs, "cusolverDnDpotrf_bufferSize"));
      L.potrf = reinterpret_cast<decltype(L.potrf)>(dlsym(hs, "cusolverDnDpotrf"));
      L.dtrmm = reinterpret_cast<decltype(L.dtrmm)>(dlsym(hb, "cublasDtrmm_v2"));
      L.dtrsm = reinterpret_cast<decltype(L.dtrsm)>(dlsym(hb, "cublasDtrsm_v2"));
      L.dsymv = reinterpret_cast<decltype(L.dsymv)>(dlsym(hb, "cublasDsymv_v2"));
      L.ok = L.create && L.set_stream && L.dgemm && L.dsyrk && L.dsymm && L.sv_create && L.sv_set_stream &&
             L.syevd_size && L.syevd && L.potrf_size && L.potrf && L.dtrmm && L.dtrsm && L.dsymv;
    }
  }
  if (!L.ok) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!L.hb[dev] && L.create(&L.hb[dev]) != CUBLAS_STATUS_SUCCESS) return nullptr;
  if (!L.hs[dev] && L.sv_create(&L.hs[dev]) != CUSOLVER_STATUS_SUCCESS) return nullptr;
  if (L.set_stream(L.hb[dev], st) != CUBLAS_STATUS_SUCCESS) return nullptr;
  if (L.sv_set_stream(L.hs[dev], st) != CUSOLVER_STATUS_SUCCESS) return nullptr;
  return &L;
}

int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// dW column-major [d x n]: dW(i, j) = s_i w_ij - dw_j code_ji   (32 x 32 tiles, W transposed via smem)
template <typename WT>
__global__ void dw64_kernel(const WT* __restrict__ W, const float* __restrict__ s, const int8_t* __restrict__ qw,
                            const float* __restrict__ dw, int64_t d, int64_t n, double* __restrict__ out) {
  __shared__ float tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {                 // load W[i0 + r][j0 + tx]
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < d && j < n) ? (float)W[i * n + j] : 0.f;
  }
  __syncthreads();
  for (int c = threadIdx.y; c < 32; c += 8) {                 // write column j0 + c, rows i0 + tx
    const int64_t i = i0 + threadIdx.x, j = j0 + c;
    if (i < d && j < n)
      out[j * d + i] = (double)s[i] * (double)tile[threadIdx.x][c] - (double)dw[j] * (double)qw[j * d + i];
  }
}

// sq[k] = sqrt(Lambda'_k), isq[k] = 1/sq[k] (0 when Lambda' is 0: an all-zero A)
__global__ void whiten_kernel(const double* __restrict__ lam, int64_t d, double eps_rel, double* __restrict__ sq,
                              double* __restrict__ isq) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d) return;
  const double lmax = fmax(lam[d - 1], 0.0);
  const double l = fmax(lam[k], 0.0) + eps_rel * lmax;
  const double q = sqrt(l);
  sq[k] = q;
  isq[k] = q > 0.0 ? 1.0 / q : 0.0;
}

// power iteration on the (lower-stored) Gram matrix: w = G u computed by Dsymv; this single-CTA
// kernel sets lam = u . w (Rayleigh quotient, u unit) and u = w / |w| (fixed-order reductions)
__global__ void __launch_bounds__(1024) power_step_kernel(double* __restrict__ u, const double* __restrict__ w,
                                                          int64_t d, double* __restrict__ lam) {
  __shared__ double s1[1024], s2[1024];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += 1024) {
    a += u[i] * w[i];
    b += w[i] * w[i];
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  const double nrm = sqrt(s2[0]);
  if (threadIdx.x == 0) *lam = s1[0];
  const double sc = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int64_t i = threadIdx.x; i < d; i += 1024) u[i] = w[i] * sc;
}

__global__ void fill_kernel(double* __restrict__ u, int64_t d, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) u[i] = v;
}

// G'[i][i] = G[i][i] + eps_rel * max(lam, 0) (the relative regulariser of Q27), other entries copied
__global__ void regularize_kernel(const double* __restrict__ G, int64_t d, const double* __restrict__ lam,
                                  double eps_rel, double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d * d) return;
  const int64_t i = idx % d, j = idx / d;
  out[idx] = G[idx] + (i == j ? eps_rel * fmax(*lam, 0.0) : 0.0);
}

// column-major [rows x cols]: row k scaled by f[k]
__global__ void scale_rows_kernel(const double* in, int64_t rows, int64_t cols, const double* __restrict__ f,
                                  double* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  out[idx] = in[idx] * f[idx % rows];
}

// F += eps_rel * max(lam, 0) * dW  (the regulariser of Q27 applied to G dW)
__global__ void add_reg_kernel(double* __restrict__ F, const double* __restrict__ dW, int64_t count,
                               const double* __restrict__ lam, double eps_rel) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  F[idx] += eps_rel * fmax(*lam, 0.0) * dW[idx];
}

// small-side factors from V_r (n x r column-major, ascending eigen order) and sig2 (n):
// L1t (d x r, column-major, = dW V_r on entry) column k scaled by 1 / sigma_k; L2t (r x n,
// column-major) = Sigma_r V_r^T; sigma_k = sqrt(max(sig2[n - r + k], 0)) (0 -> zero factors)
__global__ void small_side_factors_kernel(double* __restrict__ L1t, double* __restrict__ L2t,
                                          const double* __restrict__ Vr, const double* __restrict__ sig2, int64_t d,
                                          int64_t n, int r) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = d * r, n2 = (int64_t)r * n;
  if (idx < n1) {
    const int k = (int)(idx / d);
    const double sg = sqrt(fmax(sig2[n - r + k], 0.0));
    L1t[idx] = sg > 0.0 ? L1t[idx] / sg : 0.0;
  } else if (idx < n1 + n2) {
    const int64_t e = idx - n1;
    const int64_t j = e / r;
    const int k = (int)(e - j * r);
    const double sg = sqrt(fmax(sig2[n - r + k], 0.0));
    L2t[e] = sg * Vr[(int64_t)k * n + j];
  }
}

template <typename OT>
__device__ __forceinline__ OT cvt_out(double v);
template <>
__device__ __forceinline__ float cvt_out<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(double v) { return __float2bfloat16_rn((float)v); }

// L1 out [d x r] row-major from L1t column-major [d x r] (column k = ascending eigen order, so
// output column c takes k = r - 1 - c: descending singular values); L2 out [r x n] row-major
// from L2t column-major [r x n] with the same row reversal.
template <typename OT>
__global__ void out_factors_kernel(const double* __restrict__ L1t, const double* __restrict__ L2t, int64_t d,
                                   int64_t n, int r, OT* __restrict__ L1, OT* __restrict__ L2) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = d * r, n2 = (int64_t)r * n;
  if (idx < n1) {
    const int64_t i = idx / r;
    const int c = (int)(idx - i * r);
    L1[idx] = cvt_out<OT>(L1t[(int64_t)(r - 1 - c) * d + i]);
  } else if (idx < n1 + n2) {
    const int64_t e = idx - n1;
    const int c = (int)(e / n);
    const int64_t j = e - (int64_t)c * n;
    L2[e] = cvt_out<OT>(L2t[j * r + (r - 1 - c)]);
  }
}

// sum_k a_k b_k, two stages, fixed order (deterministic)
__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t count,
                                   double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x; k < count; k += (int64_t)gridDim.x * 256)
    acc += a[k] * b[k];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void dot_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a = 0.0;
    for (int k = 0; k < nb; ++k) a += part[k];
    *out = a;
  }
}
constexpr int kDotBlocks = 592;

}  // namespace

bool cmc_linalg_available() { return linalg(0) != nullptr; }

bool cmc_eig_route() {
  static const int env = [] {                         // MASQ_CMC_EIG=1: the paper's eigen route (A/B)
    const char* ev = getenv("MASQ_CMC_EIG");
    return ev && atoi(ev) ? 1 : 0;
  }();
  return env == 1;
}

size_t cmc_syevd_lwork(int64_t d, int64_t n) {
  LinAlg* L = linalg(0);
  if (!L || d <= 0) return 0;
  // eigensolves: d x d (the eigen route's G and M M^T) or min(d, n) (Cholesky / small-side routes)
  const int64_t e = cmc_eig_route() ? d : std::min(d, n);
  int lw = 0, lp = 0;
  if (L->syevd_size(L->hs[cur_dev()], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)e, nullptr, (int)e,
                    nullptr, &lw) != CUSOLVER_STATUS_SUCCESS)
    return 0;
  if (L->potrf_size(L->hs[cur_dev()], CUBLAS_FILL_MODE_LOWER, (int)d, nullptr, (int)d, &lp) != CUSOLVER_STATUS_SUCCESS)
    return 0;
  return (size_t)(lw > lp ? lw : lp);
}

// phase 1: G[m-1] (+)= A_m^T A_m for m = 1..n_mod-1 (full symmetric, row-major) on the tensor
// cores (gram.cu): route the tokens into modality-grouped order, then the exact int8-slice Gram
cudaError_t launch_cmc_gram(const CmcArgs& a, double* G, int accumulate, cudaStream_t st) {
  const int64_t T = a.T, d = a.d;
  if (T == 0) {
    if (!accumulate) return cudaMemsetAsync(G, 0, sizeof(double) * (size_t)(a.n_mod - 1) * d * d, st);
    return cudaSuccess;
  }
  cudaError_t e = launch_route(a.ids, T, a.n_mod, a.perm, a.tile_mod, a.cnt, st);
  if (e != cudaSuccess) return e;
  return launch_cmc_gram_tc(a.X, a.xt, a.ld_x, a.ids, T, d, a.n_mod, a.inv, a.perm, a.tile_mod, a.R, a.cnt, a.ex,
                            a.slices, a.gram_part, a.status, G, accumulate, st);
}

// phase 2: factors (and the Theorem-2 residual <E, G E>) from the Gram matrices
cudaError_t launch_cmc_from_gram(const CmcArgs& a, const double* Gall, cudaStream_t st) {
  LinAlg* L = linalg(st);
  if (!L) return cudaErrorNotSupported;
  const int dev = cur_dev();
  cublasHandle_t hb = L->hb[dev];
  cusolverDnHandle_t hs = L->hs[dev];
  const int64_t d = a.d, n = a.n;
  const int r = a.r;
  const int di = (int)d, ni = (int)n;
  const double one = 1.0, zero = 0.0, mone = -1.0;
  const bool use_eig = cmc_eig_route();
#define CK_B(x) do { if ((x) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown; } while (0)
#define CK_S(x) do { if ((x) != CUSOLVER_STATUS_SUCCESS) return cudaErrorUnknown; } while (0)
  for (int m = 1; m < a.n_mod; ++m) {
    const double* Gm = Gall + (int64_t)(m - 1) * d * d;
    {
      // dW = S_m W - Q(S_t W)
      ProfScope ps_("cmc_dw", st);
      dim3 grid((unsigned)ceil_div(d, 32), (unsigned)ceil_div(n, 32)), block(32, 8);
      const float* sm = a.s + (int64_t)m * d;
      if (a.wt == MASQ_BF16)
        dw64_kernel<<<grid, block, 0, st>>>(static_cast<const __nv_bfloat16*>(a.W), sm, a.qw_t, a.dw_t, d, n, a.dW);
      else
        dw64_kernel<<<grid, block, 0, st>>>(static_cast<const float*>(a.W), sm, a.qw_t, a.dw_t, d, n, a.dW);
    }
    if (!use_eig && n < d) {
      // small side (n < d, e.g. the down projection 18944 -> 3584): with T^T T = G' = G +
      // eps lambda_max I, the right singular vectors of M = T dW are the eigenvectors of
      // M^T M = dW^T G' dW (n x n), and the best rank-r L1 L2 is T^-1 M V_r V_r^T = dW V_r V_r^T:
      // L2 = Sigma_r V_r^T, L1 = dW V_r Sigma_r^-1 (no d x d factorisation or eigensolve)
      ProfScope ps_("cmc_small_side", st);
      double* u = a.sq;
      double* w = a.isq;
      fill_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, st>>>(u, d, 1.0 / sqrt((double)d));
      for (int it = 0; it < 32; ++it) {
        CK_B(L->dsymv(hb, CUBLAS_FILL_MODE_LOWER, di, &one, Gm, di, u, 1, &zero, w, 1));
        power_step_kernel<<<1, 1024, 0, st>>>(u, w, d, a.lam);
      }
      CK_B(L->dsymm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, di, ni, &one, Gm, di, a.dW, di, &zero, a.Mb, di));
      add_reg_kernel<<<(unsigned)ceil_div(d * n, 256), 256, 0, st>>>(a.Mb, a.dW, d * n, a.lam, a.eps_rel);
      CK_B(L->dgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, ni, ni, di, &one, a.dW, di, a.Mb, di, &zero, a.C, ni));
      {
        ProfScope ps2_("cmc_eig_small", st);
        CK_S(L->syevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, ni, a.C, ni, a.sig2, a.work,
                      (int)a.lwork, a.info + 1));
      }
      const double* Vr = a.C + (int64_t)(n - r) * n;              // columns n-r .. n-1 (ascending)
      CK_B(L->dgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, di, r, ni, &one, a.dW, di, Vr, ni, &zero, a.L1t, di));
      const int64_t cnt = d * r + (int64_t)r * n;
      small_side_factors_kernel<<<(unsigned)ceil_div(cnt, 256), 256, 0, st>>>(a.L1t, a.L2t, Vr, a.sig2, d, n, r);
    } else if (use_eig) {
      // the paper's route: eig G = P Lambda P^T, T = diag(sqrt Lambda') P^T
      cudaError_t e = cudaMemcpyAsync(a.G, Gm, sizeof(double) * d * d, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return e;
      {
        ProfScope ps_("cmc_eig_gram", st);
        CK_S(L->syevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, di, a.G, di, a.lam, a.work, (int)a.lwork,
                      a.info));
      }
      whiten_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, st>>>(a.lam, d, a.eps_rel, a.sq, a.isq);
      ProfScope ps_("cmc_whiten_gemm", st);
      CK_B(L->dgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, di, ni, di, &one, a.G, di, a.dW, di, &zero, a.Mb, di));
      scale_rows_kernel<<<(unsigned)ceil_div(d * n, 256), 256, 0, st>>>(a.Mb, d, n, a.sq, a.Mb);
    } else {
      // any T with T^T T = G + eps*lambda_max*I gives the same optimum L1 L2 (T' = Q T for an
      // orthogonal Q): take the Cholesky factor, G' = Lc Lc^T, T = Lc^T.  lambda_max by 32
      // power-iteration steps (the regulariser only needs it to O(1e-6))
      ProfScope ps_("cmc_chol", st);
      double* u = a.sq;                                            // scratch vectors (d)
      double* w = a.isq;
      fill_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, st>>>(u, d, 1.0 / sqrt((double)d));
      for (int it = 0; it < 32; ++it) {
        CK_B(L->dsymv(hb, CUBLAS_FILL_MODE_LOWER, di, &one, Gm, di, u, 1, &zero, w, 1));
        power_step_kernel<<<1, 1024, 0, st>>>(u, w, d, a.lam);
      }
      regularize_kernel<<<(unsigned)ceil_div(d * d, 256), 256, 0, st>>>(Gm, d, a.lam, a.eps_rel, a.G);
      CK_S(L->potrf(hs, CUBLAS_FILL_MODE_LOWER, di, a.G, di, a.work, (int)a.lwork, a.info));
      // M = Lc^T dW
      CK_B(L->dtrmm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, di, ni, &one, a.G,
                    di, a.dW, di, a.Mb, di));
    }
    if (use_eig || n >= d) {
    // top-r left singular vectors of M from eig(M M^T)
    {
      ProfScope ps_("cmc_mmt", st);
      CK_B(L->dsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, di, ni, &one, a.Mb, di, &zero, a.C, di));
    }
    {
      ProfScope ps_("cmc_eig_mmt", st);
      CK_S(L->syevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, di, a.C, di, a.sig2, a.work, (int)a.lwork,
                    a.info + 1));
    }
    const double* Ur = a.C + (int64_t)(d - r) * d;            // columns d-r .. d-1 (ascending)
    {
      ProfScope ps_("cmc_factors_gemm", st);
      CK_B(L->dgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, r, ni, di, &one, Ur, di, a.Mb, di, &zero, a.L2t, r));
      if (use_eig) {
        scale_rows_kernel<<<(unsigned)ceil_div(d * r, 256), 256, 0, st>>>(Ur, d, r, a.isq, a.Urs);
        CK_B(L->dgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, di, r, di, &one, a.G, di, a.Urs, di, &zero, a.L1t, di));
      } else {
        // L1 = Lc^-T U_r
        cudaError_t e = cudaMemcpyAsync(a.L1t, Ur, sizeof(double) * d * r, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        CK_B(L->dtrsm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, di, r, &one,
                      a.G, di, a.L1t, di));
      }
    }
    }
    {
      const int64_t cnt = d * r + (int64_t)r * n;
      const unsigned g = (unsigned)ceil_div(cnt, 256);
      if (a.lt == MASQ_BF16)
        out_factors_kernel<<<g, 256, 0, st>>>(a.L1t, a.L2t, d, n, r,
                                              static_cast<__nv_bfloat16*>(a.L1) + (int64_t)(m - 1) * d * r,
                                              static_cast<__nv_bfloat16*>(a.L2) + (int64_t)(m - 1) * r * n);
      else
        out_factors_kernel<<<g, 256, 0, st>>>(a.L1t, a.L2t, d, n, r, static_cast<float*>(a.L1) + (int64_t)(m - 1) * d * r,
                                              static_cast<float*>(a.L2) + (int64_t)(m - 1) * r * n);
    }
    if (a.resid) {
      // E = dW - L1t L2t (in place), F = G E with the (caller's) Gram, <E, F>
      ProfScope ps_("cmc_resid", st);
      CK_B(L->dgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, di, ni, r, &mone, a.L1t, di, a.L2t, r, &one, a.dW, di));
      CK_B(L->dsymm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, di, ni, &one, Gm, di, a.dW, di, &zero, a.Mb, di));
      dot_partial_kernel<<<kDotBlocks, 256, 0, st>>>(a.dW, a.Mb, d * n, a.dot);
      dot_final_kernel<<<1, 32, 0, st>>>(a.dot, kDotBlocks, a.resid + (m - 1));
    }
  }
#undef CK_B
#undef CK_S
  return cudaGetLastError();
}

int cmc_dot_blocks() { return kDotBlocks; }

}  // namespace masq
