// ftc_backward.cu -- checksum-protected back-propagation.
//
// conv_backward (conv.hpp:150-185) and run_protected_backward (workflow.hpp:340-417)
// on the device.  Gradients are accumulated in FP64 from the FP32 operands; the
// protection runs on those FP64 gradients exactly as the reference does at T=double:
//   rows[n] = sum_m dO[n,m], cols[m] = sum_n dO[n,m]            (workflow.hpp:358-367)
//   cdw = conv_backward(D, 0, rows).dW, cdd = conv_backward(0, W, cols).dD  (:369-374)
//   check: sum_m dW[m] vs cdw and sum_n dD[n] vs cdd, values_differ(tau)    (:376-401)
//   mismatch -> one recompute; a second mismatch -> IntegrityError        (:403-416)
// and the FP32 outputs are the checked FP64 gradients rounded once.  The reference's
// std::function post_hook is a POD substitution list (ftc_grad_fault) applied to the
// first pass only, as the hook is.
#include <cuda_runtime.h>

#include <cstring>

#include "ftc_common.cuh"

#ifndef CK
#define CK(x)                      \
  do {                             \
    int _st = (x);                 \
    if (_st != FTC_OK) return _st; \
  } while (0)
#endif

namespace ftc {
namespace {

constexpr int kT = 256;

inline int nblocks(long long n) {
  long long b = (n + kT - 1) / kT;
  return (int)(b < 1 ? 1 : b);
}

// rows[n][f] = sum_m dO[n][m][f], cols[m][f] = sum_n dO[n][m][f]  (FP64)
__global__ void k_grad_block_sums(const float* __restrict__ dO, int N, int M, int E2, double* __restrict__ rows,
                                  double* __restrict__ cols) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < (long long)N * E2) {
    const int n = (int)(q / E2), f = (int)(q % E2);
    double s = 0.0;
    for (int m = 0; m < M; ++m) s += (double)dO[((long long)n * M + m) * E2 + f];
    rows[q] = s;
  }
  if (q < (long long)M * E2) {
    const int m = (int)(q / E2), f = (int)(q % E2);
    double s = 0.0;
    for (int n = 0; n < N; ++n) s += (double)dO[((long long)n * M + m) * E2 + f];
    cols[q] = s;
  }
}

// dW[m][k][i][j] = sum_{n,x,y} D[n][k][Ux+i-p][Uy+j-p] * G[n][m][x][y]  (FP64)
// Block = one (m, k); per filter row i the 256 threads sweep the (n, x, y) space (warps
// over output rows, lanes over columns) keeping R column accumulators, then reduce.
template <typename TG>
__global__ void __launch_bounds__(kT) k_bwd_dw(const float* __restrict__ D, const TG* __restrict__ G, int N, int C,
                                               int H, int Mg, int R, int U, int pad, int E,
                                               double* __restrict__ dW) {
  extern __shared__ double red[];  // [R][kT]
  const int m = blockIdx.x / C, k = blockIdx.x % C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long HH = (long long)H * H, E2 = (long long)E * E;
  for (int i = 0; i < R; ++i) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    for (int row = warp; row < N * E; row += kT / 32) {
      const int n = row / E, x = row - (row / E) * E;
      const int h = U * x + i - pad;
      if (h < 0 || h >= H) continue;
      const float* drow = D + ((long long)n * C + k) * HH + (long long)h * H;
      const TG* grow = G + ((long long)n * Mg + m) * E2 + (long long)x * E;
      for (int y = lane; y < E; y += 32) {
        const double g = (double)grow[y];
        const int w0 = U * y - pad;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j >= R) break;
          const int w = w0 + j;
          if (w >= 0 && w < H) acc[j] += (double)drow[w] * g;
        }
      }
    }
    for (int j = 0; j < R; ++j) red[j * kT + tid] = acc[j];
    __syncthreads();
    for (int j = warp; j < R; j += kT / 32) {
      double s = 0.0;
      for (int t = lane; t < kT; t += 32) s += red[j * kT + t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) dW[(((long long)m * C + k) * R + i) * R + j] = s;
    }
    __syncthreads();
  }
}

// dD[n][k][h][w] = sum_{m,i,j} W[m][k][i][j] * G[n][m][x][y] over the (x, y) with
// Ux+i-p = h, Uy+j-p = w  (FP64); one thread per (n, k, h, w)
template <typename TG>
__global__ void __launch_bounds__(kT) k_bwd_dd(const float* __restrict__ W, const TG* __restrict__ G, int Nn, int C,
                                               int H, int M, int R, int U, int pad, int E,
                                               double* __restrict__ dD) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long HH = (long long)H * H;
  if (q >= (long long)Nn * C * HH) return;
  const int w = (int)(q % H), h = (int)((q / H) % H);
  const int k = (int)((q / HH) % C), n = (int)(q / (HH * C));
  const long long E2 = (long long)E * E;
  double acc = 0.0;
  for (int i = 0; i < R; ++i) {
    const int xs = h + pad - i;
    if (xs < 0 || xs % U) continue;
    const int x = xs / U;
    if (x >= E) continue;
    for (int j = 0; j < R; ++j) {
      const int ys = w + pad - j;
      if (ys < 0 || ys % U) continue;
      const int y = ys / U;
      if (y >= E) continue;
      const TG* g = G + (long long)n * M * E2 + (long long)x * E + y;
      const float* wk = W + ((long long)k * R + i) * R + j;
      for (int m = 0; m < M; ++m) acc += (double)wk[(long long)m * C * R * R] * (double)g[(long long)m * E2];
    }
  }
  dD[q] = acc;
}

// families: sum over the leading index (count slabs) vs the checksum, values_differ
__global__ void k_grad_check(const double* __restrict__ g, int count, long long per, const double* __restrict__ ref,
                             double tau, int* bad) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per) return;
  double s = 0.0;
  for (int a = 0; a < count; ++a) s += g[(long long)a * per + e];
  if (values_differ(ref[e], s, tau)) atomicOr(bad, 1);
}

__global__ void k_grad_faults(const ftc_grad_fault* __restrict__ f, int nf, double* dW, long long nW, double* dD,
                              long long nD) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int t = 0; t < nf; ++t) {  // in list order, like a hook body
    double* base = f[t].target == 0 ? dW : dD;
    const long long n = f[t].target == 0 ? nW : nD;
    if (f[t].index < 0 || f[t].index >= n) continue;
    double& v = base[f[t].index];
    v = f[t].mode == 0 ? f[t].value : v + f[t].value;
  }
}

__global__ void k_round(const double* __restrict__ a, float* __restrict__ o, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    o[e] = (float)a[e];
}

struct Bwd {
  int N, C, H, M, R, U, pad, E;
  long long nW, nD, E2;
};

int validate_bwd(const ftc_conv_desc* d, Bwd* b) {
  if (!d) {
    set_error(FTC_INVALID_ARGUMENT, "null descriptor");
    return FTC_INVALID_ARGUMENT;
  }
  if (d->groups != 1) {
    set_error(FTC_CONFIG_ERROR, "grouped back-propagation is unsupported");  // conv.hpp:154
    return FTC_CONFIG_ERROR;
  }
  if (d->bias_enabled) {
    set_error(FTC_CONFIG_ERROR, "back-propagation takes no bias");
    return FTC_CONFIG_ERROR;
  }
  int E = 0;
  const int st = ftc_output_extent(d->H, d->R, d->pad, d->stride, &E);
  if (st != FTC_OK) return st;
  if (d->N <= 0 || d->C <= 0 || d->M <= 0 || d->R > 4096) {
    set_error(FTC_SHAPE_ERROR, "tensor dimensions must be positive");
    return FTC_SHAPE_ERROR;
  }
  *b = Bwd{d->N, d->C, d->H, d->M, d->R, d->stride, d->pad, E, (long long)d->M * d->C * d->R * d->R,
           (long long)d->N * d->C * d->H * d->H, (long long)E * E};
  return FTC_OK;
}

template <typename TG>
int launch_grads(const Bwd& b, const float* D, const float* W, const TG* G, int Nn, int Mg, double* dW, double* dD,
                 cudaStream_t s) {
  if (dW) {
    const size_t smem = (size_t)b.R * kT * sizeof(double);
    if (b.R > 16) {
      set_error(FTC_CONFIG_ERROR, "back-propagation supports kernels up to 16 x 16");
      return FTC_CONFIG_ERROR;
    }
    FTC_LAUNCH(k_bwd_dw<TG><<<Mg * b.C, kT, smem, s>>>(D, G, Nn, b.C, b.H, Mg, b.R, b.U, b.pad, b.E, dW));
  }
  if (dD) {
    const long long n = (long long)Nn * b.C * b.H * b.H;
    FTC_LAUNCH(k_bwd_dd<TG><<<nblocks(n), kT, 0, s>>>(W, G, Nn, b.C, b.H, Mg, b.R, b.U, b.pad, b.E, dD));
  }
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

// Stream-ordered scratch owned by one call: every buffer allocated through it is freed
// on every return path (early FTC_CUDA_CHECK returns included).
struct Scratch {
  cudaStream_t s;
  void* p[16] = {};
  int n = 0;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (int i = 0; i < n; ++i)
      if (p[i]) cudaFreeAsync(p[i], s);
  }
  template <class T>
  int alloc(T** out, size_t bytes) {
    *out = nullptr;
    if (n == 16) {
      set_error(FTC_CUDA_ERROR, "backward scratch: too many buffers");
      return FTC_CUDA_ERROR;
    }
    FTC_CUDA_CHECK(cudaMallocAsync((void**)out, bytes, s));
    p[n++] = (void*)*out;
    return FTC_OK;
  }
};

int round_out(const double* a, float* o, long long n, cudaStream_t s) {
  FTC_LAUNCH(k_round<<<nblocks(n) < 1184 ? nblocks(n) : 1184, kT, 0, s>>>(a, o, n));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace
}  // namespace ftc

using namespace ftc;

extern "C" {

int ftc_conv_backward(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, float* dW,
                      float* dD, void* stream) {
  Bwd b;
  int st = validate_bwd(desc, &b);
  if (st != FTC_OK) return st;
  if (!D || !W || !dO || !dW || !dD) {
    set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(s);
  double *w64 = nullptr, *d64 = nullptr;
  CK(sc.alloc(&w64, b.nW * sizeof(double)));
  CK(sc.alloc(&d64, b.nD * sizeof(double)));
  CK(launch_grads<float>(b, D, W, dO, b.N, b.M, w64, d64, s));
  CK(round_out(w64, dW, b.nW, s));
  return round_out(d64, dD, b.nD, s);
}

int ftc_protected_backward(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, double tau,
                           const ftc_grad_fault* hook, int32_t n_hook, float* dW, float* dD,
                           ftc_backward_report* rep, void* stream) {
  Bwd b;
  int st = validate_bwd(desc, &b);
  if (st != FTC_OK) return st;
  if (!D || !W || !dO || !dW || !dD || !rep || (n_hook > 0 && !hook) || n_hook < 0) {
    set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  std::memset(rep, 0, sizeof *rep);
  cudaStream_t s = (cudaStream_t)stream;
  const long long per_w = (long long)b.C * b.R * b.R, per_d = (long long)b.C * b.H * b.H;
  // scratch: FP64 gradients, block sums, checksum gradients, flags, fault list
  Scratch sc(s);
  double *w64, *d64, *rows, *cols, *cdw, *cdd;
  int* flags;
  ftc_grad_fault* fl = nullptr;
  CK(sc.alloc(&w64, b.nW * sizeof(double)));
  CK(sc.alloc(&d64, b.nD * sizeof(double)));
  CK(sc.alloc(&rows, (size_t)b.N * b.E2 * sizeof(double)));
  CK(sc.alloc(&cols, (size_t)b.M * b.E2 * sizeof(double)));
  CK(sc.alloc(&cdw, per_w * sizeof(double)));
  CK(sc.alloc(&cdd, per_d * sizeof(double)));
  CK(sc.alloc(&flags, 2 * sizeof(int)));
  if (n_hook > 0) {
    CK(sc.alloc(&fl, n_hook * sizeof(ftc_grad_fault)));
    FTC_CUDA_CHECK(cudaMemcpyAsync(fl, hook, n_hook * sizeof(ftc_grad_fault), cudaMemcpyHostToDevice, s));
  }
  auto check = [&](int* bad_w, int* bad_d) -> int {
    FTC_CUDA_CHECK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    FTC_LAUNCH(k_grad_check<<<nblocks(per_w), kT, 0, s>>>(w64, b.M, per_w, cdw, tau, flags));
    FTC_LAUNCH(k_grad_check<<<nblocks(per_d), kT, 0, s>>>(d64, b.N, per_d, cdd, tau, flags + 1));
    int h[2] = {0, 0};
    FTC_CUDA_CHECK(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, s));
    FTC_CUDA_CHECK(cudaStreamSynchronize(s));
    *bad_w = h[0];
    *bad_d = h[1];
    return FTC_OK;
  };
  do {
    const long long nb = (b.N > b.M ? b.N : b.M) * b.E2;
    FTC_LAUNCH(k_grad_block_sums<<<nblocks(nb), kT, 0, s>>>(dO, b.N, b.M, (int)b.E2, rows, cols));
    // checksum gradients: a one-kernel dW against the row sums, a one-image dD against
    // the column sums
    if ((st = launch_grads<double>(b, D, W, rows, b.N, 1, cdw, nullptr, s))) break;
    if ((st = launch_grads<double>(b, D, W, cols, 1, b.M, nullptr, cdd, s))) break;
    if ((st = launch_grads<float>(b, D, W, dO, b.N, b.M, w64, d64, s))) break;
    if (n_hook > 0) FTC_LAUNCH(k_grad_faults<<<1, 32, 0, s>>>(fl, n_hook, w64, b.nW, d64, b.nD));
    int bw = 0, bd = 0;
    if ((st = check(&bw, &bd))) break;
    rep->dw_detected = bw;
    rep->dd_detected = bd;
    if (bw || bd) {
      if ((st = launch_grads<float>(b, D, W, dO, b.N, b.M, w64, d64, s))) break;
      rep->recomputed = 1;
      if ((st = check(&bw, &bd))) break;
      if (bw || bd) {
        set_error(FTC_INTEGRITY_ERROR, "gradient recomputation failed verification");
        st = FTC_INTEGRITY_ERROR;
        break;
      }
    }
    if ((st = round_out(w64, dW, b.nW, s))) break;
    st = round_out(d64, dD, b.nD, s);
  } while (false);
  return st;
}

// host-buffer forms (the reference's calling convention): copies in, device pass, copies out
static int bwd_host(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, float* dW, float* dD,
                    bool prot, double tau, const ftc_grad_fault* hook, int32_t n_hook, ftc_backward_report* rep,
                    void* stream) {
  Bwd b;
  int st = validate_bwd(desc, &b);
  if (st != FTC_OK) return st;
  if (!D || !W || !dO || !dW || !dD) {
    set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nW = b.nW * sizeof(float), nD = b.nD * sizeof(float), nO = (size_t)b.N * b.M * b.E2 * sizeof(float);
  float *d_D = nullptr, *d_W = nullptr, *d_O = nullptr, *d_dW = nullptr, *d_dD = nullptr;
  {
  Scratch sc(s);
  CK(sc.alloc(&d_D, nD));
  CK(sc.alloc(&d_W, nW));
  CK(sc.alloc(&d_O, nO));
  CK(sc.alloc(&d_dW, nW));
  CK(sc.alloc(&d_dD, nD));
  FTC_CUDA_CHECK(cudaMemcpyAsync(d_D, D, nD, cudaMemcpyHostToDevice, s));
  FTC_CUDA_CHECK(cudaMemcpyAsync(d_W, W, nW, cudaMemcpyHostToDevice, s));
  FTC_CUDA_CHECK(cudaMemcpyAsync(d_O, dO, nO, cudaMemcpyHostToDevice, s));
  st = prot ? ftc_protected_backward(desc, d_D, d_W, d_O, tau, hook, n_hook, d_dW, d_dD, rep, stream)
            : ftc_conv_backward(desc, d_D, d_W, d_O, d_dW, d_dD, stream);
  if (st == FTC_OK) {
    cudaMemcpyAsync(dW, d_dW, nW, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(dD, d_dD, nD, cudaMemcpyDeviceToHost, s);
  }
  }  // scratch freed (stream-ordered) before the synchronisation
  FTC_CUDA_CHECK(cudaStreamSynchronize(s));
  return st;
}

int ftc_conv_backward_host(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, float* dW,
                           float* dD, void* stream) {
  return bwd_host(desc, D, W, dO, dW, dD, false, 0.0, nullptr, 0, nullptr, stream);
}

int ftc_protected_backward_host(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO,
                                double tau, const ftc_grad_fault* hook, int32_t n_hook, float* dW, float* dD,
                                ftc_backward_report* report, void* stream) {
  if (!report) {
    set_error(FTC_INVALID_ARGUMENT, "null report");
    return FTC_INVALID_ARGUMENT;
  }
  return bwd_host(desc, D, W, dO, dW, dD, true, tau, hook, n_hook, report, stream);
}

}  // extern "C"
