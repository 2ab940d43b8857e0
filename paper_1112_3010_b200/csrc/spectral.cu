// Engine-level spectral API: the reference's stand-alone transforms and the
// FftConvolver building blocks (R/convolution.py:164-313: fft_forward,
// fft_inverse, _check_sizes, kernel_hat / impulse_hat, forward_pair,
// inverse_to_grid, inverse_pair_to_grid, product) on the GPU.
//
// The fused distance pipeline never goes through these entry points (its own
// padded power-of-two passes live in kernels.cuh); they exist so that callers
// of the reference's engine API -- which hands spectra of arbitrary padded
// shapes (next_fast_len sizes, 2*3*5*7*11-smooth) back and forth as arrays --
// get the same arrays from the device.
//
// Transform engine: one axis at a time, Stockham autosort radix stages
// (radices 4, 2, 3, 5, 7, 11, ... up to 31, each an in-register DFT with
// table twiddles), a CTA per tile of lines.  Lines up to 4096 points run in
// shared memory (ping-pong); longer lines in a global-memory ping-pong.  Axis
// lengths with a prime factor above 31 go through Bluestein's chirp-z with a
// power-of-two inner transform.  Twiddles come from correctly rounded long
// double tables (cached per length).  Inverse transforms scale by 1/n per axis
// (scipy's ifftn normalisation, 1/P overall).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/eikfld_b200.h"

int eik_fail(int code, const std::string& msg);

namespace {

#define CKS(x)                                                                                    \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) return eik_fail(EIK_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int MAX_RADIX = 31;
constexpr int MAX_STAGES = 40;
constexpr int SMEM_LINE = 4096;  // complex points per CTA tile held in shared memory (x2 ping-pong = 128 KB)
constexpr int NT = 256;

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t b) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, b ? b : 16);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

struct AxisArgs {
  double2* data;      // [outer][n][inner]
  double2* scratch;   // global ping-pong (long lines): 2 * n per line of the launch
  int64_t n, inner, outer, nlines;
  int tl;             // lines per CTA tile (consecutive inner indices)
  int nst;
  int radix[MAX_STAGES];
  const double2* tw;  // W_n^k = exp(-2 pi i k / n), k in [0, n)
  int inverse;
  double scale;       // applied on store
  int smem;           // 1: tile in shared memory
};

// One radix-R Stockham step (Bainville's formulation): Ns = product of the
// previous radices; j runs over n / R butterflies of every line of the tile.
__device__ void stockham_stage(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n, int tl, int R,
                               int64_t Ns, const double2* __restrict__ tw, int inverse) {
  const int64_t nb = n / R, stride_t = n / R;  // input stride between the R legs
  const int64_t twstep = n / (Ns * R);         // W_{Ns R}^x = W_n^{x * twstep}
  double2 v[MAX_RADIX];
  for (int64_t w = threadIdx.x; w < (int64_t)tl * nb; w += blockDim.x) {
    const int t = (int)(w / nb);
    const int64_t j = w % nb;
    const double2* s = src + (int64_t)t * n;
    double2* d = dst + (int64_t)t * n;
    const int64_t k = j % Ns;
    for (int r = 0; r < R; ++r) {
      double2 x = s[j + r * stride_t];
      if (r && k) {
        double2 wv = __ldg(tw + ((int64_t)r * k * twstep) % n);
        if (inverse) wv.y = -wv.y;
        x = cmulc(x, wv);
      }
      v[r] = x;
    }
    // R-point DFT (R = 2 / 4 by hand; others direct with table roots)
    double2 o[MAX_RADIX];
    if (R == 2) {
      o[0] = make_double2(v[0].x + v[1].x, v[0].y + v[1].y);
      o[1] = make_double2(v[0].x - v[1].x, v[0].y - v[1].y);
    } else if (R == 4) {
      const double2 a = make_double2(v[0].x + v[2].x, v[0].y + v[2].y);
      const double2 b = make_double2(v[0].x - v[2].x, v[0].y - v[2].y);
      const double2 c = make_double2(v[1].x + v[3].x, v[1].y + v[3].y);
      double2 e = make_double2(v[1].x - v[3].x, v[1].y - v[3].y);
      // forward: multiply e by -i; inverse: by +i
      e = inverse ? make_double2(-e.y, e.x) : make_double2(e.y, -e.x);
      o[0] = make_double2(a.x + c.x, a.y + c.y);
      o[1] = make_double2(b.x + e.x, b.y + e.y);
      o[2] = make_double2(a.x - c.x, a.y - c.y);
      o[3] = make_double2(b.x - e.x, b.y - e.y);
    } else {
      const int64_t rstep = n / R;  // W_R^m = W_n^{m n / R}
      for (int q = 0; q < R; ++q) {
        double2 acc = v[0];
        for (int r = 1; r < R; ++r) {
          double2 wv = __ldg(tw + ((int64_t)((q * r) % R)) * rstep);
          if (inverse) wv.y = -wv.y;
          const double2 p = cmulc(v[r], wv);
          acc.x += p.x;
          acc.y += p.y;
        }
        o[q] = acc;
      }
    }
    const int64_t base = (j / Ns) * Ns * R + k;
    for (int r = 0; r < R; ++r) d[base + r * Ns] = o[r];
  }
}

__global__ void __launch_bounds__(NT) axis_fft_kernel(const AxisArgs a) {
  extern __shared__ double2 sm[];
  const int64_t tiles_per_outer = (a.inner + a.tl - 1) / a.tl;
  const int64_t tile = blockIdx.x;
  const int64_t o = tile / tiles_per_outer;
  const int64_t i0 = (tile % tiles_per_outer) * a.tl;
  const int tl = (int)(a.inner - i0 < a.tl ? a.inner - i0 : a.tl);
  const int64_t n = a.n;
  double2 *b0, *b1;
  if (a.smem) {
    b0 = sm;
    b1 = sm + (int64_t)a.tl * n;
  } else {
    b0 = a.scratch + (int64_t)tile * 2 * n;
    b1 = b0 + n;
  }
  const double2* src = a.data + (o * n) * a.inner + i0;
  for (int64_t e = threadIdx.x; e < (int64_t)tl * n; e += blockDim.x) {
    const int64_t j = e / tl, t = e % tl;
    b0[t * n + j] = src[j * a.inner + t];
  }
  __syncthreads();
  int64_t Ns = 1;
  for (int s = 0; s < a.nst; ++s) {
    stockham_stage(b0, b1, n, tl, a.radix[s], Ns, a.tw, a.inverse);
    Ns *= a.radix[s];
    __syncthreads();
    double2* t = b0;
    b0 = b1;
    b1 = t;
  }
  double2* dst = a.data + (o * n) * a.inner + i0;
  for (int64_t e = threadIdx.x; e < (int64_t)tl * n; e += blockDim.x) {
    const int64_t j = e / tl, t = e % tl;
    double2 x = b0[t * n + j];
    dst[j * a.inner + t] = make_double2(x.x * a.scale, x.y * a.scale);
  }
}

// ---- Bluestein: X_k = w_k sum_j (x_j w_j) conj(w_{k-j}),  w_j = exp(-i pi j^2 / n)
__global__ void chirp_load_kernel(const double2* __restrict__ data, int64_t n, int64_t inner, int64_t nlines, int64_t M,
                                  const double2* __restrict__ w2n, int inverse, double2* __restrict__ tmp) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nlines * M) return;
  const int64_t line = e / M, j = e % M;
  if (j >= n) {
    tmp[e] = make_double2(0.0, 0.0);
    return;
  }
  const int64_t o = line / inner, i = line % inner;
  double2 w = w2n[(j * j) % (2 * n)];
  if (inverse) w.y = -w.y;
  tmp[e] = cmulc(data[(o * n + j) * inner + i], w);
}

__global__ void chirp_mul_kernel(double2* __restrict__ tmp, int64_t nlines, int64_t M, const double2* __restrict__ bhat) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nlines * M) return;
  tmp[e] = cmulc(tmp[e], bhat[e % M]);
}

__global__ void chirp_store_kernel(double2* __restrict__ data, int64_t n, int64_t inner, int64_t nlines, int64_t M,
                                   const double2* __restrict__ w2n, int inverse, double scale,
                                   const double2* __restrict__ tmp) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nlines * n) return;
  const int64_t line = e / n, k = e % n;
  const int64_t o = line / inner, i = line % inner;
  double2 w = w2n[(k * k) % (2 * n)];
  if (inverse) w.y = -w.y;
  const double2 x = cmulc(tmp[line * M + k], w);
  data[(o * n + k) * inner + i] = make_double2(x.x * scale, x.y * scale);
}

__global__ void chirp_filter_kernel(int64_t n, int64_t M, const double2* __restrict__ w2n, int inverse,
                                    double2* __restrict__ b) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= M) return;
  int64_t m = -1;
  if (j < n) m = j;
  else if (j > M - n) m = M - j;
  if (m < 0) {
    b[j] = make_double2(0.0, 0.0);
    return;
  }
  double2 w = w2n[(m * m) % (2 * n)];
  if (!inverse) w.y = -w.y;  // conj of the forward chirp
  b[j] = w;
}

// ---- pack / unpack / window / product
__global__ void pad_pair_kernel(int nd, const int64_t* __restrict__ pdims, const double* __restrict__ a,
                                const int64_t* __restrict__ ad, const double* __restrict__ b,
                                const int64_t* __restrict__ bd, int64_t P, double2* __restrict__ z) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= P) return;
  int64_t rem = e, ia = 0, ib = 0;
  bool ina = a != nullptr, inb = b != nullptr;
  int64_t sa = 1, sb = 1;
  for (int d = nd - 1; d >= 0; --d) {
    const int64_t x = rem % pdims[d];
    rem /= pdims[d];
    if (ina) {
      if (x >= ad[d]) ina = false;
      else ia += x * sa, sa *= ad[d];
    }
    if (inb) {
      if (x >= bd[d]) inb = false;
      else ib += x * sb, sb *= bd[d];
    }
  }
  z[e] = make_double2(ina ? a[ia] : 0.0, inb ? b[ib] : 0.0);
}

// a_hat = (z + conj z(-k)) / 2,  b_hat = -i/2 (z - conj z(-k))   (R/convolution.py:264-276)
__global__ void unpack_pair_kernel(int nd, const int64_t* __restrict__ pdims, int64_t P, const double2* __restrict__ z,
                                   double2* __restrict__ ah, double2* __restrict__ bh) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= P) return;
  int64_t rem = e, r = 0, s = 1;
  for (int d = nd - 1; d >= 0; --d) {
    const int64_t x = rem % pdims[d];
    rem /= pdims[d];
    r += ((pdims[d] - x) % pdims[d]) * s;
    s *= pdims[d];
  }
  const double2 u = z[e], v = z[r];
  const double2 zr = make_double2(v.x, -v.y);  // conj z(-k)
  ah[e] = make_double2(0.5 * (u.x + zr.x), 0.5 * (u.y + zr.y));
  // -0.5i (u - zr) = (0.5 (u - zr).y, -0.5 (u - zr).x)
  bh[e] = make_double2(0.5 * (u.y - zr.y), -0.5 * (u.x - zr.x));
}

__global__ void combine_kernel(int64_t P, const double2* __restrict__ a, const double2* __restrict__ b,
                               double2* __restrict__ z) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= P) return;
  const double2 x = a[e];
  if (!b) {
    z[e] = x;
    return;
  }
  const double2 y = b[e];
  z[e] = make_double2(x.x - y.y, x.y + y.x);  // a + i b
}

__global__ void window_kernel(int nd, const int64_t* __restrict__ pdims, const int64_t* __restrict__ w0,
                              const int64_t* __restrict__ wn, int64_t Nw, const double2* __restrict__ z,
                              double* __restrict__ re, double* __restrict__ im) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= Nw) return;
  int64_t rem = e, src = 0, s = 1;
  for (int d = nd - 1; d >= 0; --d) {
    const int64_t x = rem % wn[d];
    rem /= wn[d];
    src += (w0[d] + x) * s;
    s *= pdims[d];
  }
  const double2 v = z[src];
  if (re) re[e] = v.x;
  if (im) im[e] = v.y;
}

__global__ void cmul_kernel(int64_t P, const double2* __restrict__ a, const double2* __restrict__ b,
                            double2* __restrict__ o) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= P) return;
  const double2 x = a[e], y = b[e];
  // numpy's complex multiply: (ac - bd) + (ad + bc) i, unfused
  o[e] = make_double2(__dsub_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)),
                      __dadd_rn(__dmul_rn(x.x, y.y), __dmul_rn(x.y, y.x)));
}

__global__ void real_to_complex_kernel(int64_t P, const double* __restrict__ x, double2* __restrict__ z) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < P) z[e] = make_double2(x[e], 0.0);
}

// ---- host side: cached twiddle tables and Bluestein filters

std::vector<int> factorize(int64_t n) {
  std::vector<int> r;
  while (n % 4 == 0) r.push_back(4), n /= 4;
  if (n % 2 == 0) r.push_back(2), n /= 2;
  for (int p = 3; p <= MAX_RADIX && n > 1; p += 2)
    while (n % p == 0) r.push_back(p), n /= p;
  if (n != 1) r.clear();  // prime factor above MAX_RADIX: Bluestein
  return r;
}

struct Tables {
  std::mutex mu;
  std::map<std::pair<int, int64_t>, std::unique_ptr<DBuf>> tw;        // (device, n) -> W_n^k
  std::map<std::tuple<int, int64_t, int>, std::unique_ptr<DBuf>> bl;  // (device, n, inverse) -> FFT_M(b)
};
Tables& tables() {
  static Tables t;
  return t;
}

int twiddle_table(int dev, int64_t n, const double2** out) {
  Tables& T = tables();
  std::lock_guard<std::mutex> lk(T.mu);
  auto& slot = T.tw[{dev, n}];
  if (!slot) {
    std::vector<double2> h(n);
    const long double PI_L = 3.141592653589793238462643383279502884L;
    for (int64_t k = 0; k < n; ++k) {
      // exp(-2 pi i k / n), argument reduced to the first octant for accuracy
      const int64_t k8 = 8 * k;
      long double c, s;
      const long double a = 2.0L * PI_L * (long double)k / (long double)n;
      if (k8 <= n || k8 >= 7 * n) {
        const long double aa = k8 >= 7 * n ? -2.0L * PI_L * (long double)(n - k) / (long double)n : a;
        c = cosl(aa), s = sinl(aa);
      } else if (k8 <= 3 * n) {
        const long double aa = 2.0L * PI_L * ((long double)(n - 4 * k)) / (4.0L * n);  // pi/2 - a
        c = sinl(aa), s = cosl(aa);
      } else if (k8 <= 5 * n) {
        const long double aa = 2.0L * PI_L * ((long double)(2 * k - n)) / (2.0L * n);  // a - pi
        c = -cosl(aa), s = -sinl(aa);
      } else {
        const long double aa = 2.0L * PI_L * ((long double)(4 * k - 3 * n)) / (4.0L * n);  // a - 3pi/2
        c = sinl(aa), s = -cosl(aa);
      }
      h[k] = make_double2((double)c, -(double)s);
    }
    auto b = std::make_unique<DBuf>();
    CKS(b->alloc(n * sizeof(double2)));
    CKS(cudaMemcpy(b->p, h.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
    slot = std::move(b);
  }
  *out = slot->as<double2>();
  return EIK_OK;
}

int launch_axis(double2* data, int64_t n, int64_t inner, int64_t outer, const std::vector<int>& rad,
                const double2* tw, int inverse, double scale, int dev, cudaStream_t st) {
  AxisArgs a{};
  a.data = data;
  a.n = n;
  a.inner = inner;
  a.outer = outer;
  a.nst = (int)rad.size();
  if (a.nst > MAX_STAGES) return eik_fail(EIK_EVALIDATION, "transform length has too many factors");
  for (int i = 0; i < a.nst; ++i) a.radix[i] = rad[i];
  a.tw = tw;
  a.inverse = inverse;
  a.scale = scale;
  DBuf scratch;
  if (n <= SMEM_LINE) {
    a.smem = 1;
    a.tl = (int)std::max<int64_t>(1, std::min<int64_t>(inner, SMEM_LINE / n));
  } else {
    a.smem = 0;
    a.tl = 1;
  }
  const int64_t tiles = outer * ((inner + a.tl - 1) / a.tl);
  if (!a.smem) {
    CKS(scratch.alloc((size_t)tiles * 2 * n * sizeof(double2)));
    a.scratch = scratch.as<double2>();
  }
  const size_t smem = a.smem ? (size_t)2 * a.tl * n * sizeof(double2) : 0;
  if (smem > 48 * 1024) CKS(cudaFuncSetAttribute(axis_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t t0 = 0; t0 < tiles; t0 += 2147483647LL) {
    axis_fft_kernel<<<(unsigned)std::min<int64_t>(tiles - t0, 2147483647LL), NT, smem, st>>>(a);
    CKS(cudaGetLastError());
  }
  if (!a.smem) CKS(cudaStreamSynchronize(st));  // scratch is freed on return
  (void)dev;
  return EIK_OK;
}

int bluestein_filter(int dev, int64_t n, int64_t M, int inverse, const double2* w2n, const double2* twM,
                     const std::vector<int>& radM, const double2** out, cudaStream_t st) {
  Tables& T = tables();
  {
    std::lock_guard<std::mutex> lk(T.mu);
    auto it = T.bl.find({dev, n, inverse});
    if (it != T.bl.end()) {
      *out = it->second->as<double2>();
      return EIK_OK;
    }
  }
  auto b = std::make_unique<DBuf>();
  CKS(b->alloc(M * sizeof(double2)));
  chirp_filter_kernel<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(n, M, w2n, inverse, b->as<double2>());
  CKS(cudaGetLastError());
  int rc = launch_axis(b->as<double2>(), M, 1, 1, radM, twM, 0, 1.0, dev, st);
  if (rc) return rc;
  CKS(cudaStreamSynchronize(st));
  std::lock_guard<std::mutex> lk(T.mu);
  auto& slot = T.bl[{dev, n, inverse}];
  if (!slot) slot = std::move(b);
  *out = slot->as<double2>();
  return EIK_OK;
}

// In-place transform of one axis: data [outer][n][inner].
int fft_axis(double2* data, int64_t n, int64_t inner, int64_t outer, int inverse, int dev, cudaStream_t st) {
  if (n == 1) return EIK_OK;
  const double scale = inverse ? 1.0 / (double)n : 1.0;
  std::vector<int> rad = factorize(n);
  if (!rad.empty()) {
    const double2* tw = nullptr;
    int rc = twiddle_table(dev, n, &tw);
    if (rc) return rc;
    return launch_axis(data, n, inner, outer, rad, tw, inverse, scale, dev, st);
  }
  int64_t M = 1;
  while (M < 2 * n - 1) M <<= 1;
  const double2 *w2n = nullptr, *twM = nullptr, *bhat = nullptr;
  int rc;
  if ((rc = twiddle_table(dev, 2 * n, &w2n))) return rc;  // exp(-i pi j / n) = W_{2n}^j
  if ((rc = twiddle_table(dev, M, &twM))) return rc;
  const std::vector<int> radM = factorize(M);
  if ((rc = bluestein_filter(dev, n, M, inverse, w2n, twM, radM, &bhat, st))) return rc;
  const int64_t nlines = outer * inner;
  DBuf tmp;
  CKS(tmp.alloc((size_t)nlines * M * sizeof(double2)));
  const int64_t tot = nlines * M;
  chirp_load_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(data, n, inner, nlines, M, w2n, inverse,
                                                                   tmp.as<double2>());
  CKS(cudaGetLastError());
  if ((rc = launch_axis(tmp.as<double2>(), M, 1, nlines, radM, twM, 0, 1.0, dev, st))) return rc;
  chirp_mul_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tmp.as<double2>(), nlines, M, bhat);
  CKS(cudaGetLastError());
  if ((rc = launch_axis(tmp.as<double2>(), M, 1, nlines, radM, twM, 1, 1.0 / (double)M, dev, st))) return rc;
  const int64_t outn = nlines * n;
  chirp_store_kernel<<<(unsigned)((outn + 255) / 256), 256, 0, st>>>(data, n, inner, nlines, M, w2n, inverse, scale,
                                                                     tmp.as<double2>());
  CKS(cudaGetLastError());
  CKS(cudaStreamSynchronize(st));  // tmp is freed on return
  return EIK_OK;
}

int fftn_device(int nd, const int64_t* shape, double2* data, int inverse, int dev, cudaStream_t st) {
  for (int ax = 0; ax < nd; ++ax) {
    int64_t outer = 1, inner = 1;
    for (int d = 0; d < ax; ++d) outer *= shape[d];
    for (int d = ax + 1; d < nd; ++d) inner *= shape[d];
    int rc = fft_axis(data, shape[ax], inner, outer, inverse, dev, st);
    if (rc) return rc;
  }
  return EIK_OK;
}

int check_shape(int nd, const int64_t* shape, int64_t* P) {
  if (nd < 1 || nd > 8 || !shape) return eik_fail(EIK_EVALIDATION, "transform rank must be 1..8");
  int64_t p = 1;
  for (int d = 0; d < nd; ++d) {
    if (shape[d] < 1) return eik_fail(EIK_EVALIDATION, "zero-length FFT axis in shape");
    if (shape[d] > (int64_t(1) << 30)) return eik_fail(EIK_EVALIDATION, "FFT axis too long");
    p *= shape[d];
  }
  *P = p;
  return EIK_OK;
}

unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

// device copy of a small int64 vector (dimension lists)
struct Dims {
  DBuf b;
  int put(const int64_t* v, int n, cudaStream_t st) {
    CKS(b.alloc(n * sizeof(int64_t)));
    CKS(cudaMemcpyAsync(b.p, v, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    return EIK_OK;
  }
  const int64_t* get() const { return b.as<int64_t>(); }
};

}  // namespace

extern "C" {

int eik_fftn(int ndim, const int64_t* shape, const double* in, int in_real, double* out, int inverse, uint32_t flags,
             int device, void* stream) {
  int64_t P = 0;
  int rc = check_shape(ndim, shape, &P);
  if (rc) return rc;
  if (!in || !out) return eik_fail(EIK_EVALIDATION, "null argument");
  CKS(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  DBuf work, rin;
  double2* z = reinterpret_cast<double2*>(out);
  if (host_out) {
    CKS(work.alloc((size_t)P * sizeof(double2)));
    z = work.as<double2>();
  }
  if (in_real) {
    const double* src = in;
    if (host_in) {
      CKS(rin.alloc((size_t)P * sizeof(double)));
      CKS(cudaMemcpyAsync(rin.p, in, P * sizeof(double), cudaMemcpyHostToDevice, st));
      src = rin.as<double>();
    }
    real_to_complex_kernel<<<blocks(P), 256, 0, st>>>(P, src, z);
    CKS(cudaGetLastError());
  } else {
    CKS(cudaMemcpyAsync(z, in, P * sizeof(double2), host_in ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  }
  if ((rc = fftn_device(ndim, shape, z, inverse, device, st))) return rc;
  if (host_out) CKS(cudaMemcpyAsync(out, z, P * sizeof(double2), cudaMemcpyDeviceToHost, st));
  if (host_in || host_out || (flags & EIK_SYNC)) CKS(cudaStreamSynchronize(st));
  return EIK_OK;
}

int eik_fft_pair(int ndim, const int64_t* pshape, const double* a, const int64_t* ashape, const double* b,
                 const int64_t* bshape, double* a_hat, double* b_hat, uint32_t flags, int device, void* stream) {
  int64_t P = 0;
  int rc = check_shape(ndim, pshape, &P);
  if (rc) return rc;
  if (!a_hat || !b_hat || !ashape || !bshape) return eik_fail(EIK_EVALIDATION, "null argument");
  int64_t Pa = 1, Pb = 1;
  for (int d = 0; d < ndim; ++d) {
    if (ashape[d] < 0 || bshape[d] < 0 || ashape[d] > pshape[d] || bshape[d] > pshape[d])
      return eik_fail(EIK_EVALIDATION, "input extent exceeds the padded shape");
    Pa *= ashape[d];
    Pb *= bshape[d];
  }
  CKS(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  DBuf da, db, z, ah, bh;
  const double* pa = a;
  const double* pb = b;
  if (host_in) {
    if (a && Pa) {
      CKS(da.alloc(Pa * sizeof(double)));
      CKS(cudaMemcpyAsync(da.p, a, Pa * sizeof(double), cudaMemcpyHostToDevice, st));
      pa = da.as<double>();
    }
    if (b && Pb) {
      CKS(db.alloc(Pb * sizeof(double)));
      CKS(cudaMemcpyAsync(db.p, b, Pb * sizeof(double), cudaMemcpyHostToDevice, st));
      pb = db.as<double>();
    }
  }
  if (!Pa) pa = nullptr;
  if (!Pb) pb = nullptr;
  Dims dp, dA, dB;
  if ((rc = dp.put(pshape, ndim, st)) || (rc = dA.put(ashape, ndim, st)) || (rc = dB.put(bshape, ndim, st))) return rc;
  CKS(z.alloc((size_t)P * sizeof(double2)));
  pad_pair_kernel<<<blocks(P), 256, 0, st>>>(ndim, dp.get(), pa, dA.get(), pb, dB.get(), P, z.as<double2>());
  CKS(cudaGetLastError());
  if ((rc = fftn_device(ndim, pshape, z.as<double2>(), 0, device, st))) return rc;
  double2* oa = reinterpret_cast<double2*>(a_hat);
  double2* ob = reinterpret_cast<double2*>(b_hat);
  if (host_out) {
    CKS(ah.alloc((size_t)P * sizeof(double2)));
    CKS(bh.alloc((size_t)P * sizeof(double2)));
    oa = ah.as<double2>();
    ob = bh.as<double2>();
  }
  unpack_pair_kernel<<<blocks(P), 256, 0, st>>>(ndim, dp.get(), P, z.as<double2>(), oa, ob);
  CKS(cudaGetLastError());
  if (host_out) {
    CKS(cudaMemcpyAsync(a_hat, oa, P * sizeof(double2), cudaMemcpyDeviceToHost, st));
    CKS(cudaMemcpyAsync(b_hat, ob, P * sizeof(double2), cudaMemcpyDeviceToHost, st));
  }
  CKS(cudaStreamSynchronize(st));  // temporaries are freed on return
  return EIK_OK;
}

int eik_ifft_window(int ndim, const int64_t* pshape, const double* hat_a, const double* hat_b,
                    const int64_t* window_start, const int64_t* window_counts, double* out_re, double* out_im,
                    uint32_t flags, int device, void* stream) {
  int64_t P = 0;
  int rc = check_shape(ndim, pshape, &P);
  if (rc) return rc;
  if (!hat_a || !window_start || !window_counts) return eik_fail(EIK_EVALIDATION, "null argument");
  int64_t Nw = 1;
  for (int d = 0; d < ndim; ++d) {
    if (window_start[d] < 0 || window_counts[d] < 0 || window_start[d] + window_counts[d] > pshape[d])
      return eik_fail(EIK_EVALIDATION, "window outside the padded shape");
    Nw *= window_counts[d];
  }
  CKS(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  DBuf ha, hb, z, ore, oim;
  const double2* pa = reinterpret_cast<const double2*>(hat_a);
  const double2* pb = reinterpret_cast<const double2*>(hat_b);
  if (host_in) {
    CKS(ha.alloc(P * sizeof(double2)));
    CKS(cudaMemcpyAsync(ha.p, hat_a, P * sizeof(double2), cudaMemcpyHostToDevice, st));
    pa = ha.as<double2>();
    if (hat_b) {
      CKS(hb.alloc(P * sizeof(double2)));
      CKS(cudaMemcpyAsync(hb.p, hat_b, P * sizeof(double2), cudaMemcpyHostToDevice, st));
      pb = hb.as<double2>();
    }
  }
  CKS(z.alloc((size_t)P * sizeof(double2)));
  combine_kernel<<<blocks(P), 256, 0, st>>>(P, pa, pb, z.as<double2>());
  CKS(cudaGetLastError());
  if ((rc = fftn_device(ndim, pshape, z.as<double2>(), 1, device, st))) return rc;
  Dims dp, d0, dn;
  if ((rc = dp.put(pshape, ndim, st)) || (rc = d0.put(window_start, ndim, st)) || (rc = dn.put(window_counts, ndim, st)))
    return rc;
  double* r = out_re;
  double* im = out_im;
  if (host_out) {
    if (out_re) { CKS(ore.alloc(Nw * sizeof(double))); r = ore.as<double>(); }
    if (out_im) { CKS(oim.alloc(Nw * sizeof(double))); im = oim.as<double>(); }
  }
  if (Nw) {
    window_kernel<<<blocks(Nw), 256, 0, st>>>(ndim, dp.get(), d0.get(), dn.get(), Nw, z.as<double2>(), r, im);
    CKS(cudaGetLastError());
  }
  if (host_out) {
    if (out_re) CKS(cudaMemcpyAsync(out_re, r, Nw * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (out_im) CKS(cudaMemcpyAsync(out_im, im, Nw * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  CKS(cudaStreamSynchronize(st));
  return EIK_OK;
}

int eik_cmul(int64_t n, const double* a, const double* b, double* out, uint32_t flags, int device, void* stream) {
  if (n < 0 || (n && (!a || !b || !out))) return eik_fail(EIK_EVALIDATION, "null argument");
  if (!n) return EIK_OK;
  CKS(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  DBuf da, db, dout;
  const double2* pa = reinterpret_cast<const double2*>(a);
  const double2* pb = reinterpret_cast<const double2*>(b);
  double2* po = reinterpret_cast<double2*>(out);
  if (host_in) {
    CKS(da.alloc(n * sizeof(double2)));
    CKS(db.alloc(n * sizeof(double2)));
    CKS(cudaMemcpyAsync(da.p, a, n * sizeof(double2), cudaMemcpyHostToDevice, st));
    CKS(cudaMemcpyAsync(db.p, b, n * sizeof(double2), cudaMemcpyHostToDevice, st));
    pa = da.as<double2>();
    pb = db.as<double2>();
  }
  if (host_out) {
    CKS(dout.alloc(n * sizeof(double2)));
    po = dout.as<double2>();
  }
  cmul_kernel<<<blocks(n), 256, 0, st>>>(n, pa, pb, po);
  CKS(cudaGetLastError());
  if (host_out) CKS(cudaMemcpyAsync(out, po, n * sizeof(double2), cudaMemcpyDeviceToHost, st));
  CKS(cudaStreamSynchronize(st));
  return EIK_OK;
}

}  // extern "C"
