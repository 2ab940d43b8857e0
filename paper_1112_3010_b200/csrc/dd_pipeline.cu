// Extended-precision (double-double) FFT convolution: SURVEY.md §8(f) rank 4.
//
// The reference's big-float path (R/convolution.py:67-143, R/distance.py:38-45,
// R/precision.py:74-99) evaluates phi = exp(-|x|/tau) * delta_Y with p-bit
// MPFR/MPC arithmetic so that far nodes, where the float64 FFT's round-off
// (~1e-16 of max phi) swamps phi, keep a positive, accurate value.  This path
// carries every sample, twiddle, butterfly and product as a double-double
// (dd.cuh, ~106-bit significand): the FFT round-off floor drops to ~1e-30 of
// max phi.  It is the reference algorithm with p = 106 except for the
// exponent range (double's), so kernel samples below ~1e-300 flush to zero
// where MPFR would keep them.
//
// Layout: full complex DD arrays over the padded lattice M0 x M1 (x M2),
// M = nextpow2(2c - 1) per axis (as the float64 path), last axis fastest,
// 32 bytes per point (re.hi, re.lo, im.hi, im.lo).  One CTA transforms one
// line in shared memory (bit-reversed load, in-place radix-2 stages, DD
// twiddles from a binary128-rounded table), so M <= 4096 per axis.
//
// Per run: impulse scatter -> forward along every axis -> per component
// (phi, grad numerators, Hessian numerators) multiply by the cached kernel
// spectrum, inverse along every axis, real part / P kept as (hi, lo) ->
// epilogue (S = -tau log phi, ratios, S_ab = t_ab + S_a S_b / tau in float64
// exactly as R/derivatives.py:99-107 does after converting the big-float
// ratios to float64).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/eikfld_b200.h"
#include "dd.cuh"
#include "launch.cuh"

void eik_dd_twiddles_host(int lmax, double* out);
void eik_dd_div_host(double a, double b, double* hi, double* lo);

namespace {

constexpr int DD_LMAX = 12;  // lines of up to 4096 points (128 KB of shared memory)
constexpr int DD_NT = 256;

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { if (p) cudaFree(p); }
  cudaError_t ensure(size_t b) {
    if (b <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, b ? b : 16);
    if (e == cudaSuccess) bytes = b ? b : 16;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// ---------------------------------------------------------------- kernels

struct DDGen {
  int D;
  int c[3], M[3];
  int ref_axis0;
  double h, tau, inv_tau;
  dd scale;  // h / tau in DD (the reference computes mpfr(h) / mpfr(tau))
  int ktype;
};

// Kernel sample at signed offsets (o0, o1, o2): the exponential in DD from
// the exact integer r^2 (R/distance.py:38-45), times the float64 directional
// factor of the float64 path (R/derivatives.py:26-57,135-153 keep the factors
// in float64 in big-float mode too).
__device__ dd dd_sample(const DDGen& g, int o0, int o1, int o2) {
  const long long r2i = (long long)o0 * o0 + (long long)o1 * o1 + (long long)o2 * o2;
  const dd r = dd_sqrt(dd{(double)r2i, 0.0});  // exact integer < 2^53
  const dd base = dd_exp(dd_neg(dd_mul(r, g.scale)));
  if (g.ktype == KT_EXP) return base;
  const double h = g.h;
  const double m0 = h * (double)o0, m1 = h * (double)o1, m2 = h * (double)o2;
  if (o0 == 0 && o1 == 0 && o2 == 0) return dd{0.0, 0.0};
  double rr;
  if (g.D == 3) rr = sqrt((m0 * m0 + m1 * m1) + m2 * m2);
  else if (g.ref_axis0 == 1) rr = sqrt(m1 * m1);
  else rr = sqrt(m0 * m0 + m1 * m1);
  const double ir = 1.0 / rr;
  double f;
  if (g.ktype <= KT_GRAD2) {
    const int a = g.ktype - KT_GRAD0 + g.ref_axis0;
    f = ((a == 0) ? m0 : (a == 1 ? m1 : m2)) / rr;
  } else {
    const double fc = m0 / rr, fs = m1 / rr, it = g.inv_tau;
    if (g.ktype == KT_HXX) f = ((-it) * fc) * fc + (fs * fs) * ir;
    else if (g.ktype == KT_HYY) f = ((-it) * fs) * fs + (fc * fc) * ir;
    else f = ((-(it + ir)) * fc) * fs;
  }
  return dd_mul_d(base, f);
}

__global__ void dd_fill_kernel(const __grid_constant__ DDGen g, double4* out, int64_t P) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int j[3] = {0, 0, 0};
    int64_t rest = i;
    for (int a = g.D - 1; a >= 0; --a) {
      j[a] = (int)(rest % g.M[a]);
      rest /= g.M[a];
    }
    int o[3] = {0, 0, 0};
    bool inside = true;
    for (int a = 0; a < g.D; ++a) {
      const int oa = wrap_offset(j[a], g.c[a], g.M[a]);
      if (oa == -0x40000000) inside = false;
      o[a] = oa;
    }
    dd v = dd{0.0, 0.0};
    if (inside) v = dd_sample(g, o[0], o[1], o[2]);
    out[i] = make_double4(v.hi, v.lo, 0.0, 0.0);
  }
}

// delta_Y on the padded lattice; validates sorted, distinct, in-range nodes
__global__ void dd_impulse_kernel(const int64_t* __restrict__ nodes, int64_t K, int D, int c0, int c1, int c2, int M1,
                                  int M2, int64_t N, double4* X, int* err) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < K; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nd = nodes[p];
    if (nd < 0 || nd >= N || (p > 0 && nodes[p - 1] >= nd)) {
      atomicExch(err, 1);
      continue;
    }
    int64_t i0, i1, i2;
    if (D == 3) {
      i2 = nd % c2;
      i1 = (nd / c2) % c1;
      i0 = nd / ((int64_t)c1 * c2);
    } else {
      i2 = 0;
      i1 = nd % c1;
      i0 = nd / c1;
    }
    (void)c0;
    const int64_t idx = D == 3 ? (i0 * M1 + i1) * M2 + i2 : i0 * M1 + i1;
    X[idx] = make_double4(1.0, 0.0, 0.0, 0.0);
  }
}

// One radix-2 DIT transform per CTA of the line l: elements base + e * inner,
// base = (l / inner) * M * inner + (l % inner).
// Pruned passes (wc < wM): only the lines whose index on the nearest lower axis lies inside the
// grid window [0, wc) of its wM padded points are transformed (the launch enumerates those);
// the others are all-zero inputs of a forward pass or unused outputs of an inverse pass.
template <bool INV>
__global__ void __launch_bounds__(DD_NT) dd_lines_kernel(double4* data, int L, int64_t inner, const double4* tw,
                                                         int lmax, int64_t wc, int64_t wM) {
  extern __shared__ double4 sl[];
  const int M = 1 << L;
  const int64_t l = blockIdx.x;
  const int64_t op = l / inner;
  const int64_t outer = (op / wc) * wM + (op % wc);
  const int64_t base = outer * ((int64_t)M * inner) + (l % inner);
  for (int e = threadIdx.x; e < M; e += blockDim.x) {
    const int be = L ? (int)(__brev((unsigned)e) >> (32 - L)) : 0;
    sl[be] = data[base + (int64_t)e * inner];
  }
  __syncthreads();
  for (int s = 1; s <= L; ++s) {
    const int half = 1 << (s - 1);
    for (int b = threadIdx.x; b < M / 2; b += blockDim.x) {
      const int pos = b & (half - 1);
      const int i = ((b >> (s - 1)) << s) + pos;
      const int j = i + half;
      const ddc w = ddc_load(tw + ((int64_t)pos << (lmax - s)));
      const ddc x = ddc_load(sl + i), y = ddc_load(sl + j);
      const ddc t = INV ? ddc_mulc(y, w) : ddc_mul(y, w);
      ddc_store(sl + i, ddc_add(x, t));
      ddc_store(sl + j, ddc_sub(x, t));
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < M; e += blockDim.x) data[base + (int64_t)e * inner] = sl[e];
}

__global__ void dd_product_kernel(const double4* __restrict__ K, const double4* __restrict__ X, double4* Y,
                                  int64_t P) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x)
    ddc_store(Y + i, ddc_mul(ddc_load(K + i), ddc_load(X + i)));
}

// Real part of the grid window [0, c) per axis, times 2^-log2(P) (exact): fld[n] = (hi, lo)
__global__ void dd_extract_kernel(const double4* __restrict__ Y, int D, int c1, int c2, int M1, int M2, int64_t N,
                                  int log2P, double2* fld) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx;
    if (D == 3) {
      const int64_t i2 = n % c2, i1 = (n / c2) % c1, i0 = n / ((int64_t)c1 * c2);
      idx = (i0 * M1 + i1) * M2 + i2;
    } else {
      idx = (n / c1) * M1 + (n % c1);
    }
    const double4 v = Y[idx];
    fld[n] = make_double2(ldexp(v.x, -log2P), ldexp(v.y, -log2P));
  }
}

struct DDEpi {
  const double2* comp[6];  // phi, grad numerators (D), Hessian numerators (3)
  int ngrad, hess;
  double tau, inv_tau;
  double *phi_hi, *phi_lo, *S;
  double* grad[3];
  double* hess_out[3];
  uint8_t* uf;
  unsigned long long* count;
  int64_t N;
};

__global__ void dd_epilogue_kernel(const __grid_constant__ DDEpi e) {
  unsigned cnt = 0;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < e.N; n += (int64_t)gridDim.x * blockDim.x) {
    const double2 p2 = e.comp[0][n];
    const dd phi = dd{p2.x, p2.y};
    const bool bad = !(phi.hi > 0.0);
    cnt += bad;
    if (e.phi_hi) e.phi_hi[n] = phi.hi;
    if (e.phi_lo) e.phi_lo[n] = phi.lo;
    if (e.uf) e.uf[n] = bad;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    if (e.S) e.S[n] = bad ? nan : (-e.tau) * (log(phi.hi) + phi.lo / phi.hi);
    double g[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < e.ngrad; ++a) {
      const double2 u = e.comp[1 + a][n];
      g[a] = bad ? nan : dd_div(dd{u.x, u.y}, phi).hi;
      if (e.grad[a]) e.grad[a][n] = g[a];
    }
    if (e.hess) {
      for (int d = 0; d < 3; ++d) {
        const double2 u = e.comp[1 + e.ngrad + d][n];
        const double t = bad ? nan : dd_div(dd{u.x, u.y}, phi).hi;
        const double a = (d == 1) ? g[1] : g[0];
        const double b = (d == 0) ? g[0] : g[1];
        e.hess_out[d][n] = t + (e.inv_tau * a) * b;  // R/derivatives.py:99-107 (float64 after the ratios)
      }
    }
  }
  if (e.count) {
    const unsigned tot = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(e.count, (unsigned long long)tot);
  }
}

int grid_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

struct eik_dd_plan {
  int dim = 0, D = 0, ref0 = 0;
  int c[3] = {1, 1, 1}, M[3] = {1, 1, 1}, L[3] = {0, 0, 0};
  int64_t N = 0, P = 0;
  int lmax = 1;
  double h = 1.0, tau = 1.0;
  uint32_t fields = 0;
  int device = 0;
  int ngrad = 0, hess = 0, nk = 0;
  DBuf tw, ks, X, Y, fld, err, count;
  std::mutex mu;
};

namespace {

// window = false: full transform of every line (kernel spectra).  window = true: the input of
// a forward transform is zero outside the grid window [0, c) per axis and only that window of
// an inverse transform is read, so the forward runs the last axis first and the inverse the
// first axis first, each pass skipping the lines that lie outside the window on the axes the
// other passes have not touched yet / have already finished (2-D: 3/4 of the line transforms,
// 3-D: 7/12).
int dd_transform(eik_dd_plan* p, double4* a, bool inv, cudaStream_t st, bool window = false) {
  for (int step = 0; step < p->D; ++step) {
    const int ax = (inv && window) ? step : p->D - 1 - step;
    int64_t inner = 1, outer = 1;
    for (int b = ax + 1; b < p->D; ++b) inner *= p->M[b];
    for (int b = 0; b < ax; ++b) outer *= window ? p->c[b] : p->M[b];
    const int64_t wc = (window && ax > 0) ? p->c[ax - 1] : 1, wM = (window && ax > 0) ? p->M[ax - 1] : 1;
    const int64_t lines = outer * inner;
    if (lines > 0x7fffffffLL) return fail(EIK_EVALIDATION, "too many lines in one double-double pass");
    const size_t smem = (size_t)p->M[ax] * sizeof(double4);
    if (inv) {
      CK(prep_kernel_attr(dd_lines_kernel<true>, smem));
      dd_lines_kernel<true><<<(unsigned)lines, DD_NT, smem, st>>>(a, p->L[ax], inner, p->tw.as<double4>(), p->lmax, wc,
                                                                  wM);
    } else {
      CK(prep_kernel_attr(dd_lines_kernel<false>, smem));
      dd_lines_kernel<false><<<(unsigned)lines, DD_NT, smem, st>>>(a, p->L[ax], inner, p->tw.as<double4>(), p->lmax, wc,
                                                                   wM);
    }
    CK(cudaGetLastError());
  }
  return EIK_OK;
}

}  // namespace

extern "C" {

int eik_dd_plan_create(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields, int device,
                       eik_dd_plan** out) {
  if (!out || !counts) return fail(EIK_EVALIDATION, "null argument");
  *out = nullptr;
  if (dim < 1 || dim > 3) return fail(EIK_EVALIDATION, "dim must be 1, 2 or 3");
  if (!(tau > 0)) return fail(EIK_EVALIDATION, "tau must be > 0");
  if (!(spacing > 0)) return fail(EIK_EVALIDATION, "spacing must be > 0");
  if (fields & (EIK_FIELD_WINDING | EIK_FIELD_DEGREE))
    return fail(EIK_EVALIDATION, "the double-double path computes phi, S, gradient and Hessian");
  if ((fields & EIK_FIELD_HESS) && dim != 2) return fail(EIK_EVALIDATION, "second derivatives are implemented for 2D grids");
  CK(cudaSetDevice(device));
  auto p = std::make_unique<eik_dd_plan>();
  p->dim = dim;
  p->device = device;
  p->h = spacing;
  p->tau = tau;
  p->fields = fields;
  // 1-D grids run as 2-D with a unit leading axis (as the float64 path)
  int64_t cc[3] = {1, 1, 1};
  p->D = dim == 3 ? 3 : 2;
  p->ref0 = dim == 1 ? 1 : 0;
  for (int a = 0; a < dim; ++a) cc[p->D - dim + a] = counts[a];
  int64_t N = 1, P = 1;
  for (int a = 0; a < p->D; ++a) {
    if (cc[a] < 1) return fail(EIK_EVALIDATION, "every axis needs at least one node");
    if (cc[a] > (int64_t(1) << (DD_LMAX - 1))) return fail(EIK_EVALIDATION, "double-double path: axes up to 2048 nodes");
    p->c[a] = (int)cc[a];
    int l = 0;
    while ((int64_t(1) << l) < 2 * cc[a] - 1) ++l;
    p->L[a] = l;
    p->M[a] = 1 << l;
    N *= cc[a];
    P *= p->M[a];
    p->lmax = std::max(p->lmax, l);
  }
  p->N = N;
  p->P = P;
  // twiddles W_MAX^j, j < MAX/2, binary128-rounded DD
  std::vector<double> tw((size_t)2 << p->lmax);
  eik_dd_twiddles_host(p->lmax, tw.data());
  CK(p->tw.ensure(tw.size() * sizeof(double)));
  CK(cudaMemcpy(p->tw.p, tw.data(), tw.size() * sizeof(double), cudaMemcpyHostToDevice));
  // kernel spectra: exp, grad (dim), Hessian (3)
  std::vector<int> kt{KT_EXP};
  if (fields & (EIK_FIELD_GRAD | EIK_FIELD_HESS)) {
    p->ngrad = dim;
    for (int a = 0; a < dim; ++a) kt.push_back(KT_GRAD0 + a);
  }
  if (fields & EIK_FIELD_HESS) {
    p->hess = 1;
    kt.push_back(KT_HXX);
    kt.push_back(KT_HYY);
    kt.push_back(KT_HXY);
  }
  p->nk = (int)kt.size();
  CK(p->ks.ensure((size_t)p->nk * P * sizeof(double4)));
  CK(p->X.ensure((size_t)P * sizeof(double4)));
  CK(p->Y.ensure((size_t)P * sizeof(double4)));
  CK(p->fld.ensure((size_t)p->nk * N * sizeof(double2)));
  CK(p->err.ensure(sizeof(int)));
  CK(p->count.ensure(sizeof(unsigned long long)));
  DDGen g{};
  g.D = p->D;
  for (int a = 0; a < 3; ++a) { g.c[a] = p->c[a]; g.M[a] = p->M[a]; }
  g.ref_axis0 = p->ref0;
  g.h = spacing;
  g.tau = tau;
  g.inv_tau = 1.0 / tau;
  eik_dd_div_host(spacing, tau, &g.scale.hi, &g.scale.lo);  // mpfr(h) / mpfr(tau), R/distance.py:41-43
  for (int k = 0; k < p->nk; ++k) {
    g.ktype = kt[k];
    double4* dst = p->ks.template as<double4>() + (int64_t)k * P;
    dd_fill_kernel<<<grid_blocks(P), 256>>>(g, dst, P);
    CK(cudaGetLastError());
    int rc = dd_transform(p.get(), dst, false, nullptr);
    if (rc) return rc;
  }
  CK(cudaDeviceSynchronize());
  *out = p.release();
  return EIK_OK;
}

int eik_dd_plan_destroy(eik_dd_plan* p) {
  delete p;
  return EIK_OK;
}

int eik_dd_run(eik_dd_plan* p, const int64_t* nodes, int64_t n_nodes, const eik_dd_outputs* o, uint32_t flags,
               void* stream) {
  if (!p || !o || !nodes) return fail(EIK_EVALIDATION, "null argument");
  if (n_nodes < 1) return fail(EIK_EVALIDATION, "empty point set");
  if (o->hess[0] && !p->hess) return fail(EIK_EVALIDATION, "plan was built without Hessian kernels");
  if ((o->grad[0] || o->hess[0]) && !p->ngrad) return fail(EIK_EVALIDATION, "plan was built without gradient kernels");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host = flags & EIK_HOST_INPUTS;
  const bool host_out = flags & EIK_HOST_OUTPUTS;
  // inputs
  DBuf dn;
  const int64_t* d_nodes = nodes;
  if (host) {
    CK(dn.ensure((size_t)n_nodes * sizeof(int64_t)));
    CK(cudaMemcpyAsync(dn.p, nodes, (size_t)n_nodes * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    d_nodes = dn.as<int64_t>();
  }
  CK(cudaMemsetAsync(p->err.p, 0, sizeof(int), st));
  CK(cudaMemsetAsync(p->count.p, 0, sizeof(unsigned long long), st));
  double4* X = p->X.as<double4>();
  double4* Y = p->Y.as<double4>();
  CK(cudaMemsetAsync(X, 0, (size_t)p->P * sizeof(double4), st));
  dd_impulse_kernel<<<grid_blocks(n_nodes), 256, 0, st>>>(d_nodes, n_nodes, p->D, p->c[0], p->c[1], p->c[2], p->M[1],
                                                         p->M[2], p->N, X, p->err.as<int>());
  CK(cudaGetLastError());
  int rc = dd_transform(p, X, false, st, true);
  if (rc) return rc;
  // components: phi, then the gradient / Hessian numerators when requested
  const bool want_grad = o->grad[0] || o->grad[1] || o->grad[2] || o->hess[0];
  const int ncomp = 1 + (want_grad ? p->ngrad : 0) + ((o->hess[0] && p->hess) ? 3 : 0);
  int log2P = 0;
  for (int a = 0; a < p->D; ++a) log2P += p->L[a];
  double2* fld = p->fld.as<double2>();
  for (int j = 0; j < ncomp; ++j) {
    dd_product_kernel<<<grid_blocks(p->P), 256, 0, st>>>(p->ks.as<double4>() + (int64_t)j * p->P, X, Y, p->P);
    CK(cudaGetLastError());
    if ((rc = dd_transform(p, Y, true, st, true))) return rc;
    dd_extract_kernel<<<grid_blocks(p->N), 256, 0, st>>>(Y, p->D, p->c[1], p->c[2], p->M[1], p->M[2], p->N, log2P,
                                                         fld + (int64_t)j * p->N);
    CK(cudaGetLastError());
  }
  // epilogue into device outputs (staged when the caller's are host arrays)
  DBuf stage;
  std::vector<std::pair<void*, void*>> copies;  // (host dst, device src)
  std::vector<size_t> sizes;
  size_t off = 0;
  auto dev = [&](void* user, size_t bytes) -> void* {
    if (!user || !host_out) return user;
    copies.push_back({user, (void*)off});
    sizes.push_back(bytes);
    off += (bytes + 255) / 256 * 256;
    return user;
  };
  const size_t f64 = (size_t)p->N * sizeof(double);
  void* ptrs[10] = {dev(o->phi_hi, f64), dev(o->phi_lo, f64), dev(o->S, f64),     dev(o->grad[0], f64),
                    dev(o->grad[1], f64), dev(o->grad[2], f64), dev(o->hess[0], f64), dev(o->hess[1], f64),
                    dev(o->hess[2], f64), dev(o->underflow, (size_t)p->N)};
  if (host_out && off) {
    CK(stage.ensure(off));
    size_t k = 0;
    for (int i = 0; i < 10; ++i)
      if (ptrs[i]) {
        const size_t at = (size_t)copies[k].second;
        copies[k].second = (char*)stage.p + at;
        ptrs[i] = copies[k].second;
        ++k;
      }
  }
  DDEpi e{};
  for (int j = 0; j < ncomp && j < 6; ++j) e.comp[j] = fld + (int64_t)j * p->N;
  e.ngrad = want_grad ? p->ngrad : 0;
  e.hess = (o->hess[0] && p->hess) ? 1 : 0;
  e.tau = p->tau;
  e.inv_tau = 1.0 / p->tau;
  e.phi_hi = (double*)ptrs[0];
  e.phi_lo = (double*)ptrs[1];
  e.S = (double*)ptrs[2];
  for (int a = 0; a < 3; ++a) { e.grad[a] = (double*)ptrs[3 + a]; e.hess_out[a] = (double*)ptrs[6 + a]; }
  e.uf = (uint8_t*)ptrs[9];
  e.count = p->count.as<unsigned long long>();
  e.N = p->N;
  dd_epilogue_kernel<<<grid_blocks(p->N), 256, 0, st>>>(e);
  CK(cudaGetLastError());
  for (size_t k = 0; k < copies.size(); ++k)
    CK(cudaMemcpyAsync(copies[k].first, copies[k].second, sizes[k], cudaMemcpyDeviceToHost, st));
  int err = 0;
  unsigned long long nuf = 0;
  CK(cudaMemcpyAsync(&err, p->err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nuf, p->count.p, sizeof(nuf), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (err) return fail(EIK_EVALIDATION, "node indices must be sorted, distinct and inside the grid");
  if (o->n_underflow) *o->n_underflow = (int64_t)nuf;
  if ((flags & EIK_CHECK_UNDERFLOW) && nuf > 0)
    return fail(EIK_EUNDERFLOW, "phi has non-positive entries after the double-double convolution; "
                                "increase the precision bits beyond 106 (not supported) or raise tau");
  return EIK_OK;
}

}  // extern "C"
