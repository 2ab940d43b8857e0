// Host side of libeikfld_b200: plans (geometry, twiddles, cached kernel
// spectra, workspaces), the pass schedule of the 2-D / 3-D pipelines, and the
// extern "C" entry points declared in include/eikfld_b200.h.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/eikfld_b200.h"
#include "launch.cuh"

using namespace eik;

namespace {

thread_local std::string g_err;

}  // namespace

int eik_fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace {
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t b) {
    if (b <= bytes && p) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&p, b ? b : 16);
    if (e == cudaSuccess) bytes = b ? b : 16;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

int ilog2_exact(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

constexpr int LMAX_SUPPORTED = 13;  // line lengths up to 8192 (grid axes up to 4096 nodes)

void build_twiddles(int lmax, std::vector<double2>& tw) {
  const int64_t M = int64_t(1) << lmax;
  const int64_t Q = M / 4, O = M / 8;
  const long double PI_L = 3.141592653589793238462643383279502884L;
  tw.resize(M);
  for (int64_t j = 0; j < M; ++j) {
    const int64_t quad = j / Q, k = j % Q;
    double c, s;  // cos / sin of 2 pi k / M, k in [0, M/4)
    if (k == 0) {
      c = 1.0;
      s = 0.0;
    } else if (k <= O) {
      const long double a = 2.0L * PI_L * (long double)k / (long double)M;
      c = (double)cosl(a);
      s = (double)sinl(a);
    } else {
      const long double a = 2.0L * PI_L * (long double)(Q - k) / (long double)M;
      c = (double)sinl(a);
      s = (double)cosl(a);
    }
    double cc, ss;  // angle + quad * pi/2
    switch (quad) {
      case 0: cc = c; ss = s; break;
      case 1: cc = -s; ss = c; break;
      case 2: cc = -c; ss = -s; break;
      default: cc = s; ss = -c; break;
    }
    tw[j] = make_double2(cc, -ss);  // exp(-i angle)
  }
}

struct KDev {
  int ktype = 0;
  int imag = 0;
  int odd0 = 0;
  double sign = 1.0;
  DevBuf buf;  // folded real/imag spectrum [(M0/2+1) x lines]
};

}  // namespace

struct eik_plan {
  int dim = 0, D = 0, ref0 = 0;
  int c[3] = {1, 1, 1}, M[3] = {1, 1, 1}, L[3] = {0, 0, 0};
  int64_t N = 0, H = 0, lines = 0;
  double h = 1.0, tau = 1.0;
  uint32_t fields = 0;
  int device = 0;
  int lmax = 2;
  DevBuf tw;
  std::vector<std::unique_ptr<KDev>> kdist;  // EXP, GRAD..., HXX, HYY, HXY (subset)
  int k_exp = -1, k_grad = -1, k_hess = -1;
  std::vector<std::unique_ptr<KDev>> ksign;
  DevBuf comp, vin, rowid, cols, rowptr, srowid, scols, srowptr, off1, soff;
  DevBuf h_nodes, h_off, h_snodes, h_sw, stage, counter, err, work;
  std::mutex mu;
  cudaEvent_t ev[2 * EIK_NPASS] = {};
  bool ev_used[EIK_NPASS] = {};
  ~eik_plan() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }

  int64_t comp_elems() const {  // complex elements of one component of one item
    return D == 2 ? (int64_t)c[0] * H : (int64_t)c[0] * M[1] * H;
  }
  int64_t held() const {
    int64_t b = tw.bytes + comp.bytes + vin.bytes + rowid.bytes + cols.bytes + rowptr.bytes + srowid.bytes +
                scols.bytes + srowptr.bytes + stage.bytes + work.bytes + h_nodes.bytes + h_off.bytes +
                h_snodes.bytes + h_sw.bytes;
    for (auto& k : kdist) b += k->buf.bytes;
    for (auto& k : ksign) b += k->buf.bytes;
    return b;
  }
};

namespace {

int setup_geometry(eik_plan* p, int dim, const int64_t* counts, double h) {
  if (dim < 1 || dim > 3) return fail(EIK_EVALIDATION, "dimension must be 1, 2 or 3");
  if (!(h > 0)) return fail(EIK_EVALIDATION, "spacing must be > 0");
  p->dim = dim;
  p->D = dim == 3 ? 3 : 2;
  p->ref0 = dim == 1 ? 1 : 0;
  int64_t cc[3] = {1, 1, 1};
  for (int a = 0; a < dim; ++a) {
    if (counts[a] < 1) return fail(EIK_EVALIDATION, "zero-length axis");
    cc[a] = counts[a];
  }
  if (dim == 1) { cc[0] = 1; cc[1] = counts[0]; }
  int64_t N = 1;
  for (int a = 0; a < p->D; ++a) {
    if (cc[a] > (int64_t(1) << (LMAX_SUPPORTED - 1))) return fail(EIK_EVALIDATION, "axis longer than 4096 nodes");
    p->c[a] = (int)cc[a];
    const int64_t need = 2 * cc[a] - 1;
    p->L[a] = ilog2_exact(need);
    p->M[a] = 1 << p->L[a];
    N *= cc[a];
  }
  if (p->L[p->D - 1] < 1) p->L[p->D - 1] = 1, p->M[p->D - 1] = 2;
  p->N = N;
  const int last = p->D - 1;
  p->H = p->M[last] / 2 + 1;
  p->lines = p->D == 2 ? p->H : (int64_t)p->M[1] * p->H;
  p->h = h;
  int lm = 2;
  for (int a = 0; a < p->D; ++a) lm = std::max(lm, p->L[a]);
  p->lmax = lm;
  std::vector<double2> tw;
  build_twiddles(lm, tw);
  CK(p->tw.ensure(tw.size() * sizeof(double2)));
  CK(cudaMemcpy(p->tw.p, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
  return EIK_OK;
}

GenArgs gen_args(const eik_plan* p, int ktype, double sign) {
  GenArgs g{};
  g.D = p->D;
  for (int a = 0; a < 3; ++a) { g.c[a] = p->c[a]; g.M[a] = p->M[a]; }
  g.ref_axis0 = p->ref0;
  g.h = p->h;
  g.tau = p->tau;
  g.inv_tau = 1.0 / p->tau;
  g.sign = sign;
  g.ktype = ktype;
  return g;
}

// Forward-transform one real padded lattice function (generated by `g`) and
// keep its real or imaginary part, transposed and folded: dst[k0 * lines + l].
// work must hold M0 * lines complex values.
int spectrum_of(eik_plan* p, const GenArgs& g, int part, double* dst_re, double2* dst_c, double2* work,
                cudaStream_t st) {
  const int last = p->D - 1;
  const int64_t nrows = p->D == 2 ? p->M[0] : (int64_t)p->M[0] * p->M[1];
  const double2* tw = p->tw.as<double2>();
  int rc = launch_r2c(p->L[last] - 1, g, nrows, work, p->H, tw, p->lmax, st);
  if (rc) return rc;
  if (p->D == 3) {
    LinesArgs la{};
    la.in[0] = work;
    la.out[0] = work;
    la.nlines = (int64_t)p->M[0] * p->H;
    la.inner = p->H;
    la.outer_in = la.outer_out = (int64_t)p->M[1] * p->H;
    la.es_in = la.es_out = p->H;
    la.n_valid = la.n_out = p->M[1];
    la.scale = 1.0;
    la.tw = tw;
    la.lmax = p->lmax;
    rc = launch_lines<false, false>(p->L[1], la, 1, st);
    if (rc) return rc;
  }
  ColArgs a{};
  a.nlines = p->lines;
  a.n_valid = p->M[0];
  a.n_out = p->M[0];
  a.n_in = 1;
  a.din[0] = work;
  a.din_es = p->lines;
  a.din_item = 0;
  a.spec_mode = part;
  a.spec_re[0] = dst_re;
  a.out[0] = dst_c;
  a.spec_ld = p->lines;
  a.tw = tw;
  a.lmax = p->lmax;
  return launch_col<IN_DENSE, OUT_SPECTRUM, false>(p->L[0], a, 1, st);
}

int add_kernel(eik_plan* p, std::vector<std::unique_ptr<KDev>>& v, int ktype, int n_odd_axes, bool odd0,
               double sign, double2* work, cudaStream_t st) {
  auto k = std::make_unique<KDev>();
  k->ktype = ktype;
  k->imag = n_odd_axes % 2;
  k->odd0 = odd0 ? 1 : 0;
  k->sign = sign;
  const int64_t n = (int64_t)(p->M[0] / 2 + 1) * p->lines;
  CK(k->buf.ensure(n * sizeof(double)));
  int rc = spectrum_of(p, gen_args(p, ktype, sign), k->imag ? SPEC_IMAG_T : SPEC_REAL_T, k->buf.as<double>(), nullptr,
                       work, st);
  if (rc) return rc;
  v.push_back(std::move(k));
  return EIK_OK;
}

KSpec kspec_of(const eik_plan* p, const KDev& k) {
  KSpec s{};
  s.re = k.buf.as<double>();
  s.ld = p->lines;
  s.imag = k.imag;
  s.odd0 = k.odd0;
  return s;
}

// per-row CSR for a sorted node list (validates order and bounds)
int prep_nodes(eik_plan* p, const int64_t* d_nodes, const int64_t* d_off, int64_t K, int64_t items,
               DevBuf& rowid, DevBuf& cols, DevBuf& rowptr, cudaStream_t st) {
  const int last = p->D - 1;
  const int64_t rows_per_item = p->N / p->c[last];
  const int64_t nrows = rows_per_item * items;
  CK(rowid.ensure(std::max<int64_t>(K, 1) * sizeof(int64_t)));
  CK(cols.ensure(std::max<int64_t>(K, 1) * sizeof(int32_t)));
  CK(rowptr.ensure((nrows + 1) * sizeof(int64_t)));
  CK(p->err.ensure(sizeof(int)));
  CK(cudaMemsetAsync(p->err.p, 0, sizeof(int), st));
  if (K > 0) {
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>(1024, (K / std::max<int64_t>(items, 1) + 255) / 256));
    prep_nodes_kernel<<<dim3((unsigned)per, (unsigned)items), 256, 0, st>>>(
        d_nodes, d_off, p->c[last], rows_per_item, p->N, rowid.as<int64_t>(), cols.as<int32_t>(), p->err.as<int>());
    CK(cudaGetLastError());
  }
  rowptr_kernel<<<(unsigned)((nrows + 1 + 255) / 256), 256, 0, st>>>(rowid.as<int64_t>(), K, nrows,
                                                                       rowptr.as<int64_t>());
  CK(cudaGetLastError());
  return EIK_OK;
}

}  // namespace

extern "C" {

const char* eik_last_error(void) { return g_err.c_str(); }
int eik_version(void) { return 10000; }

int eik_plan_create(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields, int device,
                    eik_plan** out) {
  if (!out || !counts) return fail(EIK_EVALIDATION, "null argument");
  *out = nullptr;
  if (!(tau > 0)) return fail(EIK_EVALIDATION, "tau must be > 0");
  if ((fields & EIK_FIELD_HESS) && dim != 2) return fail(EIK_EVALIDATION, "second derivatives are implemented for 2D grids");
  if ((fields & EIK_FIELD_WINDING) && dim != 2) return fail(EIK_EVALIDATION, "winding numbers need a 2D grid");
  if ((fields & EIK_FIELD_DEGREE) && dim != 3) return fail(EIK_EVALIDATION, "topological degree needs a 3D grid");
  CK(cudaSetDevice(device));
  auto p = std::make_unique<eik_plan>();
  p->device = device;
  p->tau = tau;
  p->fields = fields;
  int rc = setup_geometry(p.get(), dim, counts, spacing);
  if (rc) return rc;
  cudaStream_t st = nullptr;
  const bool need_phi = fields & (EIK_FIELD_PHI | EIK_FIELD_S | EIK_FIELD_GRAD | EIK_FIELD_HESS);
  const bool need_sign = fields & (EIK_FIELD_WINDING | EIK_FIELD_DEGREE);
  if (need_phi || need_sign) {
    CK(p->work.ensure((size_t)p->M[0] * p->lines * sizeof(double2)));
    double2* work = p->work.as<double2>();
    if (need_phi) {
      p->k_exp = (int)p->kdist.size();
      if ((rc = add_kernel(p.get(), p->kdist, KT_EXP, 0, false, 1.0, work, st))) return rc;
    }
    if (fields & (EIK_FIELD_GRAD | EIK_FIELD_HESS)) {
      p->k_grad = (int)p->kdist.size();
      for (int a = 0; a < dim; ++a) {
        const int internal_axis = a + p->ref0;
        if ((rc = add_kernel(p.get(), p->kdist, KT_GRAD0 + a, 1, internal_axis == 0, 1.0, work, st))) return rc;
      }
    }
    if (fields & EIK_FIELD_HESS) {
      p->k_hess = (int)p->kdist.size();
      if ((rc = add_kernel(p.get(), p->kdist, KT_HXX, 0, false, 1.0, work, st))) return rc;
      if ((rc = add_kernel(p.get(), p->kdist, KT_HYY, 0, false, 1.0, work, st))) return rc;
      if ((rc = add_kernel(p.get(), p->kdist, KT_HXY, 2, true, 1.0, work, st))) return rc;
    }
    if (fields & EIK_FIELD_WINDING) {
      // h = ksr*g1 - kcr*g2 (R/sign.py:126-127): y/r^2 for g1, -(x/r^2) for g2
      if ((rc = add_kernel(p.get(), p->ksign, KT_RAT2_1, 1, false, 1.0, work, st))) return rc;
      if ((rc = add_kernel(p.get(), p->ksign, KT_RAT2_0, 1, true, -1.0, work, st))) return rc;
    }
    if (fields & EIK_FIELD_DEGREE) {
      for (int a = 0; a < 3; ++a)
        if ((rc = add_kernel(p.get(), p->ksign, KT_RAT3_0 + a, 1, a == 0, 1.0, work, st))) return rc;
    }
    CK(cudaDeviceSynchronize());
    p->work.release();
  }
  CK(p->counter.ensure(sizeof(unsigned long long)));
  CK(p->off1.ensure(2 * sizeof(int64_t)));
  *out = p.release();
  return EIK_OK;
}

int eik_plan_destroy(eik_plan* plan) {
  if (!plan) return EIK_OK;
  cudaSetDevice(plan->device);
  delete plan;
  return EIK_OK;
}

int eik_pass_times(eik_plan* p, double* ms, int n) {
  if (!p || !ms) return fail(EIK_EVALIDATION, "null argument");
  for (int i = 0; i < n && i < EIK_NPASS; ++i) {
    ms[i] = -1.0;
    if (!p->ev_used[i]) continue;
    CK(cudaEventSynchronize(p->ev[2 * i + 1]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, p->ev[2 * i], p->ev[2 * i + 1]));
    ms[i] = f;
  }
  return EIK_OK;
}

int eik_plan_info(const eik_plan* p, int64_t* padded, int64_t* lines, int64_t* bytes) {
  if (!p) return fail(EIK_EVALIDATION, "null plan");
  if (padded)
    for (int a = 0; a < 3; ++a) padded[a] = a < p->D ? p->M[a] : 1;
  if (lines) *lines = p->lines;
  if (bytes) *bytes = p->held();
  return EIK_OK;
}

int eik_run(eik_plan* p, const eik_inputs* in, const eik_outputs* out, uint32_t flags, void* stream) {
  if (!p || !in || !out) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t B = in->batch < 1 ? 1 : in->batch;
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  const bool want_grad = out->grad[0] || out->grad[1] || out->grad[2];
  const bool want_hess = out->hess[0] || out->hess[1] || out->hess[2];
  const bool want_sign = out->mu || out->mask;
  const bool want_phi = out->phi || out->S || want_grad || want_hess || out->underflow || out->n_underflow ||
                        out->d_underflow_count || (flags & EIK_CHECK_UNDERFLOW);
  if (want_phi && p->k_exp < 0) return fail(EIK_EVALIDATION, "plan was built without the distance kernels");
  if ((want_grad || want_hess) && p->k_grad < 0) return fail(EIK_EVALIDATION, "plan was built without gradient kernels");
  if (want_hess && p->k_hess < 0) return fail(EIK_EVALIDATION, "plan was built without Hessian kernels");
  if (want_sign && p->ksign.empty()) return fail(EIK_EVALIDATION, "plan was built without sign kernels");
  if (want_sign && B != 1) return fail(EIK_EVALIDATION, "sign fields are computed for batch 1");
  if (want_phi && (!in->nodes || in->n_nodes < 1)) return fail(EIK_EVALIDATION, "empty point set");
  if (want_sign && (in->n_sign_nodes < 1 || !in->sign_nodes || !in->sign_weights))
    return fail(EIK_EVALIDATION, "sign field needs weighted nodes");
  if (B > 1 && !in->item_offsets) return fail(EIK_EVALIDATION, "batch > 1 needs item offsets");

  const int D = p->D, last = D - 1;
  const double2* tw = p->tw.as<double2>();
  const bool prof = flags & EIK_PROFILE;
  for (bool& u : p->ev_used) u = false;
  auto mark = [&](int pass, bool end) -> int {
    if (!prof) return EIK_OK;
    cudaEvent_t& e = p->ev[2 * pass + (end ? 1 : 0)];
    if (!e) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, st));
    if (end) p->ev_used[pass] = true;
    return EIK_OK;
  };
  // ---- inputs
  const int64_t* d_nodes = in->nodes;
  const int64_t* d_off = in->item_offsets;
  const int64_t* d_snodes = in->sign_nodes;
  const double* d_sw = in->sign_weights;
  if (want_phi && host_in) {
    CK(p->h_nodes.ensure(in->n_nodes * sizeof(int64_t)));
    CK(cudaMemcpyAsync(p->h_nodes.p, in->nodes, in->n_nodes * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    d_nodes = p->h_nodes.as<int64_t>();
    if (B > 1) {
      CK(p->h_off.ensure((B + 1) * sizeof(int64_t)));
      CK(cudaMemcpyAsync(p->h_off.p, in->item_offsets, (B + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      d_off = p->h_off.as<int64_t>();
    }
  }
  if (want_phi && B == 1) {
    if (!d_off || host_in) {
      const int64_t off[2] = {0, in->n_nodes};
      CK(cudaMemcpyAsync(p->off1.p, off, sizeof(off), cudaMemcpyHostToDevice, st));
      d_off = p->off1.as<int64_t>();
    }
  }
  if (want_sign) {
    const int64_t Ks = in->n_sign_nodes;
    if (host_in) {
      CK(p->h_snodes.ensure(Ks * sizeof(int64_t)));
      CK(p->h_sw.ensure(Ks * p->dim * sizeof(double)));
      CK(cudaMemcpyAsync(p->h_snodes.p, in->sign_nodes, Ks * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(p->h_sw.p, in->sign_weights, Ks * p->dim * sizeof(double), cudaMemcpyHostToDevice, st));
      d_snodes = p->h_snodes.as<int64_t>();
      d_sw = p->h_sw.as<double>();
    }
    CK(p->soff.ensure(2 * sizeof(int64_t)));
    const int64_t off[2] = {0, Ks};
    CK(cudaMemcpyAsync(p->soff.p, off, sizeof(off), cudaMemcpyHostToDevice, st));
  }
  // ---- outputs (device pointers, possibly staged)
  const int64_t NB = p->N * B;
  struct OutSlot { void* user; size_t bytes; void* dev; };
  std::vector<OutSlot> slots;
  auto reg = [&](void* user, size_t elem) -> void* {
    if (!user) return nullptr;
    if (!host_out) return user;
    slots.push_back({user, (size_t)NB * elem, nullptr});
    return (void*)1;  // placeholder, resolved below
  };
  double* o_phi = (double*)reg(out->phi, 8);
  double* o_S = (double*)reg(out->S, 8);
  double* o_g[3] = {(double*)reg(out->grad[0], 8), (double*)reg(out->grad[1], 8), (double*)reg(out->grad[2], 8)};
  double* o_h[3] = {(double*)reg(out->hess[0], 8), (double*)reg(out->hess[1], 8), (double*)reg(out->hess[2], 8)};
  double* o_mu = (double*)reg(out->mu, 8);
  uint8_t* o_mask = (uint8_t*)reg(out->mask, 1);
  uint8_t* o_uf = (uint8_t*)reg(out->underflow, 1);
  if (host_out && !slots.empty()) {
    size_t tot = 0;
    for (auto& s : slots) tot += (s.bytes + 255) / 256 * 256;
    CK(p->stage.ensure(tot));
    size_t off = 0;
    for (auto& s : slots) { s.dev = (char*)p->stage.p + off; off += (s.bytes + 255) / 256 * 256; }
    size_t i = 0;
    auto fix = [&](void* ptr) -> void* { return ptr ? slots[i++].dev : nullptr; };
    o_phi = (double*)fix(o_phi); o_S = (double*)fix(o_S);
    for (auto& g : o_g) g = (double*)fix(g);
    for (auto& h : o_h) h = (double*)fix(h);
    o_mu = (double*)fix(o_mu); o_mask = (uint8_t*)fix(o_mask); o_uf = (uint8_t*)fix(o_uf);
  }
  // ---- component buffers
  const int ngrad = (want_grad || want_hess) ? p->dim : 0;
  const int n_dist = want_phi ? 1 + ngrad + (want_hess ? 3 : 0) : 0;
  const int n_comp = n_dist + (want_sign ? 1 : 0);
  const int64_t ce = p->comp_elems();
  CK(p->comp.ensure((size_t)n_comp * B * ce * sizeof(double2)));
  double2* comp = p->comp.as<double2>();
  auto compp = [&](int j) { return comp + (int64_t)j * B * ce; };
  int rc;
  const int n_in_sign = p->dim;
  if (D == 3) CK(p->vin.ensure((size_t)std::max(want_phi ? 1 : 0, want_sign ? n_in_sign : 0) * B * ce * sizeof(double2)));
  // ---- forward + multiply + first inverse (per group)
  auto run_group = [&](bool sign_group) -> int {
    const int64_t K = sign_group ? in->n_sign_nodes : in->n_nodes;
    DevBuf& rid = sign_group ? p->srowid : p->rowid;
    DevBuf& cl = sign_group ? p->scols : p->cols;
    DevBuf& rp = sign_group ? p->srowptr : p->rowptr;
    const int64_t items = sign_group ? 1 : B;
    int r = mark(EIK_PASS_PREP, false);
    if (r) return r;
    r = prep_nodes(p, sign_group ? d_snodes : d_nodes, sign_group ? p->soff.as<int64_t>() : d_off, K, items, rid, cl,
                       rp, st);
    if (r) return r;
    ColArgs a{};
    a.rowptr = rp.as<int64_t>();
    a.cols = cl.as<int32_t>();
    a.n_in = sign_group ? n_in_sign : 1;
    for (int i = 0; i < 3; ++i) a.w[i] = (sign_group && i < n_in_sign) ? d_sw + (int64_t)i * K : nullptr;
    a.last_shift = p->lmax - p->L[last];
    a.last_mask = p->M[last] - 1;
    a.tw = tw;
    a.lmax = p->lmax;
    if ((r = mark(EIK_PASS_PREP, true))) return r;
    const int pass = sign_group ? EIK_PASS_COL_SIGN : EIK_PASS_COL;
    if ((r = mark(pass, false))) return r;
    const auto& kv = sign_group ? p->ksign : p->kdist;
    auto set_ks = [&](ColArgs& x) {
      if (sign_group) {
        x.n_comp = 1;
        for (int i = 0; i < n_in_sign; ++i) x.ks[i] = kspec_of(p, *kv[i]);
        x.out[0] = compp(n_dist);
      } else {
        int j = 0;
        x.ks[j] = kspec_of(p, *kv[p->k_exp]); x.out[j] = compp(j); ++j;
        for (int d = 0; d < ngrad; ++d, ++j) { x.ks[j] = kspec_of(p, *kv[p->k_grad + d]); x.out[j] = compp(j); }
        if (want_hess)
          for (int d = 0; d < 3; ++d, ++j) { x.ks[j] = kspec_of(p, *kv[p->k_hess + d]); x.out[j] = compp(j); }
        x.n_comp = j;
      }
    };
    if (D == 2) {
      a.nlines = p->H;
      a.n_valid = p->c[0];
      a.n_out = p->c[0];
      a.rows_per_item = p->c[0];
      a.out_es = p->H;
      a.out_item = ce;
      set_ks(a);
      r = sign_group ? launch_col<IN_SPARSE, OUT_SUM, true>(p->L[0], a, items, st)
                     : launch_col<IN_SPARSE, OUT_COMPS, true>(p->L[0], a, items, st);
      return r ? r : mark(pass, true);
    }
    // 3-D: plane pass (axis 2 impulse DFT + axis 1 FFT) into vin, then axis 0 fused
    ColArgs pa = a;
    pa.nlines = p->H;
    pa.n_valid = p->c[1];
    pa.rows_per_item = p->c[1];
    pa.spec_mode = SPEC_COMPLEX;
    pa.out_es = p->H;
    pa.out_item = (int64_t)p->M[1] * p->H;
    double2* V = p->vin.as<double2>();
    for (int i = 0; i < pa.n_in; ++i) pa.out[i] = V + (int64_t)i * B * ce;
    r = launch_col<IN_SPARSE, OUT_SPECTRUM, true>(p->L[1], pa, items * p->c[0], st);
    if (r) return r;
    ColArgs da{};
    da.nlines = p->lines;
    da.n_valid = p->c[0];
    da.n_out = p->c[0];
    da.n_in = pa.n_in;
    for (int i = 0; i < da.n_in; ++i) da.din[i] = V + (int64_t)i * B * ce;
    da.din_es = p->lines;
    da.din_item = ce;
    da.out_es = p->lines;
    da.out_item = ce;
    da.tw = tw;
    da.lmax = p->lmax;
    set_ks(da);
    r = sign_group ? launch_col<IN_DENSE, OUT_SUM, true>(p->L[0], da, items, st)
                   : launch_col<IN_DENSE, OUT_COMPS, true>(p->L[0], da, items, st);
    return r ? r : mark(pass, true);
  };
  if (want_phi && (rc = run_group(false))) return rc;
  if (want_sign && (rc = run_group(true))) return rc;
  if (D == 3) {  // inverse along axis 1, in place, keep rows [0, c1)
    LinesArgs la{};
    for (int j = 0; j < n_comp; ++j) { la.in[j] = compp(j); la.out[j] = compp(j); }
    la.nlines = B * p->c[0] * p->H;
    la.inner = p->H;
    la.outer_in = la.outer_out = (int64_t)p->M[1] * p->H;
    la.es_in = la.es_out = p->H;
    la.n_valid = p->M[1];
    la.n_out = p->c[1];
    la.scale = 1.0;
    la.tw = tw;
    la.lmax = p->lmax;
    // components of the sign group have batch 1; the comp buffer is laid out per
    // component with B items, so lines of absent items are simply unused
    if ((rc = mark(EIK_PASS_LINES, false))) return rc;
    if ((rc = launch_lines<true, false>(p->L[1], la, n_comp, st))) return rc;
    if ((rc = mark(EIK_PASS_LINES, true))) return rc;
  }
  // ---- last axis c2r + epilogue
  RowArgs ra{};
  if (D == 2) {
    ra.rows = p->c[0];
    ra.rows_a = p->c[0];
    ra.stride_a = 0;
    ra.stride_b = p->H;
  } else {
    ra.rows = (int64_t)p->c[0] * p->c[1];
    ra.rows_a = p->c[1];
    ra.stride_a = (int64_t)p->M[1] * p->H;
    ra.stride_b = p->H;
  }
  ra.comp_item = ce;
  ra.n_out = p->c[last];
  for (int j = 0; j < n_comp; ++j) ra.comp[j] = compp(j);
  ra.n_comp = n_comp;
  ra.c_phi = want_phi ? 0 : -1;
  ra.c_grad = ngrad ? 1 : -1;
  ra.ngrad = ngrad;
  ra.c_hess = want_hess ? 1 + ngrad : -1;
  ra.c_sign = want_sign ? n_dist : -1;
  ra.sign_mode = p->dim == 2 ? 1 : 2;
  double scale = 1.0;
  for (int a = 0; a < D; ++a) scale /= (double)p->M[a];
  ra.scale = scale;
  ra.tau = p->tau;
  ra.inv_tau = 1.0 / p->tau;
  ra.S = o_S;
  for (int d = 0; d < 3; ++d) { ra.grad[d] = o_g[d]; ra.hess[d] = o_h[d]; }
  ra.mu = o_mu;
  ra.mask = o_mask;
  ra.uf = o_uf;
  ra.phi_out = o_phi;
  ra.N = p->N;
  const bool count = want_phi && (out->n_underflow || out->d_underflow_count || (flags & EIK_CHECK_UNDERFLOW));
  unsigned long long* ctr = out->d_underflow_count ? out->d_underflow_count : p->counter.as<unsigned long long>();
  if (count) {
    if (!out->d_underflow_count) CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    ra.uf_count = ctr;
  }
  ra.tw = tw;
  ra.lmax = p->lmax;
  if (want_sign && B > 1) return fail(EIK_EVALIDATION, "sign with batch");
  if ((rc = mark(EIK_PASS_ROW, false))) return rc;
  if ((rc = launch_row(p->L[last] - 1, ra, B, st))) return rc;
  if ((rc = mark(EIK_PASS_ROW, true))) return rc;
  // ---- copy back / sync / checks
  for (auto& s : slots) CK(cudaMemcpyAsync(s.user, s.dev, s.bytes, cudaMemcpyDeviceToHost, st));
  const bool sync = host_out || (flags & (EIK_SYNC | EIK_CHECK_UNDERFLOW)) || out->n_underflow;
  int err_flag = 0;
  unsigned long long nuf = 0;
  if (sync) {
    if (want_phi || want_sign) CK(cudaMemcpyAsync(&err_flag, p->err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (count) CK(cudaMemcpyAsync(&nuf, ctr, sizeof(nuf), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err_flag) return fail(EIK_EVALIDATION, "node indices must be sorted, distinct and inside the grid");
    if (out->n_underflow) *out->n_underflow = (int64_t)nuf;
    if ((flags & EIK_CHECK_UNDERFLOW) && nuf > 0)
      return fail(EIK_EUNDERFLOW, "phi has non-positive entries after convolution; increase the precision bits "
                                  "(e.g. --precision big:512) or raise tau");
  }
  return EIK_OK;
}

// ---------------------------------------------------------------------------
// Engine-level convolution with arbitrary kernels and a dense field.

int eik_convolve(int dim, const int64_t* counts, const double* kernels, int64_t n_kernels, const int64_t* kshape,
                 const double* field, double* out, uint32_t flags, int device, void* stream) {
  if (!counts || !kernels || !kshape || !field || !out || n_kernels < 1) return fail(EIK_EVALIDATION, "null argument");
  CK(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  eik_plan P;
  P.tau = 1.0;
  P.device = device;
  int rc = setup_geometry(&P, dim, counts, 1.0);
  if (rc) return rc;
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  int64_t ks[3] = {1, 1, 1}, kn = 1;
  for (int a = 0; a < dim; ++a) {
    if (kshape[a] % 2 == 0) return fail(EIK_EVALIDATION, "kernel axes must have odd length (centered)");
    if (kshape[a] < 2 * counts[a] - 1) return fail(EIK_EVALIDATION, "kernel extent must cover the grid extent");
    kn *= kshape[a];
  }
  // internal-axis shape of the kernel (1-D grids get a leading unit axis)
  if (dim == 1) { ks[0] = 1; ks[1] = kshape[0]; }
  else for (int a = 0; a < dim; ++a) ks[a] = kshape[a];
  const int D = P.D, last = D - 1;
  const double2* tw = P.tw.as<double2>();
  DevBuf dk, df, dout, work, kc, Tb, comp;
  const double* d_k = kernels;
  const double* d_f = field;
  if (host_in) {
    CK(dk.ensure(n_kernels * kn * sizeof(double)));
    CK(df.ensure(P.N * sizeof(double)));
    CK(cudaMemcpyAsync(dk.p, kernels, n_kernels * kn * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(df.p, field, P.N * sizeof(double), cudaMemcpyHostToDevice, st));
    d_k = dk.as<double>();
    d_f = df.as<double>();
  }
  double* d_out = out;
  if (host_out) {
    CK(dout.ensure(n_kernels * P.N * sizeof(double)));
    d_out = dout.as<double>();
  }
  CK(work.ensure((size_t)P.M[0] * P.lines * sizeof(double2)));
  CK(kc.ensure((size_t)std::min<int64_t>(n_kernels, MAXC) * P.M[0] * P.lines * sizeof(double2)));
  const int64_t ce = P.comp_elems();
  CK(comp.ensure((size_t)std::min<int64_t>(n_kernels, MAXC) * ce * sizeof(double2)));
  // forward transform of the field: rows -> (axis 1 for 3-D) -> kept in Tb
  const int64_t trow = D == 2 ? P.c[0] : (int64_t)P.c[0] * P.M[1];
  CK(Tb.ensure((size_t)trow * P.H * sizeof(double2)));
  GenArgs gf = gen_args(&P, KT_FIELD, 1.0);
  gf.field = d_f;
  gf.field_is_grid = 1;
  {
    int64_t s = 1;
    for (int a = D - 1; a >= 0; --a) { gf.fstride[a] = s; s *= P.c[a]; }
  }
  if ((rc = launch_r2c(P.L[last] - 1, gf, trow, Tb.as<double2>(), P.H, tw, P.lmax, st))) return rc;
  if (D == 3) {
    LinesArgs la{};
    la.in[0] = la.out[0] = Tb.as<double2>();
    la.nlines = (int64_t)P.c[0] * P.H;
    la.inner = P.H;
    la.outer_in = la.outer_out = (int64_t)P.M[1] * P.H;
    la.es_in = la.es_out = P.H;
    la.n_valid = P.c[1];
    la.n_out = P.M[1];
    la.scale = 1.0;
    la.tw = tw;
    la.lmax = P.lmax;
    if ((rc = launch_lines<false, true>(P.L[1], la, 1, st))) return rc;
  }
  double scale = 1.0;
  for (int a = 0; a < D; ++a) scale /= (double)P.M[a];
  for (int64_t k0 = 0; k0 < n_kernels; k0 += MAXC) {
    const int nk = (int)std::min<int64_t>(MAXC, n_kernels - k0);
    ColArgs a{};
    for (int j = 0; j < nk; ++j) {
      GenArgs gk = gen_args(&P, KT_FIELD, 1.0);
      gk.field = d_k + (k0 + j) * kn;
      gk.field_is_grid = 0;
      int64_t s = 1;
      for (int ax = D - 1; ax >= 0; --ax) {
        gk.fstride[ax] = s;
        gk.fcenter[ax] = (ks[ax] - 1) / 2;
        s *= ks[ax];
      }
      double2* kcj = kc.as<double2>() + (int64_t)j * P.M[0] * P.lines;
      if ((rc = spectrum_of(&P, gk, SPEC_COMPLEX_T, nullptr, kcj, work.as<double2>(), st))) return rc;
      a.ks[j].cplx = kcj;
      a.ks[j].ld = P.lines;
      a.out[j] = comp.as<double2>() + (int64_t)j * ce;
    }
    a.n_comp = nk;
    a.nlines = P.lines;
    a.n_valid = P.c[0];
    a.n_out = P.c[0];
    a.n_in = 1;
    a.din[0] = Tb.as<double2>();
    a.din_es = P.lines;
    a.din_item = 0;
    a.out_es = P.lines;
    a.out_item = ce;
    a.tw = tw;
    a.lmax = P.lmax;
    if ((rc = launch_col<IN_DENSE, OUT_COMPS, true>(P.L[0], a, 1, st))) return rc;
    if (D == 3) {
      LinesArgs la{};
      for (int j = 0; j < nk; ++j) la.in[j] = la.out[j] = a.out[j];
      la.nlines = (int64_t)P.c[0] * P.H;
      la.inner = P.H;
      la.outer_in = la.outer_out = (int64_t)P.M[1] * P.H;
      la.es_in = la.es_out = P.H;
      la.n_valid = P.M[1];
      la.n_out = P.c[1];
      la.scale = 1.0;
      la.tw = tw;
      la.lmax = P.lmax;
      if ((rc = launch_lines<true, false>(P.L[1], la, nk, st))) return rc;
    }
    RowArgs ra{};
    if (D == 2) { ra.rows = P.c[0]; ra.rows_a = P.c[0]; ra.stride_b = P.H; }
    else { ra.rows = (int64_t)P.c[0] * P.c[1]; ra.rows_a = P.c[1]; ra.stride_a = (int64_t)P.M[1] * P.H; ra.stride_b = P.H; }
    ra.comp_item = ce;
    ra.n_out = P.c[last];
    ra.c_phi = ra.c_grad = ra.c_hess = ra.c_sign = -1;
    ra.n_raw = nk;
    for (int j = 0; j < nk; ++j) { ra.comp[j] = a.out[j]; ra.raw[j] = d_out + (k0 + j) * P.N; }
    ra.scale = scale;
    ra.N = P.N;
    ra.tw = tw;
    ra.lmax = P.lmax;
    if ((rc = launch_row(P.L[last] - 1, ra, 1, st))) return rc;
  }
  if (host_out) CK(cudaMemcpyAsync(out, d_out, n_kernels * P.N * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));  // temporaries are freed on return
  return EIK_OK;
}

}  // extern "C"
