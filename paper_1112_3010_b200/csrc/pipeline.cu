// Host side of libeikfld_b200: plans (geometry, twiddles, cached kernel
// spectra, workspaces), the pass schedule of the 2-D / 3-D pipelines, and the
// extern "C" entry points declared in include/eikfld_b200.h.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler is attached

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
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

// classify.cu: flagged-node fill of the sign mask (R/sign.py:179-189)
int eik_fill_bits(const int64_t* d_nodes, int64_t K, int64_t N, uint32_t* bits, cudaStream_t st);
bool eik_fill_is_sparse(int dim, const int64_t* counts, int64_t K);
int eik_fill_search(int dim, const int64_t* counts, const int64_t* d_nodes, int64_t K, const uint32_t* bits,
                    int64_t* src, cudaStream_t st);
int eik_fill_apply(const int64_t* d_nodes, const int64_t* src, int64_t K, uint8_t* mask, cudaStream_t st);
int eik_fill_mask(int dim, const int64_t* counts, const int64_t* d_nodes, int64_t K, const uint32_t* bits,
                  uint8_t* mask, cudaStream_t st);
int eik_slab_fill_mask(const int64_t* counts, const int64_t* ext_nodes, int64_t K, int64_t e0, int64_t e1,
                       int64_t own0, int64_t c0_local, const uint8_t* mask_ext, uint8_t* mask_own, cudaStream_t st);

namespace {
// bumped on every device allocation of a DevBuf: a captured CUDA graph is
// replayed only while no plan buffer it references can have moved
std::atomic<uint64_t> g_alloc_epoch{0};

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
    g_alloc_epoch.fetch_add(1);
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
  int odd1 = 0;  // 3-D: odd along axis 1 (k1-mirrored lines change sign)
  double sign = 1.0;
  DevBuf buf;  // folded real/imag spectrum [(M0/2+1) x lines]
  DevBuf kp;   // register-order copy for the 2-D column kernels (KSpec::perm), or empty
  bool kp_folded = false;  // kp holds mirrored k0 once (TmCfg::PFOLD): odd-kernel sign applied at use
};

}  // namespace

struct eik_plan {
  int dim = 0, D = 0, ref0 = 0;
  int c[3] = {1, 1, 1}, M[3] = {1, 1, 1}, L[3] = {0, 0, 0};
  int64_t N = 0, H = 0, lines = 0;
  int64_t ks_l0 = 0, ks_lines = 0;  // spectral lines [ks_l0, ks_l0 + ks_lines) whose kernel spectra are stored
  int64_t ks_ls = 0;  // 3-D: line-major spectra, value (k0, l) at l * ks_ls + k0 (KSpec::ls); 0: k0 * ks_lines + l
  // 3-D: the spectra are stored folded along axis 1 (every kernel is even or odd
  // there): the plan covers k1 in [k1_begin, k1_begin + k1_count) and stores the
  // lines of the folded indices min(k1, M1 - k1) in [fold_f0, fold_f0 + ks_lines / H)
  int64_t k1_begin = 0, k1_count = 0, fold_f0 = 0;
  double h = 1.0, tau = 1.0;
  uint32_t fields = 0;
  int device = 0;
  int lmax = 2;
  DevBuf tw;
  std::vector<std::unique_ptr<KDev>> kdist;  // EXP, GRAD..., HXX, HYY, HXY (subset)
  int k_exp = -1, k_grad = -1, k_hess = -1;
  std::vector<std::unique_ptr<KDev>> ksign;
  std::vector<std::unique_ptr<KDev>> ksweep;  // tau sweep: one exp kernel per tau
  std::vector<double> taus;
  DevBuf comp, vin, rowid, cols, rowptr, srowid, scols, srowptr;
  DevBuf h_nodes, h_off, h_snodes, h_sw, stage, counter, err, work;
  std::mutex mu;
  // run generation: prep_nodes marks an invalid node list by writing the
  // current generation into err / serr, so the flags need no reset per run
  int run_gen = 0;
  cudaEvent_t ev[2 * EIK_NPASS] = {};
  bool ev_used[EIK_NPASS] = {};
  // side stream: the 2-D sign group runs concurrently with the distance group
  cudaStream_t st2 = nullptr, st_copy = nullptr, st_copy2 = nullptr, st3 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_chunk = nullptr, ev_copies = nullptr;
  cudaEvent_t ev_fill0 = nullptr, ev_fill1 = nullptr;  // side stream of the mask-fill search
  bool copies_pending = false;  // EIK_ASYNC: D2H of the last run still reads `stage`
  DevBuf serr, trows, tsign;
  DevBuf fillbits;  // flagged-node bitmap of the sign nodes (mask fill)
  DevBuf fillsrc;   // per sign node: flat index of its nearest unflagged node (split fill)
  // peer-to-peer slab exchange: own arena [P2P_NV V slots][n_comp W slots]
  // and every rank's arena base (own, same-process or IPC-opened)
  DevBuf p2p;
  int p2p_world = 0, p2p_rank = 0;
  int64_t p2p_c0loc = 0, p2p_ks = 0, p2p_slot = 0;  // complex elements per slot
  std::vector<double2*> p2p_peer;
  std::vector<void*> p2p_opened;
  // CUDA graph of a repeated device-resident eik_run (see eik_run)
  cudaStream_t st_cap = nullptr;
  cudaGraphExec_t gexec = nullptr;
  bool gkey_valid = false, seen_valid = false;
  unsigned char gkey[sizeof(eik_inputs) + sizeof(eik_outputs) + sizeof(uint32_t)] = {};
  unsigned char seen[sizeof(eik_inputs) + sizeof(eik_outputs) + sizeof(uint32_t)] = {};
  uint64_t gepoch = 0, seen_epoch = 0;
  ~eik_plan() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (st_cap) cudaStreamDestroy(st_cap);
    for (void* q : p2p_opened) cudaIpcCloseMemHandle(q);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (st2) cudaStreamDestroy(st2);
    if (ev_fill0) cudaEventDestroy(ev_fill0);
    if (ev_fill1) cudaEventDestroy(ev_fill1);
    if (st3) cudaStreamDestroy(st3);
    if (st_copy) cudaStreamDestroy(st_copy);
    if (st_copy2) cudaStreamDestroy(st_copy2);
    if (ev_chunk) cudaEventDestroy(ev_chunk);
    if (ev_copies) cudaEventDestroy(ev_copies);
  }

  // Row stride (complex elements) of the 2-D row-major intermediates T and U_j:
  // H rounded up to 8 (128 bytes), so every row starts on a cache line and the
  // column kernels' 2- / 4-line warp accesses are whole, aligned sectors (with
  // H = M/2 + 1 odd rows began 16 bytes into a sector)
  int64_t rs() const { return D == 2 ? (H + 7) & ~int64_t(7) : H; }
  int64_t comp_elems() const {  // complex elements of one component of one item
    return D == 2 ? (int64_t)c[0] * rs() : (int64_t)c[0] * M[1] * H;
  }
  int64_t held() const {
    int64_t b = fillbits.bytes + p2p.bytes + tw.bytes + comp.bytes + vin.bytes + trows.bytes + tsign.bytes + rowid.bytes + cols.bytes + rowptr.bytes + srowid.bytes +
                scols.bytes + srowptr.bytes + stage.bytes + work.bytes + h_nodes.bytes + h_off.bytes +
                h_snodes.bytes + h_sw.bytes;
    for (auto& k : kdist) b += k->buf.bytes;
    for (auto& k : ksign) b += k->buf.bytes;
    return b;
  }
};

namespace {

constexpr int NOSPLIT = 30;  // split shift meaning "no split"

ColArgs col_defaults(const eik_plan* p) {
  ColArgs a{};
  a.din_ls = 1;
  a.out_split_shift = NOSPLIT;
  a.out_split_stride = 0;
  a.tw = p->tw.as<double2>();
  a.lmax = p->lmax;
  return a;
}
LinesArgs lines_defaults(const eik_plan* p) {
  LinesArgs la{};
  la.split_shift = la.split_shift_out = NOSPLIT;
  la.split_stride = la.split_stride_out = 0;
  la.scale = 1.0;
  la.tw = p->tw.as<double2>();
  la.lmax = p->lmax;
  return la;
}

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
  p->ks_l0 = 0;
  p->ks_lines = p->lines;
  // line-major 3-D spectra where the axis-0 column kernel holds few lines per CTA (axis 0 of
  // 1024 points and more: C4@512^3 94 -> 66 ms, C4 1909 -> 914 ms); 512-point lines keep the
  // k0-major layout (8 lines per CTA: C3 3.12 ms against 3.33 ms line-major)
  p->ks_ls = (p->D == 3 && p->L[0] >= 10 && p->L[0] <= 12) ? ((int64_t)(p->M[0] / 2 + 1) + 3) / 4 * 4 : 0;
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
    LinesArgs la = lines_defaults(p);
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
  ColArgs a = col_defaults(p);
  a.nlines = p->ks_lines;
  a.n_valid = p->M[0];
  a.n_out = p->M[0];
  a.n_in = 1;
  a.din[0] = work + p->ks_l0;
  a.din_es = p->lines;
  a.din_item = 0;
  a.spec_mode = part;
  a.spec_re[0] = dst_re;
  a.out[0] = dst_c;
  a.spec_ld = p->ks_lines;
  a.spec_ls = (part == SPEC_REAL_T || part == SPEC_IMAG_T) ? p->ks_ls : 0;
  a.tw = tw;
  a.lmax = p->lmax;
  return launch_col<IN_DENSE, OUT_SPECTRUM, false>(p->L[0], a, 1, st);
}

// 3-D plans store their kernel spectra folded along axis 1: the image of the
// k1 slab under k1 -> min(k1, M1 - k1) is an interval of stored lines
void init_fold(eik_plan* p, int64_t k1_begin, int64_t k1_count) {
  p->k1_begin = k1_begin;
  p->k1_count = k1_count;
  const int64_t M1 = p->M[1], half = M1 / 2, a = k1_begin, b = k1_begin + k1_count - 1;
  auto fold = [&](int64_t k) { return k > half ? M1 - k : k; };
  int64_t lo = std::min(fold(a), fold(b)), hi = std::max(fold(a), fold(b));
  if (a <= half && half <= b) hi = half;
  p->fold_f0 = lo;
  p->ks_l0 = lo * p->H;
  p->ks_lines = (hi - lo + 1) * p->H;
}

int add_kernel(eik_plan* p, std::vector<std::unique_ptr<KDev>>& v, int ktype, int n_odd_axes, bool odd0,
               double sign, double2* work, cudaStream_t st, double tau = 0.0, bool odd1 = false) {
  auto k = std::make_unique<KDev>();
  k->ktype = ktype;
  k->imag = n_odd_axes % 2;
  k->odd0 = odd0 ? 1 : 0;
  k->odd1 = (p->D == 3 && odd1) ? 1 : 0;
  k->sign = sign;
  const int64_t n = (p->ks_ls ? p->ks_ls : (int64_t)(p->M[0] / 2 + 1)) * p->ks_lines;
  CK(k->buf.ensure(n * sizeof(double)));
  GenArgs g = gen_args(p, ktype, sign);
  if (tau > 0.0) {
    g.tau = tau;
    g.inv_tau = 1.0 / tau;
  }
  int rc = spectrum_of(p, g, k->imag ? SPEC_IMAG_T : SPEC_REAL_T, k->buf.as<double>(), nullptr, work, st);
  if (rc) return rc;
  if (p->D == 2 && p->ks_l0 == 0 && p->ks_lines == p->lines) {
    int64_t elems = 0;
    int folded = 0;
    const bool sum = &v == &p->ksign;  // the sign group runs the SUM column kernel
    if ((rc = launch_spectrum_perm(p->L[0], sum, nullptr, 0, p->ks_lines, 0, nullptr, &elems, &folded, st)))
      return rc;
    CK(k->kp.ensure(elems * sizeof(double)));
    if ((rc = launch_spectrum_perm(p->L[0], sum, k->buf.as<double>(), p->ks_lines, p->ks_lines, k->odd0,
                                   k->kp.as<double>(), &elems, &folded, st)))
      return rc;
    k->kp_folded = folded != 0;
  }
  v.push_back(std::move(k));
  return EIK_OK;
}

KSpec kspec_of(const eik_plan* p, const KDev& k) {
  KSpec s{};
  s.re = k.buf.as<double>();
  s.ld = p->ks_lines;
  s.ls = p->ks_ls;
  s.imag = k.imag;
  s.odd0 = k.odd0;
  s.odd1 = k.odd1;
  if (k.kp.bytes) {
    s.perm = k.kp.as<double>();
    s.odd0 = k.kp_folded ? k.odd0 : 0;
  }
  return s;
}

// Host-side validation of host node lists before anything is queued (so the
// asynchronous host path reports bad inputs too): item offsets start at 0,
// never decrease and end at K; nodes are strictly increasing inside [0, N)
// within each item.
int host_check_nodes(const int64_t* nodes, int64_t K, const int64_t* off, int64_t B, int64_t N_item) {
  if (off) {
    if (off[0] != 0 || off[B] != K) return fail(EIK_EVALIDATION, "item offsets must start at 0 and end at n_nodes");
    for (int64_t b = 0; b < B; ++b)
      if (off[b + 1] < off[b]) return fail(EIK_EVALIDATION, "item offsets must be non-decreasing");
  }
  for (int64_t b = 0; b < (off ? B : 1); ++b) {
    const int64_t p0 = off ? off[b] : 0, p1 = off ? off[b + 1] : K;
    for (int64_t q = p0; q < p1; ++q)
      if (nodes[q] < 0 || nodes[q] >= N_item || (q > p0 && nodes[q] <= nodes[q - 1]))
        return fail(EIK_EVALIDATION, "node indices must be sorted, distinct and inside the grid");
  }
  return EIK_OK;
}

// per-row CSR for a sorted node list (validates order and bounds): rows of
// length clast, rows_per_item rows and N_item nodes per item.
int prep_nodes(eik_plan* p, const int64_t* d_nodes, const int64_t* d_off, int64_t K, int64_t items, int64_t N_item,
               int64_t rows_per_item, int64_t clast, DevBuf& rowid, DevBuf& cols, DevBuf& rowptr, cudaStream_t st,
               DevBuf* errbuf = nullptr) {
  const int64_t nrows = rows_per_item * items;
  DevBuf& err = errbuf ? *errbuf : p->err;
  CK(rowid.ensure(std::max<int64_t>(K, 1) * sizeof(int64_t)));
  CK(cols.ensure(std::max<int64_t>(K, 1) * sizeof(int32_t)));
  const void* rp_old = rowptr.p;
  CK(rowptr.ensure((nrows + 1) * sizeof(int64_t)));
  if (rowptr.p != rp_old) CK(cudaMemsetAsync(rowptr.p, 0, rowptr.bytes, st));
  const void* err_old = err.p;
  CK(err.ensure(sizeof(int)));
  if (err.p != err_old) CK(cudaMemsetAsync(err.p, 0, sizeof(int), st));
  // node validation, row ids / columns and the row CSR in one launch
  const int64_t per = std::max<int64_t>(1, std::min<int64_t>(1024, (K / std::max<int64_t>(items, 1) + 255) / 256));
  prep_nodes_kernel<<<dim3((unsigned)per, (unsigned)items), 256, 0, st>>>(
      d_nodes, d_off, K, clast, rows_per_item, N_item, rowid.as<int64_t>(), cols.as<int32_t>(), rowptr.as<int64_t>(),
      err.as<int>(), p->run_gen);
  CK(cudaGetLastError());
  return EIK_OK;
}

}  // namespace

extern "C" {

const char* eik_last_error(void) { return g_err.c_str(); }
int eik_version(void) { return 10000; }

int eik_plan_create(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields, int device,
                    eik_plan** out) {
  return eik_plan_create_slab(dim, counts, spacing, tau, fields, device, 0, -1, out);
}

int eik_plan_create_slab(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields, int device,
                         int64_t k1_begin, int64_t k1_count, eik_plan** out) {
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
  if (k1_count >= 0) {
    if (p->D != 3) return fail(EIK_EVALIDATION, "k1 slabs apply to 3-D plans");
    if (k1_begin < 0 || k1_count < 1 || k1_begin + k1_count > p->M[1])
      return fail(EIK_EVALIDATION, "k1 slab outside the padded axis");
  }
  if (p->D == 3) init_fold(p.get(), k1_count >= 0 ? k1_begin : 0, k1_count >= 0 ? k1_count : p->M[1]);
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
        if ((rc = add_kernel(p.get(), p->kdist, KT_GRAD0 + a, 1, internal_axis == 0, 1.0, work, st, 0.0,
                             internal_axis == 1)))
          return rc;
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
        if ((rc = add_kernel(p.get(), p->ksign, KT_RAT3_0 + a, 1, a == 0, 1.0, work, st, 0.0, a == 1))) return rc;
    }
    CK(cudaDeviceSynchronize());
    p->work.release();
  }
  CK(p->counter.ensure(sizeof(unsigned long long)));
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

}  // extern "C"

// ---------------------------------------------------------------------------
// Pass building blocks shared by eik_run and the slab API.

namespace {

// Which components a run carries, in buffer order [phi, grad..., hess..., sign].
struct Roles {
  bool phi = false, hess = false, sign = false;
  int ngrad = 0;
  int n_dist() const { return phi ? 1 + ngrad + (hess ? 3 : 0) : 0; }
  int n_comp() const { return n_dist() + (sign ? 1 : 0); }
};

// NVTX range over a pass (visible in Nsight Systems / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// run_locked's profiling hook, visible to the pass functions (nullptr: not profiling)
using MarkFn = std::function<int(int, bool)>;
thread_local const MarkFn* g_mark = nullptr;
int mark_pass(int pass, bool end) { return g_mark ? (*g_mark)(pass, end) : EIK_OK; }

int set_components(const eik_plan* p, bool sign_group, const Roles& r, ColArgs& x, double2* const* W,
                   int64_t k1_offset_lines) {
  if (p->D == 3) {  // folded storage along axis 1: the kernels map pass lines to stored lines
    x.fold_H = (int)p->H;
    x.fold_M1 = p->M[1];
    x.fold_k1base = k1_offset_lines / p->H;
    x.fold_f0 = p->fold_f0;
  }
  auto ks = [&](const KDev& k) {
    KSpec s = kspec_of(p, k);
    if (p->D == 3) return s;
    s.re += k1_offset_lines - p->ks_l0;
    if (k1_offset_lines != p->ks_l0) {  // the register-order copy covers the plan's own lines only
      s.perm = nullptr;
      s.odd0 = k.odd0;
    }
    return s;
  };
  if (sign_group) {
    x.n_comp = 1;
    for (int i = 0; i < x.n_in; ++i) x.ks[i] = ks(*p->ksign[i]);
    x.out[0] = W[r.n_dist()];
    return EIK_OK;
  }
  int j = 0;
  x.ks[j] = ks(*p->kdist[p->k_exp]);
  x.out[j] = W[j];
  ++j;
  for (int d = 0; d < r.ngrad; ++d, ++j) { x.ks[j] = ks(*p->kdist[p->k_grad + d]); x.out[j] = W[j]; }
  if (r.hess)
    for (int d = 0; d < 3; ++d, ++j) { x.ks[j] = ks(*p->kdist[p->k_hess + d]); x.out[j] = W[j]; }
  x.n_comp = j;
  return EIK_OK;
}

// 2-D: fused column pass of one group straight from the node list.
// b0 / prep: item-wave mode (items [b0, b0 + B) of a batch whose node CSR was
// prepared by an earlier call with prep = true over the whole batch)
int pass_col2d(eik_plan* p, bool sg, const int64_t* nodes, const int64_t* off, int64_t K, int64_t B, const double* w,
               const Roles& r, double2* const* W, cudaStream_t st, int64_t b0 = 0, bool prep = true) {
  NvtxRange nv(sg ? "eik:col2d(sign)" : "eik:col2d(distance)");
  DevBuf& rid = sg ? p->srowid : p->rowid;
  DevBuf& cl = sg ? p->scols : p->cols;
  DevBuf& rp = sg ? p->srowptr : p->rowptr;
  if (prep) {
    int rc = prep_nodes(p, nodes, off, K, B, p->N, p->c[0], p->c[1], rid, cl, rp, st, sg ? &p->serr : nullptr);
    if (rc) return rc;
  }
  const int64_t* rowptr = rp.as<int64_t>() + b0 * p->c[0];
  const int n_in = sg ? p->dim : 1;
  // Sparse inputs (the BASELINE configs: K << N) go through the row-DFT pass
  // into a dense T[row][k1] and the dense column kernel; EIK_ROWDFT=0 keeps the
  // node-list walk inside the column kernel.
  // EIK_ROWDFT: 0 = node-list walk for both groups, 2 = for the sign group only
  static const int rowdft_env = [] {
    const char* e = std::getenv("EIK_ROWDFT");
    return e ? e[0] - '0' : 1;
  }();
  const bool rowdft = rowdft_env == 1 || (rowdft_env == 2 && !sg);
  if (rowdft && p->H <= (int64_t)ROWDFT_NF * ROWDFT_NT) {
    DevBuf& T = sg ? p->tsign : p->trows;
    const int64_t per = (int64_t)p->c[0] * p->rs();
    CK(T.ensure((size_t)n_in * B * per * sizeof(double2)));
    RowDftArgs ra{};
    ra.rowptr = rowptr;
    ra.cols = cl.as<int32_t>();
    ra.n_in = n_in;
    for (int i = 0; i < 3; ++i) {
      ra.w[i] = (sg && i < n_in) ? w + (int64_t)i * K : nullptr;
      ra.out[i] = i < n_in ? T.as<double2>() + (int64_t)i * B * per : nullptr;
    }
    ra.rows_per_item = p->c[0];
    ra.H = p->H;
    ra.out_item = per;
    // T layout: [k1][row] (transposed) where the column kernel holds one line
    // per CTA (the sign group): its warp loads are then contiguous runs of a
    // column instead of one 16-byte half sector per row
    const bool tt = (EIK_T_TRANSPOSE >> (sg ? 0 : 1)) & 1;
    ra.out_rs = tt ? 1 : p->rs();
    ra.out_ks = tt ? p->c[0] : 1;
    ra.last_shift = p->lmax - p->L[1];
    ra.last_mask = p->M[1] - 1;
    ra.tw = p->tw.as<double2>();
    CK(launch_impulse_rows(ra, n_in, p->c[0], B, st));
    ColArgs a = col_defaults(p);
    a.nlines = p->H;
    a.n_valid = p->c[0];
    a.n_out = p->c[0];
    a.n_in = n_in;
    for (int i = 0; i < n_in; ++i) a.din[i] = ra.out[i];
    a.din_es = tt ? 1 : p->rs();
    a.din_ls = tt ? p->c[0] : 1;
    a.din_item = per;
    a.out_es = p->rs();
    a.out_item = p->comp_elems();
    set_components(p, sg, r, a, W, 0);
    if (sg) return launch_col<IN_DENSE, OUT_SUM, true>(p->L[0], a, B, st);
    int rcm;
    if ((rcm = mark_pass(EIK_PASS_COL_KERNEL, false))) return rcm;
    if ((rcm = launch_col<IN_DENSE, OUT_COMPS, true>(p->L[0], a, B, st))) return rcm;
    return mark_pass(EIK_PASS_COL_KERNEL, true);
  }
  ColArgs a = col_defaults(p);
  a.rowptr = rowptr;
  a.cols = cl.as<int32_t>();
  a.n_in = sg ? p->dim : 1;
  for (int i = 0; i < 3; ++i) a.w[i] = (sg && i < a.n_in) ? w + (int64_t)i * K : nullptr;
  a.last_shift = p->lmax - p->L[1];
  a.last_mask = p->M[1] - 1;
  a.nlines = p->H;
  a.n_valid = p->c[0];
  a.n_out = p->c[0];
  a.rows_per_item = p->c[0];
  a.out_es = p->rs();
  a.out_item = p->comp_elems();
  set_components(p, sg, r, a, W, 0);
  return sg ? launch_col<IN_SPARSE, OUT_SUM, true>(p->L[0], a, B, st)
            : launch_col<IN_SPARSE, OUT_COMPS, true>(p->L[0], a, B, st);
}

// 3-D pass A: impulse DFT along axis 2 + FFT along axis 1 for planes [0, c0loc)
// of the (slab-relative) node list.  V[i] rows k1 are packed by k1-slab:
// [k1 / ks][i0][k1 % ks][k2] (ks = M1: plain [i0][k1][k2]).
// Peer-block destinations of a pass whose output is exchanged (see ColArgs::blk).
struct PeerBlk {
  double2* blk[MAXG] = {};
  int shift = 0;
  int64_t cstride = 0;
};

// in0 / nin: the sign group's inputs [in0, in0 + nin) only (streamed schedules; nin < 0: all)
int pass_planes(eik_plan* p, bool sg, const int64_t* nodes, const int64_t* off, int64_t K, int64_t B, const double* w,
                int64_t c0loc, int64_t ks, double2* const* V, cudaStream_t st, const PeerBlk* pb = nullptr,
                int in0 = 0, int nin = -1) {
  NvtxRange nv(sg ? "eik:planes(sign)" : "eik:planes(distance)");
  const int64_t H = p->H, c1 = p->c[1], c2 = p->c[2];
  DevBuf& rid = sg ? p->srowid : p->rowid;
  DevBuf& cl = sg ? p->scols : p->cols;
  DevBuf& rp = sg ? p->srowptr : p->rowptr;
  int rc = prep_nodes(p, nodes, off, K, B, c0loc * c1 * c2, c0loc * c1, c2, rid, cl, rp, st);
  if (rc) return rc;
  const int n_in = nin >= 0 ? nin : (sg ? 3 : 1);
  if (sg && w) w += (int64_t)in0 * K;
  static const bool rowdft = [] {
    const char* e = std::getenv("EIK_ROWDFT");
    return !(e && e[0] == '0');
  }();
  if (rowdft && H <= (int64_t)ROWDFT_NF * ROWDFT_NT) {
    // impulse DFT along axis 2 per row (i0, i1) into T[i0][i1][k2], then a dense
    // (half-padded) FFT along axis 1 straight into the packed V layout
    DevBuf& T = p->trows;
    const int64_t per = c0loc * c1 * H;
    CK(T.ensure((size_t)n_in * B * per * sizeof(double2)));
    RowDftArgs ra{};
    ra.rowptr = rp.as<int64_t>();
    ra.cols = cl.as<int32_t>();
    ra.n_in = n_in;
    for (int i = 0; i < 3; ++i) {
      ra.w[i] = (sg && i < n_in) ? w + (int64_t)i * K : nullptr;
      ra.out[i] = i < n_in ? T.as<double2>() + (int64_t)i * B * per : nullptr;
    }
    ra.rows_per_item = c0loc * c1;
    ra.H = H;
    ra.out_item = per;
    ra.last_shift = p->lmax - p->L[2];
    ra.last_mask = p->M[2] - 1;
    ra.tw = p->tw.as<double2>();
    CK(launch_impulse_rows(ra, n_in, c0loc * c1, B, st));
    LinesArgs la = lines_defaults(p);
    for (int i = 0; i < n_in; ++i) { la.in[i] = ra.out[i]; la.out[i] = V[i]; }
    la.nlines = B * c0loc * H;
    la.inner = H;
    la.outer_in = c1 * H;
    la.outer_out = ks * H;
    la.es_in = la.es_out = H;
    if (ks < p->M[1]) {
      la.split_shift_out = ilog2_exact(ks);
      la.split_stride_out = c0loc * ks * H;
    }
    la.n_valid = (int)c1;
    la.n_out = p->M[1];
    if (pb) {
      for (int g = 0; g < MAXG; ++g) la.blk[g] = pb->blk[g];
      la.blk_cstride = pb->cstride;
    }
    return launch_lines<false, true>(p->L[1], la, n_in, st);
  }
  if (pb) return fail(EIK_EVALIDATION, "the peer-to-peer slab exchange needs the row-DFT planes pass");
  ColArgs a = col_defaults(p);
  a.rowptr = rp.as<int64_t>();
  a.cols = cl.as<int32_t>();
  a.n_in = n_in;
  for (int i = 0; i < 3; ++i) a.w[i] = (sg && i < a.n_in) ? w + (int64_t)i * K : nullptr;
  a.last_shift = p->lmax - p->L[2];
  a.last_mask = p->M[2] - 1;
  a.nlines = H;
  a.n_valid = (int)c1;
  a.rows_per_item = c1;
  a.spec_mode = SPEC_COMPLEX;
  a.out_es = H;
  a.out_item = ks * H;
  if (ks < p->M[1]) {
    a.out_split_shift = ilog2_exact(ks);
    a.out_split_stride = c0loc * ks * H;
  }
  for (int i = 0; i < a.n_in; ++i) a.out[i] = V[i];
  return launch_col<IN_SPARSE, OUT_SPECTRUM, true>(p->L[1], a, B * c0loc, st);
}

// 3-D pass B: fused axis-0 pass for k1 in [k1b, k1b + ks) over spectra
// V[i][i0 < c0][k1'][k2]; writes W_j[n < c0][k1'][k2].
int pass_axis0(eik_plan* p, bool sg, double2* const* V, int64_t k1b, int64_t ks, int64_t B, const Roles& r,
               double2* const* W, cudaStream_t st, const PeerBlk* pb = nullptr) {
  NvtxRange nv(sg ? "eik:axis0(sign)" : "eik:axis0(distance)");
  const int64_t H = p->H;
  if (k1b < p->k1_begin || k1b + ks > p->k1_begin + p->k1_count)
    return fail(EIK_EVALIDATION, "k1 slab not covered by the plan's kernel spectra");
  ColArgs a = col_defaults(p);
  a.nlines = ks * H;
  a.n_valid = p->c[0];
  a.n_out = p->c[0];
  a.n_in = sg ? 3 : 1;
  for (int i = 0; i < a.n_in; ++i) a.din[i] = V[i];
  a.din_es = ks * H;
  a.din_item = (int64_t)p->c[0] * ks * H;
  a.out_es = ks * H;
  a.out_item = (int64_t)p->c[0] * ks * H;
  set_components(p, sg, r, a, W, k1b * H);
  if (pb) {
    for (int g = 0; g < MAXG; ++g) a.blk[g] = pb->blk[g];
    a.blk_shift = pb->shift;
    a.blk_cstride = pb->cstride;
  }
  if (sg) return launch_col<IN_DENSE, OUT_SUM, true>(p->L[0], a, B, st);
  int rcm;
  if ((rcm = mark_pass(EIK_PASS_COL_KERNEL, false))) return rcm;
  if ((rcm = launch_col<IN_DENSE, OUT_COMPS, true>(p->L[0], a, B, st))) return rcm;
  return mark_pass(EIK_PASS_COL_KERNEL, true);
}

// 3-D pass C (or the 2-D row pass): inverse along axis 1 (3-D only) + c2r along
// the last axis + epilogue, for planes [0, c0loc).  W_j laid out as
// [k1 / ks][i0][k1 % ks][k2] (3-D) or [row][k1] (2-D).
// on_chunk(row0, row1, item0, item1), when given, splits the row pass into
// chunks and is called after each chunk is queued (host copies overlap the
// remaining chunks).
using ChunkFn = std::function<int(int64_t, int64_t, int64_t, int64_t)>;
struct RawOut {
  int n = 0;
  double* dest[MAXC] = {};
  double tau[MAXC] = {};
};

int pass_finish(eik_plan* p, double2* const* W, const Roles& r, int64_t c0loc, int64_t ks, int64_t B,
                RowArgs ra, cudaStream_t st, const std::function<int(int, bool)>& mark,
                const ChunkFn& on_chunk = nullptr, const RawOut* raw = nullptr) {
  NvtxRange nv("eik:finish(lines+row)");
  const int64_t H = p->H;
  // raw: W[0..n) are written as scaled real-space convolutions (tau > 0: -tau log), no epilogue
  const int nc = raw ? raw->n : r.n_comp();
  int rc;
  if (p->D == 3) {
    LinesArgs la = lines_defaults(p);
    for (int j = 0; j < nc; ++j) { la.in[j] = W[j]; la.out[j] = W[j]; }
    la.nlines = B * c0loc * H;
    la.inner = H;
    la.outer_in = la.outer_out = ks * H;
    la.es_in = la.es_out = H;
    if (ks < p->M[1]) {
      la.split_shift = la.split_shift_out = ilog2_exact(ks);
      la.split_stride = la.split_stride_out = c0loc * ks * H;
    }
    la.n_valid = p->M[1];
    la.n_out = p->c[1];
    if ((rc = mark(EIK_PASS_LINES, false))) return rc;
    if ((rc = launch_lines<true, false>(p->L[1], la, nc, st))) return rc;
    if ((rc = mark(EIK_PASS_LINES, true))) return rc;
    ra.rows = c0loc * p->c[1];
    ra.rows_a = p->c[1];
    ra.stride_a = ks * H;
    ra.stride_b = H;
    ra.split_shift = ks < p->M[1] ? ilog2_exact(ks) : NOSPLIT;
    ra.split_stride = ks < p->M[1] ? c0loc * ks * H : 0;
    ra.comp_item = c0loc * p->M[1] * H;
    ra.N = c0loc * p->c[1] * p->c[2];
  } else {
    ra.rows = p->c[0];
    ra.rows_a = p->c[0];
    ra.stride_a = 0;
    ra.stride_b = p->rs();
    ra.split_shift = NOSPLIT;
    ra.split_stride = 0;
    ra.comp_item = p->comp_elems();
    ra.N = p->N;
  }
  for (int j = 0; j < nc; ++j) ra.comp[j] = W[j];
  ra.n_comp = nc;
  ra.n_out = p->c[p->D - 1];
  ra.c_phi = r.phi ? 0 : -1;
  ra.c_grad = r.ngrad ? 1 : -1;
  ra.ngrad = r.ngrad;
  ra.c_hess = r.hess ? 1 + r.ngrad : -1;
  ra.c_sign = r.sign ? r.n_dist() : -1;
  if (raw) {
    ra.c_phi = ra.c_grad = ra.c_hess = ra.c_sign = -1;
    ra.ngrad = 0;
    ra.n_raw = raw->n;
    for (int j = 0; j < raw->n; ++j) {
      ra.raw[j] = raw->dest[j];
      ra.raw_tau[j] = raw->tau[j];
    }
  }
  ra.sign_mode = p->dim == 2 ? 1 : 2;
  double scale = 1.0;
  for (int a = 0; a < p->D; ++a) scale /= (double)p->M[a];
  ra.scale = scale;
  ra.tau = p->tau;
  ra.inv_tau = 1.0 / p->tau;
  ra.tw = p->tw.as<double2>();
  ra.lmax = p->lmax;
  if ((rc = mark(EIK_PASS_ROW, false))) return rc;
  const int LH = p->L[p->D - 1] - 1;
  if (!on_chunk) {
    ra.row0 = 0;
    ra.row_end = ra.rows;
    ra.item0 = 0;
    if ((rc = launch_row(LH, ra, B, st))) return rc;
    return mark(EIK_PASS_ROW, true);
  }
  constexpr int kChunks = 8;
  if (B >= kChunks) {  // chunk over items
    for (int c = 0; c < kChunks; ++c) {
      const int64_t i0 = B * c / kChunks, i1 = B * (c + 1) / kChunks;
      if (i1 <= i0) continue;
      ra.row0 = 0;
      ra.row_end = ra.rows;
      ra.item0 = i0;
      if ((rc = launch_row(LH, ra, i1 - i0, st))) return rc;
      if ((rc = on_chunk(0, ra.rows, i0, i1))) return rc;
    }
  } else {  // chunk over rows (every item)
    for (int c = 0; c < kChunks; ++c) {
      const int64_t r0 = ra.rows * c / kChunks, r1 = ra.rows * (c + 1) / kChunks;
      if (r1 <= r0) continue;
      ra.row0 = r0;
      ra.row_end = r1;
      ra.item0 = 0;
      if ((rc = launch_row(LH, ra, B, st))) return rc;
      if ((rc = on_chunk(r0, r1, 0, B))) return rc;
    }
  }
  return mark(EIK_PASS_ROW, true);
}


// ---------------------------------------------------------------------------
// Streamed 3-D schedule (one GPU, grids whose fused buffers exceed the device:
// C4 at 1024^3).  One spectrum slot V and one component slot W are live at a
// time: each distance component runs its own axis-0 pass (the forward transform
// of V is repeated per component), is brought back to real space unscaled by
// the row kernel's raw mode, and a last elementwise pass applies the epilogue
// (the same double operations as the fused row epilogue).  The sign group
// accumulates W += IFFT0(K_i FFT0(V_i)) over its three flux inputs.  The
// impulse DFT's T is written inside V (first c1 entries of every axis-1 line)
// and transformed in place.

// impulse DFT along axis 2 + in-place FFT along axis 1 of ONE input -> V[i0][k1][k2]
int pass_planes_inplace(eik_plan* p, bool sg, const int64_t* nodes, int64_t K, const double* w, double2* V,
                        cudaStream_t st) {
  const int64_t H = p->H, c0 = p->c[0], c1 = p->c[1], c2 = p->c[2], M1 = p->M[1];
  if (H > (int64_t)ROWDFT_NF * ROWDFT_NT) return fail(EIK_EVALIDATION, "last axis too long for the row DFT");
  if (c0 > 65535) return fail(EIK_EVALIDATION, "axis 0 too long for the streamed planes pass");
  DevBuf& rid = sg ? p->srowid : p->rowid;
  DevBuf& cl = sg ? p->scols : p->cols;
  DevBuf& rp = sg ? p->srowptr : p->rowptr;
  int rc = prep_nodes(p, nodes, nullptr, K, 1, c0 * c1 * c2, c0 * c1, c2, rid, cl, rp, st);
  if (rc) return rc;
  RowDftArgs ra{};
  ra.rowptr = rp.as<int64_t>();
  ra.cols = cl.as<int32_t>();
  ra.n_in = 1;
  ra.w[0] = w;
  ra.out[0] = V;
  ra.rows_per_item = c1;  // "items" are the planes i0: row (i0, i1) lands at V[i0][i1][.]
  ra.H = H;
  ra.out_item = M1 * H;
  ra.last_shift = p->lmax - p->L[2];
  ra.last_mask = p->M[2] - 1;
  ra.tw = p->tw.as<double2>();
  CK(launch_impulse_rows(ra, 1, c1, c0, st));
  LinesArgs la = lines_defaults(p);
  la.in[0] = V;
  la.out[0] = V;
  la.nlines = c0 * H;
  la.inner = H;
  la.outer_in = la.outer_out = M1 * H;
  la.es_in = la.es_out = H;
  la.n_valid = (int)c1;
  la.n_out = (int)M1;
  return launch_lines<false, true>(p->L[1], la, 1, st);
}

// axis-0 pass of a list of kernels: W_j (+)= IFFT0(K_j FFT0(V)), rows [0, c0)
int pass_axis0_list(eik_plan* p, const double2* V, const KDev* const* ks, int n, double2* const* W, bool accum,
                    cudaStream_t st, int64_t k1b = 0, int64_t kslab = -1) {
  const int64_t H = p->H, M1 = p->M[1];
  const int64_t kk = kslab < 0 ? M1 : kslab;  // lines of the k1 slab [k1b, k1b + kk)
  if (k1b < p->k1_begin || k1b + kk > p->k1_begin + p->k1_count)
    return fail(EIK_EVALIDATION, "k1 slab not covered by the plan's kernel spectra");
  ColArgs a = col_defaults(p);
  a.nlines = kk * H;
  a.n_valid = p->c[0];
  a.n_out = p->c[0];
  a.n_in = 1;
  a.din[0] = V;
  a.din_es = kk * H;
  a.din_item = (int64_t)p->c[0] * kk * H;
  a.out_es = kk * H;
  a.out_item = (int64_t)p->c[0] * kk * H;
  a.fold_H = (int)H;
  a.fold_M1 = (int)M1;
  a.fold_k1base = k1b;
  a.fold_f0 = p->fold_f0;
  for (int j = 0; j < n; ++j) {
    a.ks[j] = kspec_of(p, *ks[j]);
    a.out[j] = W[j];
  }
  a.n_comp = n;
  a.accum = accum ? 1 : 0;
  return launch_col<IN_DENSE, OUT_COMPS, true>(p->L[0], a, 1, st);
}
int pass_axis0_single(eik_plan* p, const double2* V, const KDev& k, double2* W, bool accum, cudaStream_t st) {
  const KDev* kk = &k;
  return pass_axis0_list(p, V, &kk, 1, &W, accum, st);
}

struct StreamEpi {
  int64_t N;
  double* phi_raw;   // scaled phi (may alias S or phi_out)
  double* S;
  double* phi_out;
  uint8_t* uf;
  unsigned long long* uf_count;
  double* grad[3];   // in: scaled numerators, out: ratios (in place)
  double* mu_raw;    // scaled sign convolution (may alias mu)
  double* mu;
  uint8_t* mask;
  double tau;
};

// Elementwise epilogue of the streamed schedule: the operations of row_kernel's
// fused epilogue (3-D: no Hessian, ratios by division) on the raw fields.
// every double field 16-byte aligned (null fields count as aligned): the vector path applies
inline int stream_epi_vec2(const StreamEpi& e) {
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return al16(e.phi_raw) && al16(e.S) && al16(e.phi_out) && al16(e.grad[0]) && al16(e.grad[1]) && al16(e.grad[2]) &&
         al16(e.mu_raw) && al16(e.mu);
}
// One element of the streamed epilogue (same double operations as the fused row epilogue).
__device__ __forceinline__ void stream_epi_dist(const StreamEpi& e, double phi, double (&g)[3], double& S, unsigned& cnt) {
  cnt += (phi <= 0.0);
  for (int d = 0; d < 3; ++d)
    if (e.grad[d]) g[d] = g[d] / phi;
  S = phi > 0.0 ? (-e.tau) * log(phi) : __longlong_as_double(0x7ff8000000000000LL);
}
// Two elements per thread and iteration through 16-byte loads / stores when every field is
// 16-byte aligned (C4 1024^3: 23.3 ms of scalar accesses at 57% of the HBM peak before)
__global__ void stream_epilogue_kernel(const StreamEpi e, int vec2) {
  unsigned cnt = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t npair = vec2 ? e.N / 2 : 0;
  for (int64_t q = tid0; q < npair; q += stride) {
    const int64_t i = 2 * q;
    if (e.phi_raw) {
      const double2 phi = *reinterpret_cast<const double2*>(e.phi_raw + i);
      double2 gv[3];
      for (int d = 0; d < 3; ++d)
        if (e.grad[d]) gv[d] = *reinterpret_cast<const double2*>(e.grad[d] + i);
      double g0[3] = {gv[0].x, gv[1].x, gv[2].x}, g1[3] = {gv[0].y, gv[1].y, gv[2].y};
      double S0, S1;
      stream_epi_dist(e, phi.x, g0, S0, cnt);
      stream_epi_dist(e, phi.y, g1, S1, cnt);
      for (int d = 0; d < 3; ++d)
        if (e.grad[d]) *reinterpret_cast<double2*>(e.grad[d] + i) = make_double2(g0[d], g1[d]);
      if (e.phi_out && e.phi_out != e.phi_raw) *reinterpret_cast<double2*>(e.phi_out + i) = phi;
      if (e.uf) {
        e.uf[i] = phi.x <= 0.0;
        e.uf[i + 1] = phi.y <= 0.0;
      }
      if (e.S) *reinterpret_cast<double2*>(e.S + i) = make_double2(S0, S1);
    }
    if (e.mu_raw) {
      const double2 mr = *reinterpret_cast<const double2*>(e.mu_raw + i);
      const double m0 = -mr.x / 12.566370614359172, m1 = -mr.y / 12.566370614359172;
      if (e.mu) *reinterpret_cast<double2*>(e.mu + i) = make_double2(m0, m1);
      if (e.mask) {
        e.mask[i] = rint(m0) >= 1.0;
        e.mask[i + 1] = rint(m1) >= 1.0;
      }
    }
  }
  for (int64_t i = 2 * npair + tid0; i < e.N; i += stride) {
    if (e.phi_raw) {
      const double phi = e.phi_raw[i];
      double g[3] = {0.0, 0.0, 0.0}, S;
      for (int d = 0; d < 3; ++d)
        if (e.grad[d]) g[d] = e.grad[d][i];
      stream_epi_dist(e, phi, g, S, cnt);
      for (int d = 0; d < 3; ++d)
        if (e.grad[d]) e.grad[d][i] = g[d];
      if (e.phi_out && e.phi_out != e.phi_raw) e.phi_out[i] = phi;
      if (e.uf) e.uf[i] = phi <= 0.0;
      if (e.S) e.S[i] = S;
    }
    if (e.mu_raw) {
      const double m = -e.mu_raw[i] / 12.566370614359172;
      if (e.mu) e.mu[i] = m;
      if (e.mask) e.mask[i] = rint(m) >= 1.0;
    }
  }
  if (e.uf_count) {
    const unsigned tot = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(e.uf_count, (unsigned long long)tot);
  }
}

}  // namespace

extern "C" {

static int run_locked(eik_plan* p, const eik_inputs* in, const eik_outputs* out, uint32_t flags, void* stream);

// Device-resident asynchronous runs (no host buffers, no sync, no profiling)
// repeated with identical arguments are replayed as one CUDA graph: the
// second identical call is captured on the plan's private stream (the caller's
// may be the legacy default stream, which cannot be captured) and every later
// one is a single cudaGraphLaunch into the caller's stream.  Any plan-buffer
// allocation in between (g_alloc_epoch) or an argument change re-runs eagerly.
// EIK_GRAPH=0 turns this off.
int eik_run(eik_plan* p, const eik_inputs* in, const eik_outputs* out, uint32_t flags, void* stream) {
  if (!p || !in || !out) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  static const bool graphs = [] {
    const char* e = std::getenv("EIK_GRAPH");
    return !(e && e[0] == '0');
  }();
  // a caller that is itself capturing (torch.cuda.graph, cudaStreamBeginCapture)
  // records the eager launches into its own graph; the dense mask fill
  // (sign nodes > N/8) allocates temporaries and is never captured
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cap) != cudaSuccess) {
    cudaGetLastError();  // e.g. the legacy stream during another stream's global-mode capture
    cap = cudaStreamCaptureStatusActive;
  }
  const bool dense_fill = out->mask && in->n_sign_nodes > p->N / 8;
  const bool graphable = graphs && cap == cudaStreamCaptureStatusNone && !dense_fill &&
                         !(flags & (EIK_HOST_INPUTS | EIK_HOST_OUTPUTS | EIK_SYNC | EIK_CHECK_UNDERFLOW |
                                    EIK_PROFILE | EIK_SLAB_P2P)) &&
                         !out->n_underflow && !p->copies_pending;
  if (!graphable) return run_locked(p, in, out, flags, stream);
  unsigned char key[sizeof(p->gkey)];
  std::memcpy(key, in, sizeof(eik_inputs));
  std::memcpy(key + sizeof(eik_inputs), out, sizeof(eik_outputs));
  std::memcpy(key + sizeof(eik_inputs) + sizeof(eik_outputs), &flags, sizeof(flags));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t epoch = g_alloc_epoch.load();
  if (p->gexec && p->gkey_valid && p->gepoch == epoch && !std::memcmp(key, p->gkey, sizeof(key))) {
    for (bool& u : p->ev_used) u = false;  // no pass times for this run (as for any unprofiled run)
    CK(cudaGraphLaunch(p->gexec, st));
    return EIK_OK;
  }
  if (!(p->seen_valid && p->seen_epoch == epoch && !std::memcmp(key, p->seen, sizeof(key)))) {
    std::memcpy(p->seen, key, sizeof(key));
    p->seen_valid = true;
    const int rc = run_locked(p, in, out, flags, stream);
    p->seen_epoch = g_alloc_epoch.load();
    return rc;
  }
  // second identical call: capture it
  if (!p->st_cap) CK(cudaStreamCreateWithFlags(&p->st_cap, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(p->st_cap, cudaStreamCaptureModeRelaxed));
  const int rc = run_locked(p, in, out, flags, p->st_cap);
  const cudaError_t ce = cudaStreamEndCapture(p->st_cap, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CK(ce);
  if (p->gexec) {
    cudaGraphExecDestroy(p->gexec);
    p->gexec = nullptr;
  }
  const cudaError_t ie = cudaGraphInstantiate(&p->gexec, g, 0);
  cudaGraphDestroy(g);
  CK(ie);
  std::memcpy(p->gkey, key, sizeof(key));
  p->gkey_valid = true;
  p->gepoch = g_alloc_epoch.load();
  CK(cudaGraphLaunch(p->gexec, st));
  return EIK_OK;
}

static int run_locked(eik_plan* p, const eik_inputs* in, const eik_outputs* out, uint32_t flags, void* stream) {
  NvtxRange nv("eik_run");
  p->run_gen = p->run_gen == INT_MAX ? 1 : p->run_gen + 1;
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

  const bool prof = flags & EIK_PROFILE;
  for (bool& u : p->ev_used) u = false;
  std::function<int(int, bool)> mark = [&](int pass, bool end) -> int {
    if (!prof) return EIK_OK;
    cudaEvent_t& e = p->ev[2 * pass + (end ? 1 : 0)];
    if (!e) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, st));
    if (end) p->ev_used[pass] = true;
    return EIK_OK;
  };
  struct MarkScope {  // the pass functions reach `mark` through g_mark while this run is on the stack
    explicit MarkScope(const MarkFn* m) { g_mark = m; }
    ~MarkScope() { g_mark = nullptr; }
  } mark_scope(prof ? &mark : nullptr);
  // ---- inputs
  const int64_t* d_nodes = in->nodes;
  const int64_t* d_off = in->item_offsets;
  const int64_t* d_snodes = in->sign_nodes;
  const double* d_sw = in->sign_weights;
  const int64_t Ks = in->n_sign_nodes;
  if (B > 65535) return fail(EIK_EVALIDATION, "batch larger than 65535 items");
  if (host_in) {
    int rc0;
    if (want_phi && (rc0 = host_check_nodes(in->nodes, in->n_nodes, B > 1 ? in->item_offsets : nullptr, B, p->N)))
      return rc0;
    if (want_sign && (rc0 = host_check_nodes(in->sign_nodes, Ks, nullptr, 1, p->N))) return rc0;
  }
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
  // one item: prep_nodes takes [0, n_nodes) without an offsets array (no
  // pageable 16-byte upload on the stream)
  if (want_phi && B == 1 && (!d_off || host_in)) d_off = nullptr;
  if (want_sign) {
    if (host_in) {
      CK(p->h_snodes.ensure(Ks * sizeof(int64_t)));
      CK(p->h_sw.ensure(Ks * p->dim * sizeof(double)));
      CK(cudaMemcpyAsync(p->h_snodes.p, in->sign_nodes, Ks * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(p->h_sw.p, in->sign_weights, Ks * p->dim * sizeof(double), cudaMemcpyHostToDevice, st));
      d_snodes = p->h_snodes.as<int64_t>();
      d_sw = p->h_sw.as<double>();
    }
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
  Roles r;
  r.phi = want_phi;
  r.ngrad = want_phi && (want_grad || want_hess) ? p->dim : 0;
  r.hess = want_phi && want_hess;
  r.sign = want_sign;
  const int n_comp = r.n_comp();
  const int64_t ce = p->comp_elems();
  // sign mask: every node classified by its own mu in the row epilogue, then
  // the flagged (sign) nodes take their nearest unflagged node's class with
  // scipy's EDT ties, as classify does (R/sign.py:179-195)
  const bool want_fill = want_sign && out->mask;
  const int64_t fill_counts[3] = {p->dim == 1 ? p->c[1] : p->c[0], p->c[1], p->c[2]};
  if (want_fill) CK(p->fillbits.ensure(((p->N + 31) / 32) * sizeof(uint32_t)));
  uint32_t* fbits = p->fillbits.as<uint32_t>();
  // sparse flagged sets: the nearest-unflagged-node search needs the bitmap only, so it is
  // queued right behind it (next to the column passes); after the row pass one gather is left
  // (C2: the 19 us search kernel leaves the tail of the step).  EIK_FILL_SPLIT=0: search at the end.
  static const bool fill_split_on = [] {
    const char* e = std::getenv("EIK_FILL_SPLIT");
    return !(e && e[0] == '0');
  }();
  const bool fill_split = want_fill && fill_split_on && eik_fill_is_sparse(p->dim, fill_counts, Ks);
  if (fill_split) CK(p->fillsrc.ensure((size_t)Ks * sizeof(int64_t)));
  // side = true (2-D, the groups forked onto two streams): bitmap and search run on a third
  // stream, off both groups' chains (inside a group's stream the search only moves from the
  // step's tail to its head: measured 0.803 -> 0.810 ms), joined before the apply
  bool fill_side_pending = false;
  auto fill_prepare = [&](cudaStream_t s2, bool side = false) -> int {
    cudaStream_t sf = s2;
    if (side && fill_split) {
      if (!p->st3) CK(cudaStreamCreateWithFlags(&p->st3, cudaStreamNonBlocking));
      if (!p->ev_fill0) CK(cudaEventCreateWithFlags(&p->ev_fill0, cudaEventDisableTiming));
      if (!p->ev_fill1) CK(cudaEventCreateWithFlags(&p->ev_fill1, cudaEventDisableTiming));
      CK(cudaEventRecord(p->ev_fill0, s2));
      CK(cudaStreamWaitEvent(p->st3, p->ev_fill0, 0));
      sf = p->st3;
    }
    int rcf = eik_fill_bits(d_snodes, Ks, p->N, fbits, sf);
    if (rcf || !fill_split) return rcf;
    if ((rcf = eik_fill_search(p->dim, fill_counts, d_snodes, Ks, fbits, p->fillsrc.as<int64_t>(), sf))) return rcf;
    if (sf != s2) {
      CK(cudaEventRecord(p->ev_fill1, sf));
      fill_side_pending = true;
    }
    return EIK_OK;
  };
  auto fill_finish = [&](cudaStream_t s2) -> int {
    if (fill_side_pending) {
      CK(cudaStreamWaitEvent(s2, p->ev_fill1, 0));
      fill_side_pending = false;
    }
    if (fill_split) return eik_fill_apply(d_snodes, p->fillsrc.as<int64_t>(), Ks, o_mask, s2);
    return eik_fill_mask(p->dim, fill_counts, d_snodes, Ks, fbits, o_mask, s2);
  };
  // EIK_WAVE=n (2-D distance batches on the row-DFT path): items run in waves
  // of n, column pass then row pass per wave, so the wave's T and U_j stay in
  // L2 between the passes instead of round-tripping HBM
  static const int64_t wave_env = [] {
    const char* e = std::getenv("EIK_WAVE");
    return e ? std::atoll(e) : 0;
  }();
  static const int rowdft_on = [] {
    const char* e = std::getenv("EIK_ROWDFT");
    return e ? e[0] - '0' : 1;
  }();
  const bool waves = p->D == 2 && want_phi && !want_sign && wave_env > 0 && B > wave_env && rowdft_on == 1 &&
                     p->H <= (int64_t)ROWDFT_NF * ROWDFT_NT;
  const int64_t BW = waves ? wave_env : B;
  // 3-D, one item: the streamed schedule (one V and one W slot, see
  // pass_planes_inplace) when the fused buffers do not fit the device;
  // EIK_STREAM3D=1 forces it, =0 forbids it
  bool streamed = false;
  if (p->D == 3 && B == 1 && !(flags & EIK_SLAB_P2P)) {
    const char* e = std::getenv("EIK_STREAM3D");
    if (e && (e[0] == '0' || e[0] == '1')) {
      streamed = e[0] == '1';
    } else {
      const int n_in_max = std::max(want_phi ? 1 : 0, want_sign ? 3 : 0);
      const size_t need = (size_t)(n_in_max + n_comp) * ce * sizeof(double2) +
                          (size_t)n_in_max * p->c[0] * p->c[1] * p->H * sizeof(double2);
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      const size_t avail = fr + p->vin.bytes + p->comp.bytes + p->trows.bytes;
      streamed = need + (size_t(1) << 30) > avail;
    }
  }
  if (streamed) {
    p->trows.release();
    CK(p->vin.ensure((size_t)ce * sizeof(double2)));
  }
  CK(p->comp.ensure((size_t)(streamed ? 1 : n_comp * BW) * ce * sizeof(double2)));
  std::vector<double2*> W(n_comp);
  for (int j = 0; j < n_comp; ++j) W[j] = p->comp.as<double2>() + (streamed ? 0 : (int64_t)j * BW * ce);
  int rc;
  if (waves) {
    // node CSR over the whole batch once; the waves index into it
    if ((rc = prep_nodes(p, d_nodes, d_off, in->n_nodes, B, p->N, p->c[0], p->c[1], p->rowid, p->cols, p->rowptr,
                         st)))
      return rc;
  } else if (p->D == 2) {
    // The two groups are independent column passes: run the sign group on a
    // side stream so it fills the distance group's tail (sequential when
    // profiling, so that per-pass times stay attributable).
    const bool fork = want_phi && want_sign && !prof;
    cudaStream_t ss = st;
    if (fork) {
      if (!p->st2) CK(cudaStreamCreateWithFlags(&p->st2, cudaStreamNonBlocking));
      if (!p->ev_fork) CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
      if (!p->ev_join) CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
      CK(cudaEventRecord(p->ev_fork, st));
      CK(cudaStreamWaitEvent(p->st2, p->ev_fork, 0));
      ss = p->st2;
    }
    // the distance group is queued ahead of the sign group (C2 -0.6%);
    // EIK_SIGN_FIRST=1 restores the opposite order
    static const bool sign_first = [] {
      const char* e = std::getenv("EIK_SIGN_FIRST");
      return e && e[0] == '1';
    }();
    auto sign_group = [&]() -> int {
      if (!want_sign) return EIK_OK;
      int rc2;
      if ((rc2 = mark(EIK_PASS_COL_SIGN, false))) return rc2;
      if (want_fill && (rc2 = fill_prepare(ss, fork))) return rc2;
      if ((rc2 = pass_col2d(p, true, d_snodes, nullptr, Ks, 1, d_sw, r, W.data(), ss))) return rc2;
      if ((rc2 = mark(EIK_PASS_COL_SIGN, true))) return rc2;
      if (fork) CK(cudaEventRecord(p->ev_join, ss));
      return EIK_OK;
    };
    auto dist_group = [&]() -> int {
      if (!want_phi) return EIK_OK;
      int rc2;
      if ((rc2 = mark(EIK_PASS_COL, false))) return rc2;
      if ((rc2 = pass_col2d(p, false, d_nodes, d_off, in->n_nodes, B, nullptr, r, W.data(), st))) return rc2;
      return mark(EIK_PASS_COL, true);
    };
    if ((rc = sign_first ? sign_group() : dist_group())) return rc;
    if ((rc = sign_first ? dist_group() : sign_group())) return rc;
    if (fork) CK(cudaStreamWaitEvent(st, p->ev_join, 0));
  } else if (!streamed) {
    const int n_in_max = std::max(want_phi ? 1 : 0, want_sign ? 3 : 0);
    CK(p->vin.ensure((size_t)n_in_max * B * ce * sizeof(double2)));
    double2* V[3];
    for (int i = 0; i < 3; ++i) V[i] = p->vin.as<double2>() + (int64_t)i * B * ce;
    if (want_phi) {
      if ((rc = mark(EIK_PASS_COL, false))) return rc;
      if ((rc = pass_planes(p, false, d_nodes, d_off, in->n_nodes, B, nullptr, p->c[0], p->M[1], V, st))) return rc;
      if ((rc = pass_axis0(p, false, V, 0, p->M[1], B, r, W.data(), st))) return rc;
      if ((rc = mark(EIK_PASS_COL, true))) return rc;
    }
    if (want_sign) {
      if ((rc = mark(EIK_PASS_COL_SIGN, false))) return rc;
      if (want_fill && (rc = fill_prepare(st))) return rc;
      if ((rc = pass_planes(p, true, d_snodes, nullptr, Ks, 1, d_sw, p->c[0], p->M[1], V, st)))
        return rc;
      if ((rc = pass_axis0(p, true, V, 0, p->M[1], 1, r, W.data(), st))) return rc;
      if ((rc = mark(EIK_PASS_COL_SIGN, true))) return rc;
    }
  }
  // ---- last axis c2r + epilogue
  RowArgs ra{};
  ra.S = o_S;
  for (int d = 0; d < 3; ++d) { ra.grad[d] = o_g[d]; ra.hess[d] = o_h[d]; }
  ra.mu = o_mu;
  ra.mask = o_mask;
  ra.uf = o_uf;
  ra.phi_out = o_phi;
  const bool count = want_phi && (out->n_underflow || out->d_underflow_count || (flags & EIK_CHECK_UNDERFLOW));
  unsigned long long* ctr = out->d_underflow_count ? out->d_underflow_count : p->counter.as<unsigned long long>();
  if (count) {
    if (!out->d_underflow_count) CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    ra.uf_count = ctr;
  }
  // EIK_ASYNC (host outputs): return without synchronising; the next run's
  // column passes overlap this run's D2H, its row pass waits for it (stage reuse)
  const bool async = (flags & EIK_ASYNC) && host_out && !(flags & (EIK_SYNC | EIK_CHECK_UNDERFLOW)) &&
                     !out->n_underflow;
  if (p->copies_pending) {
    CK(cudaStreamWaitEvent(st, p->ev_copies, 0));
    p->copies_pending = false;
  }
  // streamed 3-D schedule: every component through the one V / W pair, then the elementwise epilogue
  auto run_streamed = [&]() -> int {
    int rc2;
    double2* V1 = p->vin.as<double2>();
    double2* W1 = p->comp.as<double2>();
    std::function<int(int, bool)> nomark = [](int, bool) { return EIK_OK; };
    // scratch for raw fields whose output was not requested
    const bool need_phi_scratch = want_phi && !o_S && !o_phi;
    const bool need_mu_scratch = want_sign && !o_mu;
    if (need_phi_scratch || need_mu_scratch) CK(p->work.ensure((size_t)2 * p->N * sizeof(double)));
    StreamEpi e{};
    e.N = p->N;
    e.tau = p->tau;
    RowArgs rr = ra;  // scale etc. are filled by pass_finish; outputs unused in raw mode
    rr.S = nullptr; rr.mu = nullptr; rr.mask = nullptr; rr.uf = nullptr; rr.phi_out = nullptr; rr.uf_count = nullptr;
    for (int d = 0; d < 3; ++d) rr.grad[d] = rr.hess[d] = nullptr;
    if (want_phi) {
      if ((rc2 = mark(EIK_PASS_COL, false))) return rc2;
      if ((rc2 = pass_planes_inplace(p, false, d_nodes, in->n_nodes, nullptr, V1, st))) return rc2;
      e.phi_raw = o_S ? o_S : (o_phi ? o_phi : p->work.as<double>());
      if ((rc2 = pass_axis0_single(p, V1, *p->kdist[p->k_exp], W1, false, st))) return rc2;
      RawOut ro;
      ro.n = 1;
      ro.dest[0] = e.phi_raw;
      if ((rc2 = pass_finish(p, &W1, r, p->c[0], p->M[1], 1, rr, st, nomark, nullptr, &ro))) return rc2;
      // gradient components: one axis-0 pass each, except the last two, which share one pass
      // (one forward transform and one read of V fewer): V is dead after them, so the first of
      // the pair lands in V's own lines (every CTA reads its lines before it writes them) and
      // the second in W.  Same arithmetic per component as the single passes (bit-identical).
      int gd[3], ng = 0;
      for (int d = 0; d < r.ngrad; ++d)
        if (o_g[d]) gd[ng++] = d;
      static const bool pair_last = [] {
        const char* ev = std::getenv("EIK_STREAM_PAIR");
        return !(ev && ev[0] == '0');
      }();
      for (int i = 0; i < ng; ++i) {
        const int d = gd[i];
        if (pair_last && ng >= 2 && i == ng - 2) {
          const int d2 = gd[i + 1];
          const KDev* kk[2] = {p->kdist[p->k_grad + d].get(), p->kdist[p->k_grad + d2].get()};
          double2* WW[2] = {V1, W1};
          if ((rc2 = pass_axis0_list(p, V1, kk, 2, WW, false, st))) return rc2;
          RawOut ro2;
          ro2.n = 2;
          ro2.dest[0] = o_g[d];
          ro2.dest[1] = o_g[d2];
          if ((rc2 = pass_finish(p, WW, r, p->c[0], p->M[1], 1, rr, st, nomark, nullptr, &ro2))) return rc2;
          e.grad[d] = o_g[d];
          e.grad[d2] = o_g[d2];
          break;
        }
        if ((rc2 = pass_axis0_single(p, V1, *p->kdist[p->k_grad + d], W1, false, st))) return rc2;
        ro.dest[0] = o_g[d];
        if ((rc2 = pass_finish(p, &W1, r, p->c[0], p->M[1], 1, rr, st, nomark, nullptr, &ro))) return rc2;
        e.grad[d] = o_g[d];
      }
      e.S = o_S;
      e.phi_out = o_phi;
      e.uf = o_uf;
      e.uf_count = ra.uf_count;
      if ((rc2 = mark(EIK_PASS_COL, true))) return rc2;
    }
    if (want_sign) {
      if ((rc2 = mark(EIK_PASS_COL_SIGN, false))) return rc2;
      if (want_fill && (rc2 = fill_prepare(st))) return rc2;
      for (int i = 0; i < 3; ++i) {
        if ((rc2 = pass_planes_inplace(p, true, d_snodes, Ks, d_sw + (int64_t)i * Ks, V1, st))) return rc2;
        if ((rc2 = pass_axis0_single(p, V1, *p->ksign[i], W1, i > 0, st))) return rc2;
      }
      e.mu_raw = o_mu ? o_mu : p->work.as<double>() + p->N;
      RawOut rs;
      rs.n = 1;
      rs.dest[0] = e.mu_raw;
      if ((rc2 = pass_finish(p, &W1, r, p->c[0], p->M[1], 1, rr, st, nomark, nullptr, &rs))) return rc2;
      e.mu = o_mu;
      e.mask = o_mask;
      if ((rc2 = mark(EIK_PASS_COL_SIGN, true))) return rc2;
    }
    if ((rc2 = mark(EIK_PASS_ROW, false))) return rc2;
    stream_epilogue_kernel<<<148 * 8, 256, 0, st>>>(e, stream_epi_vec2(e));
    CK(cudaGetLastError());
    return mark(EIK_PASS_ROW, true);
  };
  // the row pass (and, in wave mode, each wave's column pass + row pass)
  auto finish = [&](const ChunkFn& on_chunk) -> int {
    if (streamed) return run_streamed();
    if (!waves) return pass_finish(p, W.data(), r, p->c[0], p->M[1], B, ra, st, mark, on_chunk);
    std::function<int(int, bool)> nomark = [](int, bool) { return EIK_OK; };
    int rc2;
    if ((rc2 = mark(EIK_PASS_COL, false))) return rc2;
    for (int64_t b0 = 0; b0 < B; b0 += BW) {
      const int64_t nb = std::min(BW, B - b0);
      if ((rc2 = pass_col2d(p, false, d_nodes, d_off, in->n_nodes, nb, nullptr, r, W.data(), st, b0, false)))
        return rc2;
      RowArgs rw = ra;
      const int64_t o = b0 * p->N;
      auto sh = [o](auto* q) { return q ? q + o : q; };
      rw.S = sh(rw.S);
      for (int d = 0; d < 3; ++d) { rw.grad[d] = sh(rw.grad[d]); rw.hess[d] = sh(rw.hess[d]); }
      rw.mu = sh(rw.mu);
      rw.mask = sh(rw.mask);
      rw.uf = sh(rw.uf);
      rw.phi_out = sh(rw.phi_out);
      ChunkFn shifted = nullptr;
      if (on_chunk)
        shifted = [&, b0](int64_t r0, int64_t r1, int64_t i0, int64_t i1) { return on_chunk(r0, r1, b0 + i0, b0 + i1); };
      if ((rc2 = pass_finish(p, W.data(), r, p->c[0], p->M[1], nb, rw, st, nomark, shifted))) return rc2;
    }
    return mark(EIK_PASS_COL, true);
  };
  if (host_out && !slots.empty() && !prof && !streamed && NB >= (int64_t(1) << 22)) {
    // D2H of each finished chunk of rows on a copy stream, overlapping the rest
    // of the row pass (the end-to-end path is PCIe-bound on the outputs)
    // two copy streams: consecutive copies alternate between copy engines
    if (!p->st_copy) CK(cudaStreamCreateWithFlags(&p->st_copy, cudaStreamNonBlocking));
    if (!p->st_copy2) CK(cudaStreamCreateWithFlags(&p->st_copy2, cudaStreamNonBlocking));
    if (!p->ev_chunk) CK(cudaEventCreateWithFlags(&p->ev_chunk, cudaEventDisableTiming));
    if (!p->ev_copies) CK(cudaEventCreateWithFlags(&p->ev_copies, cudaEventDisableTiming));
    const int64_t nlast = p->c[p->D - 1];
    const int64_t item_nodes = p->N;
    ChunkFn on_chunk = [&](int64_t r0, int64_t r1, int64_t i0, int64_t i1) -> int {
      CK(cudaEventRecord(p->ev_chunk, st));
      CK(cudaStreamWaitEvent(p->st_copy, p->ev_chunk, 0));
      CK(cudaStreamWaitEvent(p->st_copy2, p->ev_chunk, 0));
      int k = 0;
      for (auto& sl : slots) {
        if (want_fill && sl.user == out->mask) continue;  // copied after the fill
        const size_t elem = sl.bytes / (size_t)NB;
        for (int64_t it = i0; it < i1; ++it) {
          const size_t off = ((size_t)it * item_nodes + (size_t)r0 * nlast) * elem;
          const size_t len = (size_t)(r1 - r0) * nlast * elem;
          CK(cudaMemcpyAsync((char*)sl.user + off, (char*)sl.dev + off, len, cudaMemcpyDeviceToHost,
                             (k++ & 1) ? p->st_copy2 : p->st_copy));
        }
      }
      return EIK_OK;
    };
    if ((rc = finish(on_chunk))) return rc;
    if (want_fill) {
      if ((rc = fill_finish(st))) return rc;
      CK(cudaEventRecord(p->ev_chunk, st));
      CK(cudaStreamWaitEvent(p->st_copy, p->ev_chunk, 0));
      for (auto& sl : slots)
        if (sl.user == out->mask) CK(cudaMemcpyAsync(sl.user, sl.dev, sl.bytes, cudaMemcpyDeviceToHost, p->st_copy));
    }
    CK(cudaEventRecord(p->ev_chunk, p->st_copy2));
    CK(cudaStreamWaitEvent(p->st_copy, p->ev_chunk, 0));
    CK(cudaEventRecord(p->ev_copies, p->st_copy));
    if (async) p->copies_pending = true;
    else CK(cudaStreamWaitEvent(st, p->ev_copies, 0));
    slots.clear();
  } else {
    if ((rc = finish(nullptr))) return rc;
    if (want_fill && (rc = fill_finish(st))) return rc;
  }
  // ---- copy back / sync / checks
  for (auto& s : slots) CK(cudaMemcpyAsync(s.user, s.dev, s.bytes, cudaMemcpyDeviceToHost, st));
  const bool sync = (host_out && !async) || (flags & (EIK_SYNC | EIK_CHECK_UNDERFLOW)) || out->n_underflow;
  int err_flag = 0;
  unsigned long long nuf = 0;
  if (sync) {
    if ((want_phi || p->D == 3) && p->err.p)
      CK(cudaMemcpyAsync(&err_flag, p->err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    int serr_flag = 0;
    if (want_sign && p->D == 2 && p->serr.p) {
      CK(cudaMemcpyAsync(&serr_flag, p->serr.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    }
    if (count) CK(cudaMemcpyAsync(&nuf, ctr, sizeof(nuf), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err_flag == p->run_gen || serr_flag == p->run_gen)
      return fail(EIK_EVALIDATION, "node indices must be sorted, distinct and inside the grid");
    if (out->n_underflow) *out->n_underflow = (int64_t)nuf;
    if ((flags & EIK_CHECK_UNDERFLOW) && nuf > 0)
      return fail(EIK_EUNDERFLOW, "phi has non-positive entries after convolution; increase the precision bits "
                                  "(e.g. --precision big:512) or raise tau");
  }
  return EIK_OK;
}

// ---------------------------------------------------------------------------
// Slab-decomposed 3-D pipeline (device pointers only).

static int slab_roles(const eik_plan* p, Roles& r) {
  if (p->D != 3) return fail(EIK_EVALIDATION, "the slab API is for 3-D grids");
  r.phi = p->k_exp >= 0;
  r.ngrad = p->k_grad >= 0 ? 3 : 0;
  r.hess = false;
  r.sign = !p->ksign.empty();
  return EIK_OK;
}

// Peer-to-peer slab arena: V slots (group 0: delta_Y -> slot 0; group 1: the
// three flux fields -> slots 1..3), then one W slot per component.
constexpr int P2P_NV = 4;
static int64_t p2p_vslot(int group) { return group ? 1 : 0; }
static int64_t p2p_block(const eik_plan* p) { return p->p2p_c0loc * p->p2p_ks * p->H; }
static int p2p_check(const eik_plan* p, int64_t c0_local, int64_t ks) {
  if (!p->p2p.p || (int)p->p2p_peer.size() != p->p2p_world)
    return fail(EIK_EVALIDATION, "peer-to-peer slab exchange not initialised / connected");
  for (auto* q : p->p2p_peer)
    if (!q) return fail(EIK_EVALIDATION, "peer-to-peer slab exchange not connected");
  if (c0_local != p->p2p_c0loc || ks != p->p2p_ks) return fail(EIK_EVALIDATION, "slab geometry differs from p2p_init");
  return EIK_OK;
}

int eik_slab_p2p_init(eik_plan* p, int world, int rank, int64_t c0_local, int64_t ks, void** arena,
                      int64_t* arena_bytes, void* ipc_handle) {
  if (!p) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  Roles r;
  int rc = slab_roles(p, r);
  if (rc) return rc;
  if (world < 1 || world > MAXG || rank < 0 || rank >= world)
    return fail(EIK_EVALIDATION, "peer-to-peer slab exchange supports 1..8 ranks");
  if (c0_local < 1 || (c0_local & (c0_local - 1)) || c0_local * world != p->c[0] || ks * world != p->M[1])
    return fail(EIK_EVALIDATION, "bad slab geometry (c0/G must be a power of two, M1 = G * ks)");
  p->p2p_world = world;
  p->p2p_rank = rank;
  p->p2p_c0loc = c0_local;
  p->p2p_ks = ks;
  p->p2p_slot = (int64_t)world * c0_local * ks * p->H;
  const size_t bytes = (size_t)(P2P_NV + r.n_comp()) * p->p2p_slot * sizeof(double2);
  CK(p->p2p.ensure(bytes));
  for (void* q : p->p2p_opened) cudaIpcCloseMemHandle(q);
  p->p2p_opened.clear();
  p->p2p_peer.assign(world, nullptr);
  p->p2p_peer[rank] = p->p2p.as<double2>();
  if (arena) *arena = p->p2p.p;
  if (arena_bytes) *arena_bytes = (int64_t)bytes;
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, p->p2p.p));
    std::memcpy(ipc_handle, &h, sizeof(h));
  }
  return EIK_OK;
}

int eik_slab_p2p_connect(eik_plan* p, void* const* peer_arenas, const void* ipc_handles) {
  if (!p || (!peer_arenas && !ipc_handles)) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  if (!p->p2p.p) return fail(EIK_EVALIDATION, "eik_slab_p2p_init first");
  for (int g = 0; g < p->p2p_world; ++g) {
    if (g == p->p2p_rank) continue;
    if (peer_arenas && peer_arenas[g]) {
      p->p2p_peer[g] = static_cast<double2*>(peer_arenas[g]);
    } else if (ipc_handles) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(ipc_handles) + (size_t)g * sizeof(h), sizeof(h));
      void* q = nullptr;
      CK(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
      p->p2p_opened.push_back(q);
      p->p2p_peer[g] = static_cast<double2*>(q);
    } else {
      return fail(EIK_EVALIDATION, "no arena or IPC handle for a peer rank");
    }
  }
  return EIK_OK;
}

int eik_slab_planes(eik_plan* p, int group, const int64_t* nodes, int64_t n_nodes, const double* weights,
                    int64_t c0_local, int64_t ks, double* const* v_out, uint32_t flags, void* stream) {
  const bool p2p = flags & EIK_SLAB_P2P;
  if (!p || (!v_out && !p2p)) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  Roles r;
  int rc = slab_roles(p, r);
  if (rc) return rc;
  PeerBlk pb;
  if (p2p) {
    if ((rc = p2p_check(p, c0_local, ks))) return rc;
    // this rank's block of every destination's V slots
    for (int g = 0; g < p->p2p_world; ++g)
      pb.blk[g] = p->p2p_peer[g] + p2p_vslot(group) * p->p2p_slot + p->p2p_rank * p2p_block(p);
    pb.cstride = p->p2p_slot;
  }
  if (group == 1 && !r.sign) return fail(EIK_EVALIDATION, "plan was built without sign kernels");
  if (group == 0 && !r.phi) return fail(EIK_EVALIDATION, "plan was built without the distance kernels");
  if (ks < 1 || p->M[1] % ks || (ks & (ks - 1)) || c0_local < 1) return fail(EIK_EVALIDATION, "bad slab geometry");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double2* V[3] = {nullptr, nullptr, nullptr};
  if (!p2p) {
    V[0] = (double2*)v_out[0];
    if (group) { V[1] = (double2*)v_out[1]; V[2] = (double2*)v_out[2]; }
  }
  if ((rc = pass_planes(p, group == 1, nodes, nullptr, n_nodes, 1, weights, c0_local, ks, V, st,
                        p2p ? &pb : nullptr)))
    return rc;
  if (flags & EIK_SYNC) CK(cudaStreamSynchronize(st));
  return EIK_OK;
}

int eik_slab_axis0(eik_plan* p, int group, double* const* v_in, int64_t k1_begin, int64_t ks, double* const* w_out,
                   uint32_t flags, void* stream) {
  const bool p2p = flags & EIK_SLAB_P2P;
  if (!p || (!p2p && (!v_in || !w_out))) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  Roles r;
  int rc = slab_roles(p, r);
  if (rc) return rc;
  if (ks < 1 || p->M[1] % ks || k1_begin < 0 || k1_begin + ks > p->M[1]) return fail(EIK_EVALIDATION, "bad slab geometry");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double2* V[3] = {nullptr, nullptr, nullptr};
  std::vector<double2*> W(r.n_comp(), nullptr);
  PeerBlk pb;
  if (p2p) {
    if ((rc = p2p_check(p, p->c[0] / (p->p2p_world ? p->p2p_world : 1), ks))) return rc;
    if (k1_begin != p->p2p_rank * ks) return fail(EIK_EVALIDATION, "k1 slab does not match the rank");
    double2* own = p->p2p_peer[p->p2p_rank];
    for (int i = 0; i < (group ? 3 : 1); ++i) V[i] = own + (p2p_vslot(group) + i) * p->p2p_slot;
    // rows of every owner's W slots; component j at + j * slot (the sign sum is slot n_dist)
    const int j0 = group ? r.n_dist() : 0;
    for (int g = 0; g < p->p2p_world; ++g)
      pb.blk[g] = p->p2p_peer[g] + (P2P_NV + j0) * p->p2p_slot + p->p2p_rank * p2p_block(p);
    pb.shift = ilog2_exact(p->p2p_c0loc);
    pb.cstride = p->p2p_slot;
  } else {
    V[0] = (double2*)v_in[0];
    if (group) { V[1] = (double2*)v_in[1]; V[2] = (double2*)v_in[2]; }
    if (group) W[r.n_dist()] = (double2*)w_out[0];
    else
      for (int j = 0; j < r.n_dist(); ++j) W[j] = (double2*)w_out[j];
  }
  if ((rc = pass_axis0(p, group == 1, V, k1_begin, ks, 1, r, W.data(), st, p2p ? &pb : nullptr))) return rc;
  if (flags & EIK_SYNC) CK(cudaStreamSynchronize(st));
  return EIK_OK;
}

int eik_slab_finish(eik_plan* p, double* const* w, int64_t c0_local, int64_t ks, const eik_outputs* out,
                    uint32_t flags, void* stream) {
  const bool p2p = flags & EIK_SLAB_P2P;
  if (!p || (!w && !p2p) || !out) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  Roles r;
  int rc = slab_roles(p, r);
  if (rc) return rc;
  if (ks < 1 || p->M[1] % ks || c0_local < 1) return fail(EIK_EVALIDATION, "bad slab geometry");
  if (p2p && (rc = p2p_check(p, c0_local, ks))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<double2*> W(r.n_comp());
  for (int j = 0; j < r.n_comp(); ++j)
    W[j] = p2p ? p->p2p_peer[p->p2p_rank] + (P2P_NV + j) * p->p2p_slot : (double2*)w[j];
  RowArgs ra{};
  ra.S = out->S;
  for (int d = 0; d < 3; ++d) ra.grad[d] = out->grad[d];
  ra.mu = out->mu;
  ra.mask = out->mask;
  ra.uf = out->underflow;
  ra.phi_out = out->phi;
  if (out->d_underflow_count) ra.uf_count = out->d_underflow_count;
  std::function<int(int, bool)> nomark = [](int, bool) { return EIK_OK; };
  if ((rc = pass_finish(p, W.data(), r, c0_local, ks, 1, ra, st, nomark))) return rc;
  if (flags & EIK_SYNC) CK(cudaStreamSynchronize(st));
  return EIK_OK;
}

// ---- streamed slab schedule: one input / one component at a time, so a rank
// holds one V and one W buffer pair instead of one per input and component
// (C4 at 1024^3 on 2 GPUs).  Kernels: 0 = exp, 1..3 = gradient, 4..6 = degree.

int eik_slab_planes_one(eik_plan* p, int group, int input, const int64_t* nodes, int64_t n_nodes,
                        const double* weights, int64_t c0_local, int64_t ks, double* v_out, void* stream) {
  if (!p || !v_out) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  Roles r;
  int rc = slab_roles(p, r);
  if (rc) return rc;
  if (group == 1 && (!r.sign || input < 0 || input > 2 || !weights))
    return fail(EIK_EVALIDATION, "sign input outside 0..2, no weights, or a plan without sign kernels");
  if (group == 0 && !r.phi) return fail(EIK_EVALIDATION, "plan was built without the distance kernels");
  if (ks < 1 || p->M[1] % ks || (ks & (ks - 1)) || c0_local < 1) return fail(EIK_EVALIDATION, "bad slab geometry");
  double2* V[3] = {(double2*)v_out, nullptr, nullptr};
  return pass_planes(p, group == 1, nodes, nullptr, n_nodes, 1, weights, c0_local, ks, V,
                     static_cast<cudaStream_t>(stream), nullptr, group == 1 ? input : 0, 1);
}

static const KDev* slab_kernel(const eik_plan* p, int kernel) {
  if (kernel == 0) return p->k_exp >= 0 ? p->kdist[p->k_exp].get() : nullptr;
  if (kernel >= 1 && kernel <= 3) return p->k_grad >= 0 ? p->kdist[p->k_grad + kernel - 1].get() : nullptr;
  if (kernel >= 4 && kernel <= 6) return (int)p->ksign.size() == 3 ? p->ksign[kernel - 4].get() : nullptr;
  return nullptr;
}

int eik_slab_axis0_one(eik_plan* p, int kernel, const double* v_in, int64_t k1_begin, int64_t ks, double* w_out,
                       int accumulate, void* stream) {
  if (!p || !v_in || !w_out) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  if (p->D != 3) return fail(EIK_EVALIDATION, "the slab API is for 3-D grids");
  const KDev* k = slab_kernel(p, kernel);
  if (!k) return fail(EIK_EVALIDATION, "kernel not in the plan (0 exp, 1..3 gradient, 4..6 degree)");
  if (ks < 1 || p->M[1] % ks || k1_begin < 0 || k1_begin + ks > p->M[1]) return fail(EIK_EVALIDATION, "bad slab geometry");
  double2* W = (double2*)w_out;
  return pass_axis0_list(p, (const double2*)v_in, &k, 1, &W, accumulate != 0, static_cast<cudaStream_t>(stream),
                         k1_begin, ks);
}

int eik_slab_finish_raw(eik_plan* p, double* w, int64_t c0_local, int64_t ks, double* raw_out, void* stream) {
  if (!p || !w || !raw_out) return fail(EIK_EVALIDATION, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  if (p->D != 3) return fail(EIK_EVALIDATION, "the slab API is for 3-D grids");
  if (ks < 1 || p->M[1] % ks || c0_local < 1) return fail(EIK_EVALIDATION, "bad slab geometry");
  Roles r;
  RawOut ro;
  ro.n = 1;
  ro.dest[0] = raw_out;
  double2* W = (double2*)w;
  RowArgs ra{};
  std::function<int(int, bool)> nomark = [](int, bool) { return EIK_OK; };
  return pass_finish(p, &W, r, c0_local, ks, 1, ra, static_cast<cudaStream_t>(stream), nomark, nullptr, &ro);
}

int eik_slab_epilogue(eik_plan* p, int64_t n_local, const double* phi_raw, const double* mu_raw,
                      const eik_outputs* out, void* stream) {
  if (!p || !out || n_local < 1) return fail(EIK_EVALIDATION, "null argument");
  CK(cudaSetDevice(p->device));
  StreamEpi e{};
  e.N = n_local;
  e.tau = p->tau;
  e.phi_raw = const_cast<double*>(phi_raw);
  e.mu_raw = const_cast<double*>(mu_raw);
  if (phi_raw) {
    e.S = out->S;
    e.phi_out = out->phi;
    e.uf = out->underflow;
    e.uf_count = out->d_underflow_count;
    for (int d = 0; d < 3; ++d) e.grad[d] = out->grad[d];
  }
  if (mu_raw) {
    e.mu = out->mu;
    e.mask = out->mask;
  }
  stream_epilogue_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(e, stream_epi_vec2(e));
  CK(cudaGetLastError());
  return EIK_OK;
}

int eik_slab_fill(eik_plan* p, const int64_t* ext_nodes, int64_t n_ext, int64_t e0, int64_t e1, int64_t own0,
                  int64_t c0_local, const uint8_t* mask_ext, uint8_t* mask_own, void* stream) {
  if (!p || (n_ext > 0 && (!ext_nodes || !mask_ext || !mask_own))) return fail(EIK_EVALIDATION, "null argument");
  if (p->D != 3) return fail(EIK_EVALIDATION, "the slab API is for 3-D grids");
  CK(cudaSetDevice(p->device));
  const int64_t counts[3] = {p->c[0], p->c[1], p->c[2]};
  return eik_slab_fill_mask(counts, ext_nodes, n_ext, e0, e1, own0, c0_local, mask_ext, mask_own,
                            static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// tau sweep: several exp kernels, one transform of delta_Y.

int eik_plan_create_sweep(int dim, const int64_t* counts, double spacing, const double* taus, int n_taus, int device,
                          eik_plan** out) {
  if (!out || !counts || !taus || n_taus < 1) return fail(EIK_EVALIDATION, "null argument");
  *out = nullptr;
  for (int i = 0; i < n_taus; ++i)
    if (!(taus[i] > 0)) return fail(EIK_EVALIDATION, "tau must be > 0");
  CK(cudaSetDevice(device));
  auto p = std::make_unique<eik_plan>();
  p->device = device;
  p->tau = taus[0];
  int rc = setup_geometry(p.get(), dim, counts, spacing);
  if (rc) return rc;
  if (p->D == 3) init_fold(p.get(), 0, p->M[1]);
  CK(p->work.ensure((size_t)p->M[0] * p->lines * sizeof(double2)));
  for (int i = 0; i < n_taus; ++i) {
    if ((rc = add_kernel(p.get(), p->ksweep, KT_EXP, 0, false, 1.0, p->work.as<double2>(), nullptr, taus[i]))) return rc;
    p->taus.push_back(taus[i]);
  }
  CK(cudaDeviceSynchronize());
  p->work.release();
  CK(p->counter.ensure(sizeof(unsigned long long)));
  *out = p.release();
  return EIK_OK;
}

int eik_run_sweep(eik_plan* p, const int64_t* nodes, int64_t n_nodes, double* const* S, int64_t* n_underflow,
                  uint32_t flags, void* stream) {
  if (!p || !nodes || !S || n_nodes < 1) return fail(EIK_EVALIDATION, "null argument");
  if (p->ksweep.empty()) return fail(EIK_EVALIDATION, "plan was not built for a tau sweep");
  std::lock_guard<std::mutex> lock(p->mu);
  CK(cudaSetDevice(p->device));
  p->run_gen = p->run_gen == INT_MAX ? 1 : p->run_gen + 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = flags & EIK_HOST_INPUTS, host_out = flags & EIK_HOST_OUTPUTS;
  const int nt = (int)p->taus.size();
  const int64_t* d_nodes = nodes;
  if (host_in) {
    CK(p->h_nodes.ensure(n_nodes * sizeof(int64_t)));
    CK(cudaMemcpyAsync(p->h_nodes.p, nodes, n_nodes * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    d_nodes = p->h_nodes.as<int64_t>();
  }
  std::vector<double*> outs(S, S + nt);
  if (host_out) {
    CK(p->stage.ensure((size_t)nt * p->N * sizeof(double)));
    for (int i = 0; i < nt; ++i) outs[i] = p->stage.as<double>() + (int64_t)i * p->N;
  }
  const int64_t ce = p->comp_elems();
  // 3-D: chunks of <= 4 taus (one component buffer each next to the spectrum V)
  const int chunk = p->D == 3 ? std::min(MAXC, 4) : MAXC;
  CK(p->comp.ensure((size_t)std::min(nt, chunk) * ce * sizeof(double2)));
  CK(p->counter.ensure(sizeof(unsigned long long)));
  CK(cudaMemsetAsync(p->counter.p, 0, sizeof(unsigned long long), st));
  int rc;
  if (p->D == 3) {
    // planes pass once (impulse DFT along axis 2 + FFT along axis 1); every chunk
    // of taus reuses V: axis-0 pass with the chunk's exp spectra, inverse along
    // axis 1, raw row pass with S_j = -tau_j log phi_j
    CK(p->vin.ensure((size_t)ce * sizeof(double2)));
    double2* V = p->vin.as<double2>();
    if ((rc = pass_planes_inplace(p, false, d_nodes, n_nodes, nullptr, V, st))) return rc;
    Roles r0;
    std::function<int(int, bool)> nomark = [](int, bool) { return EIK_OK; };
    for (int t0 = 0; t0 < nt; t0 += chunk) {
      const int nc = std::min(chunk, nt - t0);
      const KDev* kk[MAXC];
      double2* W[MAXC];
      RawOut ro;
      ro.n = nc;
      for (int j = 0; j < nc; ++j) {
        kk[j] = p->ksweep[t0 + j].get();
        W[j] = p->comp.as<double2>() + (int64_t)j * ce;
        ro.dest[j] = outs[t0 + j];
        ro.tau[j] = p->taus[t0 + j];
      }
      if ((rc = pass_axis0_list(p, V, kk, nc, W, false, st))) return rc;
      RowArgs ra{};
      ra.uf_count = p->counter.as<unsigned long long>();
      if ((rc = pass_finish(p, W, r0, p->c[0], p->M[1], 1, ra, st, nomark, nullptr, &ro))) return rc;
    }
  } else {
  rc = prep_nodes(p, d_nodes, nullptr, n_nodes, 1, p->N, p->c[0], p->c[1], p->rowid, p->cols,
                      p->rowptr, st);
  if (rc) return rc;
  // impulse DFT once; every chunk of <= 8 taus reuses T
  CK(p->trows.ensure((size_t)p->c[0] * p->rs() * sizeof(double2)));
  RowDftArgs rd{};
  rd.rowptr = p->rowptr.as<int64_t>();
  rd.cols = p->cols.as<int32_t>();
  rd.n_in = 1;
  rd.out[0] = p->trows.as<double2>();
  rd.rows_per_item = p->c[0];
  rd.H = p->H;
  rd.out_item = (int64_t)p->c[0] * p->rs();
  rd.out_rs = p->rs();
  rd.out_ks = 1;
  rd.last_shift = p->lmax - p->L[1];
  rd.last_mask = p->M[1] - 1;
  rd.tw = p->tw.as<double2>();
  if (p->H > (int64_t)ROWDFT_NF * ROWDFT_NT) return fail(EIK_EVALIDATION, "last axis too long for the sweep");
  CK(launch_impulse_rows(rd, 1, p->c[0], 1, st));
  double scale = 1.0;
  for (int a = 0; a < p->D; ++a) scale /= (double)p->M[a];
  for (int t0 = 0; t0 < nt; t0 += MAXC) {
    const int nc = std::min(MAXC, nt - t0);
    ColArgs a = col_defaults(p);
    a.nlines = p->H;
    a.n_valid = p->c[0];
    a.n_out = p->c[0];
    a.n_in = 1;
    a.din[0] = p->trows.as<double2>();
    a.din_es = p->rs();
    a.din_item = 0;
    a.out_es = p->rs();
    a.out_item = ce;
    a.n_comp = nc;
    for (int j = 0; j < nc; ++j) {
      a.ks[j] = kspec_of(p, *p->ksweep[t0 + j]);
      a.out[j] = p->comp.as<double2>() + (int64_t)j * ce;
    }
    if ((rc = launch_col<IN_DENSE, OUT_COMPS, true>(p->L[0], a, 1, st))) return rc;
    RowArgs ra{};
    ra.rows = p->c[0];
    ra.rows_a = p->c[0];
    ra.stride_b = p->rs();
    ra.split_shift = NOSPLIT;
    ra.comp_item = ce;
    ra.n_out = p->c[1];
    ra.c_phi = ra.c_grad = ra.c_hess = ra.c_sign = -1;
    ra.n_raw = nc;
    for (int j = 0; j < nc; ++j) {
      ra.comp[j] = a.out[j];
      ra.raw[j] = outs[t0 + j];
      ra.raw_tau[j] = p->taus[t0 + j];
    }
    ra.scale = scale;
    ra.N = p->N;
    ra.uf_count = p->counter.as<unsigned long long>();
    ra.tw = p->tw.as<double2>();
    ra.lmax = p->lmax;
    ra.row0 = 0;
    ra.row_end = ra.rows;
    if ((rc = launch_row(p->L[1] - 1, ra, 1, st))) return rc;
  }
  }
  if (host_out)
    for (int i = 0; i < nt; ++i)
      CK(cudaMemcpyAsync(S[i], outs[i], p->N * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (host_out || n_underflow || (flags & (EIK_SYNC | EIK_CHECK_UNDERFLOW))) {
    int err_flag = 0;
    unsigned long long nuf = 0;
    CK(cudaMemcpyAsync(&err_flag, p->err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&nuf, p->counter.p, sizeof(nuf), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err_flag == p->run_gen) return fail(EIK_EVALIDATION, "node indices must be sorted, distinct and inside the grid");
    if (n_underflow) *n_underflow = (int64_t)nuf;
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
    LinesArgs la = lines_defaults(&P);
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
    ColArgs a = col_defaults(&P);
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
      LinesArgs la = lines_defaults(&P);
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
    ra.split_shift = NOSPLIT;
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
    ra.row0 = 0;
    ra.row_end = ra.rows;
    ra.item0 = 0;
    if ((rc = launch_row(P.L[last] - 1, ra, 1, st))) return rc;
  }
  if (host_out) CK(cudaMemcpyAsync(out, d_out, n_kernels * P.N * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));  // temporaries are freed on return
  return EIK_OK;
}

}  // extern "C"
