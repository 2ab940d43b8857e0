#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "launch.cuh"

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// [item][row][2 * nlines doubles] view of a column-pass output (row stride
// out_es complex, item stride out_item complex), boxes of 2*lpc doubles x 256 rows
static bool encode_out_map(CUtensorMap* m, double2* out, const ColArgs& a, int64_t items, int lpc) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * a.nlines), (cuuint64_t)a.n_out, (cuuint64_t)items};
  const cuuint64_t strides[2] = {(cuuint64_t)a.out_es * 16, (cuuint64_t)a.out_item * 16};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * lpc), 256u, 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  if ((a.out_es * 16) % 16 || (a.out_item * 16) % 16 || ((uintptr_t)out & 15)) return false;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// EIK_TMEM=0 selects the register-resident column kernel for A/B runs.
static bool use_tmem() {
  static const bool on = [] {
    const char* e = std::getenv("EIK_TMEM");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int L, int IN, int OUT, bool HALF>
int launch_tmem_t(const ColArgs& a, int64_t items, cudaStream_t st) {
  using C = TmCfg<L, tm_lpcx(L, OUT)>;
  auto k = col_tmem_kernel<L, IN, OUT, HALF>;
  constexpr size_t SMEM_MAX = std::max({C::SMEM_FEED_BYTES, C::SMEM_SFEED_BYTES, C::SMEM_BYTES + C::TSTORE_BYTES});
  CK(prep_kernel_attr(k, SMEM_MAX));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || items <= 0) return EIK_OK;
  if (items > 65535) return fail(EIK_EVALIDATION, "too many items in one launch");
  // kernel-spectrum feed: every component has a register-order spectrum of this configuration
  ColArgs b = a;
  b.kfeed = 0;
  if (C::KFEED && OUT == OUT_COMPS && !a.blk[0]) {
    b.kfeed = 1;
    for (int j = 0; j < a.n_comp; ++j) b.kfeed &= (a.ks[j].perm != nullptr);
  }
  b.sfeed = (C::SFEED && OUT == OUT_SUM && IN == IN_DENSE && HALF) ? 1 : 0;
  // TMA output stores: plain own-buffer outputs (no slab blocks or split rows), whole 256-row boxes
  b.tstore = 0;
  if (C::TSTORE && OUT == OUT_COMPS && !b.kfeed && !a.blk[0] && a.out_split_shift >= 30 && a.n_out % 256 == 0 &&
      a.n_out <= C::LN::M / 2) {
    b.tstore = 1;
    for (int j = 0; j < a.n_comp && b.tstore; ++j)
      if (!encode_out_map(&b.umap[j], a.out[j], a, items, C::LPC)) b.tstore = 0;
  }
  const size_t smem = b.kfeed ? C::SMEM_FEED_BYTES : b.sfeed ? C::SMEM_SFEED_BYTES
                    : b.tstore ? C::SMEM_BYTES + C::TSTORE_BYTES : C::SMEM_BYTES;
  k<<<dim3((unsigned)tiles, (unsigned)items), C::NT, smem, st>>>(b);
  CK(cudaGetLastError());
  return EIK_OK;
}

template <int L, int IN, int OUT, bool HALF>
int launch_col_t(const ColArgs& a, int64_t items, cudaStream_t st) {
  if constexpr ((OUT == OUT_COMPS || OUT == OUT_SUM) && L >= 9) {
    if (use_tmem() && a.ks[0].cplx == nullptr) return launch_tmem_t<L, IN, OUT, HALF>(a, items, st);
  }
  using C = ColCfg<L>;
  auto k = col_kernel<L, IN, OUT, HALF>;
  const size_t smem = C::SMEM_BYTES + (IN == IN_SPARSE ? SPARSE_SMEM : 0);
  CK(prep_kernel_attr(k, smem));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || items <= 0) return EIK_OK;
  if (items > 65535) return fail(EIK_EVALIDATION, "too many items in one launch");
  k<<<dim3((unsigned)tiles, (unsigned)items), C::NT, smem, st>>>(a);
  CK(cudaGetLastError());
  return EIK_OK;
}

// Register-order spectrum for the column kernel launch_col picks at length 2^L
// for real spectra (COMPS / SUM).  kp == nullptr: only report the size.
template <class C>
int permute_t(const double* re, int64_t ld, int64_t nlines, int odd0, double* kp, int64_t* elems, int* folded,
              cudaStream_t st) {
  const int64_t tiles = (nlines + C::LPC - 1) / C::LPC;
  const int64_t total = tiles * C::LN::EPT * C::NTP;
  *elems = total;
  *folded = C::PFOLD ? 1 : 0;
  if (!kp || total == 0) return EIK_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 64);
  spectrum_perm_kernel<C><<<(unsigned)blocks, 256, 0, st>>>(re, ld, nlines, odd0, kp, total);
  CK(cudaGetLastError());
  return EIK_OK;
}

int launch_spectrum_perm(int L, bool sum, const double* re, int64_t ld, int64_t nlines, int odd0, double* kp,
                         int64_t* elems, int* folded, cudaStream_t st) {
#define EIK_PERM(Lc)                                                                                     \
  if constexpr (Lc >= 9) {                                                                               \
    if (use_tmem())                                                                                      \
      return sum ? permute_t<TmCfg<Lc, tm_lpcx(Lc, OUT_SUM)>>(re, ld, nlines, odd0, kp, elems, folded, st)       \
                 : permute_t<TmCfg<Lc, tm_lpcx(Lc, OUT_COMPS)>>(re, ld, nlines, odd0, kp, elems, folded, st);    \
  }                                                                                                      \
  return permute_t<ColCfg<Lc>>(re, ld, nlines, odd0, kp, elems, folded, st)
  EIK_SWITCH_L(L, EIK_PERM);
#undef EIK_PERM
  return EIK_OK;
}

template <int IN, int OUT, bool HALF>
int launch_col(int L, const ColArgs& a, int64_t items, cudaStream_t st) {
#define EIK_COL(Lc) return launch_col_t<Lc, IN, OUT, HALF>(a, items, st)
  EIK_SWITCH_L(L, EIK_COL);
#undef EIK_COL
  return EIK_OK;
}


template int launch_col<IN_DENSE, OUT_COMPS, true>(int, const ColArgs&, int64_t, cudaStream_t);
template int launch_col<IN_DENSE, OUT_SUM, true>(int, const ColArgs&, int64_t, cudaStream_t);
