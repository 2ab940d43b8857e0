#include <algorithm>
#include <cstdlib>

#include "launch.cuh"

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
  return launch_tmem_persistent<L, IN, OUT, HALF>(a, items, st);
}

template <int L, int IN, int OUT, bool HALF>
int launch_col_t(const ColArgs& a, int64_t items, cudaStream_t st) {
  if constexpr (EIK_EO && L == 12 && OUT == OUT_COMPS && HALF) {
    if (use_tmem() && use_eo() && a.ks[0].cplx == nullptr && !a.ks[0].ls && a.n_valid <= 2048 && a.n_out <= 2048)
      return launch_eo<IN>(a, items, st);
  }
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
  if constexpr (EIK_EO && Lc == 12) {                                                                    \
    if (use_tmem() && use_eo() && !sum) return permute_t<EoCfg>(re, ld, nlines, odd0, kp, elems, folded, st);  \
  }                                                                                                      \
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
