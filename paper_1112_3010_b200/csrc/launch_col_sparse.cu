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

template <int IN, int OUT, bool HALF>
int launch_col(int L, const ColArgs& a, int64_t items, cudaStream_t st) {
#define EIK_COL(Lc) return launch_col_t<Lc, IN, OUT, HALF>(a, items, st)
  EIK_SWITCH_L(L, EIK_COL);
#undef EIK_COL
  return EIK_OK;
}


template int launch_col<IN_SPARSE, OUT_COMPS, true>(int, const ColArgs&, int64_t, cudaStream_t);
template int launch_col<IN_SPARSE, OUT_SUM, true>(int, const ColArgs&, int64_t, cudaStream_t);
template int launch_col<IN_SPARSE, OUT_SPECTRUM, true>(int, const ColArgs&, int64_t, cudaStream_t);
