#include "launch.cuh"

template <int L, bool INV, bool HALF>
int launch_lines_t(const LinesArgs& a, int ncomp, cudaStream_t st) {
  using C = ColCfg<L>;
  auto k = lines_kernel<L, INV, HALF>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0) return EIK_OK;
  k<<<dim3((unsigned)tiles, (unsigned)ncomp), C::NT, C::SMEM_BYTES, st>>>(a);
  CK(cudaGetLastError());
  return EIK_OK;
}

template <bool INV, bool HALF>
int launch_lines(int L, const LinesArgs& a, int ncomp, cudaStream_t st) {
#define EIK_LIN(Lc) return launch_lines_t<Lc, INV, HALF>(a, ncomp, st)
  EIK_SWITCH_L(L, EIK_LIN);
#undef EIK_LIN
  return EIK_OK;
}


template int launch_lines<false, false>(int, const LinesArgs&, int, cudaStream_t);
template int launch_lines<true, false>(int, const LinesArgs&, int, cudaStream_t);
template int launch_lines<false, true>(int, const LinesArgs&, int, cudaStream_t);
