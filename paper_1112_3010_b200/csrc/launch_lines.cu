#include "launch.cuh"

template <int L, bool INV, bool HALF>
int launch_lines_t(const LinesArgs& a, int ncomp, cudaStream_t st) {
  using C = LinesCfg<L>;
  auto k = lines_kernel<L, INV, HALF>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || ncomp <= 0) return EIK_OK;
  const int64_t total = tiles * ncomp;
  if (total > 0x7fffffffLL) return fail(EIK_EVALIDATION, "too many line tiles in one launch");
  LinesArgs b = a;
  b.tiles = tiles;
  b.ncomp = ncomp;
  const int64_t wave = (int64_t)sm_count() * (C::NT >= 512 ? 1 : 512 / C::NT);  // 16 resident warps per SM
  const int64_t grid = (C::PERSIST && persist_mode() != 0 && total > wave) ? wave : total;
  k<<<(unsigned)grid, C::NT, C::SMEM_BYTES, st>>>(b);
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
