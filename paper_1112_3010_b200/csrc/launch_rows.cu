#include "launch.cuh"

template <int LH>
int launch_row_t(const RowArgs& a, int64_t items, cudaStream_t st) {
  using C = RowCfg<LH>;
  auto k = a.c_hess >= 0 ? row_kernel<LH, true> : row_kernel<LH, false>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (a.row_end - a.row0 + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || items <= 0) return EIK_OK;
  // persistent: one resident wave of CTAs walks the (item, tile) list, the row
  // feed running one component ahead across tiles (EIK_PERSIST=0: one CTA per tile)
  const int pm = persist_mode();
  const bool persist = pm < 0 ? true : pm > 0;
  RowArgs b = a;
  b.tiles = tiles;
  b.items = items;
  const int64_t total = tiles * items;
  if (total > 0x7fffffffLL) return fail(EIK_EVALIDATION, "too many row tiles in one launch");
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::NT, C::SMEM_BYTES));
  const int64_t wave = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
  const int64_t grid = persist ? (total < wave ? total : wave) : total;
  k<<<(unsigned)grid, C::NT, C::SMEM_BYTES, st>>>(b);
  CK(cudaGetLastError());
  return EIK_OK;
}

int launch_row(int LH, const RowArgs& a, int64_t items, cudaStream_t st) {
#define EIK_ROW(Lc) return launch_row_t<Lc>(a, items, st)
  EIK_SWITCH_L(LH, EIK_ROW);
#undef EIK_ROW
  return EIK_OK;
}

template <int LH>
int launch_r2c_t(const GenArgs& g, int64_t nrows, double2* out, int64_t out_rs, const double2* tw, int lmax,
                 cudaStream_t st) {
  using C = RowCfg<LH>;
  auto k = row_r2c_kernel<LH>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (nrows + C::LPC - 1) / C::LPC;
  if (tiles <= 0) return EIK_OK;
  k<<<(unsigned)tiles, C::NT, C::SMEM_BYTES, st>>>(g, nrows, out, out_rs, tw, lmax);
  CK(cudaGetLastError());
  return EIK_OK;
}

int launch_r2c(int LH, const GenArgs& g, int64_t nrows, double2* out, int64_t out_rs, const double2* tw, int lmax,
               cudaStream_t st) {
#define EIK_R2C(Lc) return launch_r2c_t<Lc>(g, nrows, out, out_rs, tw, lmax, st)
  EIK_SWITCH_L(LH, EIK_R2C);
#undef EIK_R2C
  return EIK_OK;
}

