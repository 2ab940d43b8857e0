#include "launch.cuh"

template <int LH>
int launch_row_t(const RowArgs& a, int64_t items, cudaStream_t st) {
  using C = RowCfg<LH>;
  auto k = a.c_hess >= 0 ? row_kernel<LH, true> : row_kernel<LH, false>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (a.row_end - a.row0 + C::LPC - 1) / C::LPC;
  if (tiles <= 0) return EIK_OK;
  if (items > 65535) return fail(EIK_EVALIDATION, "too many items in one launch");
  k<<<dim3((unsigned)tiles, (unsigned)items), C::NT, C::SMEM_BYTES, st>>>(a);
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

