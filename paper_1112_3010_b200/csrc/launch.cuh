// Shared host-side helpers for the launcher translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "../../include/eikfld_b200.h"
#include "kernels.cuh"

using namespace eik;

int eik_fail(int code, const std::string& msg);
inline int fail(int code, const std::string& msg) { return eik_fail(code, msg); }

#define CK(x)                                                                                          \
  do {                                                                                                 \
    cudaError_t e_ = (x);                                                                              \
    if (e_ != cudaSuccess) return fail(EIK_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class K>
inline cudaError_t prep_kernel_attr(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

#define EIK_SWITCH_L(Lv, MACRO)                                                         \
  switch (Lv) {                                                                         \
    case 0: MACRO(0); break;   case 1: MACRO(1); break;   case 2: MACRO(2); break;     \
    case 3: MACRO(3); break;   case 4: MACRO(4); break;   case 5: MACRO(5); break;     \
    case 6: MACRO(6); break;   case 7: MACRO(7); break;   case 8: MACRO(8); break;     \
    case 9: MACRO(9); break;   case 10: MACRO(10); break; case 11: MACRO(11); break;   \
    case 12: MACRO(12); break; case 13: MACRO(13); break;                              \
    default: return fail(EIK_EVALIDATION, "transform length out of range");            \
  }

// SMs of the current device (cached per device)
inline int sm_count() {
  static int cached[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

// EIK_PERSIST: 0 / 1 force one CTA per tile / persistent CTAs everywhere; unset: per-kernel default
inline int persist_mode() {
  static const int mode = [] {
    const char* e = std::getenv("EIK_PERSIST");
    return (e && (e[0] == '0' || e[0] == '1')) ? e[0] - '0' : -1;
  }();
  return mode;
}

// Persistent launch of the TMEM column kernel: one resident wave of CTAs walks
// the (item, tile) list (EIK_PERSIST=0: one CTA per tile, for A/B runs).
template <int L, int IN, int OUT, bool HALF>
int launch_tmem_persistent(const ColArgs& a, int64_t items, cudaStream_t st) {
  using C = TmCfg<L, tm_lpcx(L, OUT)>;
  auto k = col_tmem_kernel<L, IN, OUT, HALF>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || items <= 0) return EIK_OK;
  // measured (B200): persistent C2 col 0.377 -> 0.361 ms, C5 5.52 -> 5.36 ms, but
  // C3's 512-point lines 1.85 -> 1.95 ms, so those keep one CTA per tile
  const int pm = persist_mode();
  const bool persist = pm < 0 ? (L >= 10) : pm > 0;
  ColArgs b = a;
  b.tiles = tiles;
  b.items = items;
  const int64_t total = tiles * items;
  const int64_t wave = (int64_t)sm_count() * C::MINB;
  const int64_t grid = persist ? (total < wave ? total : wave) : total;
  if (total > 0x7fffffffLL) return fail(EIK_EVALIDATION, "too many column tiles in one launch");
  k<<<(unsigned)grid, C::NT, C::SMEM_BYTES, st>>>(b);
  CK(cudaGetLastError());
  return EIK_OK;
}

template <int IN, int OUT, bool HALF>
int launch_col(int L, const ColArgs& a, int64_t items, cudaStream_t st);
template <bool INV, bool HALF>
int launch_lines(int L, const LinesArgs& a, int ncomp, cudaStream_t st);
int launch_spectrum_perm(int L, bool sum, const double* re, int64_t ld, int64_t nlines, int odd0, double* kp, int64_t* elems,
                         int* folded, cudaStream_t st);
int launch_row(int LH, const RowArgs& a, int64_t items, cudaStream_t st);
int launch_r2c(int LH, const GenArgs& g, int64_t nrows, double2* out, int64_t out_rs, const double2* tw, int lmax,
               cudaStream_t st);
