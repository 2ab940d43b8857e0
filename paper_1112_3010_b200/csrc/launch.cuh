// Shared host-side helpers for the launcher translation units.
#pragma once
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// [item][row][2 * nlines doubles] view of a column-pass output (row stride out_es
// complex, item stride out_item complex), boxes of 2 * lpc doubles x 256 rows
inline bool encode_out_map(CUtensorMap* m, double2* out, const ColArgs& a, int64_t items, int lpc) {
  auto fn = tensor_map_encoder();
  if (!fn || !out) return false;
  if (((uintptr_t)out & 15) || a.out_es < a.nlines) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * a.nlines), (cuuint64_t)a.n_out, (cuuint64_t)items};
  const cuuint64_t strides[2] = {(cuuint64_t)a.out_es * 16, (cuuint64_t)(items > 1 ? a.out_item : a.out_es * a.n_out) * 16};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * lpc), 256u, 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
// line-major kernel spectra (KSpec::ls, 3-D plans with an axis 0 of 1024 points and more) are a
// compile-time property of the kernel: these are the instantiations that exist
template <int L, int IN, int OUT>
constexpr bool tmem_has_lm() { return L >= 10 && L <= 12 && IN == IN_DENSE && (OUT == OUT_COMPS || OUT == OUT_SUM); }

template <int L, int IN, int OUT, bool HALF, bool LM>
int launch_tmem_persistent_t(const ColArgs& a, int64_t items, cudaStream_t st);

template <int L, int IN, int OUT, bool HALF>
int launch_tmem_persistent(const ColArgs& a, int64_t items, cudaStream_t st) {
  if (a.ks[0].ls) {
    if constexpr (tmem_has_lm<L, IN, OUT>()) return launch_tmem_persistent_t<L, IN, OUT, HALF, true>(a, items, st);
    else return fail(EIK_EVALIDATION, "line-major kernel spectra: no column kernel for this shape");
  }
  return launch_tmem_persistent_t<L, IN, OUT, HALF, false>(a, items, st);
}

template <int L, int IN, int OUT, bool HALF, bool LM>
int launch_tmem_persistent_t(const ColArgs& a, int64_t items, cudaStream_t st) {
  using C = TmCfg<L, tm_lpcx(L, OUT), LM>;
  auto k = col_tmem_kernel<L, IN, OUT, HALF, LM>;
  const size_t smem_max = C::SMEM_BYTES + ((EIK_DBG_STAGEONLY || C::TSTORE) && L == 12 ? 256 + (size_t)(C::LN::M / 2) * C::LPC * 16 : 0);
  CK(prep_kernel_attr(k, smem_max));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || items <= 0) return EIK_OK;
  // measured (B200): persistent C2 col 0.377 -> 0.361 ms, C5 5.52 -> 5.36 ms, but
  // C3's 512-point lines 1.85 -> 1.95 ms, so those keep one CTA per tile
  const int pm = persist_mode();
  const bool persist = pm < 0 ? (L >= 10) : pm > 0;
  ColArgs b = a;
  b.tiles = tiles;
  b.items = items;
  // TMA output stores (4096-point four-step distance kernels): plain own-buffer
  // outputs only (no slab blocks, split rows or accumulation); EIK_TSTORE=0 at run time turns them off
  b.tstore = 0;
  size_t smem_tstore = 0;
  if constexpr (C::TSTORE && OUT == OUT_COMPS) {
    static const bool ts_on = [] {
      const char* e = std::getenv("EIK_TSTORE");
      return !(e && e[0] == '0');
    }();
    if (ts_on && !a.blk[0] && a.out_split_shift >= 30 && !a.accum && a.n_out <= C::LN::M / 2 && a.n_comp <= MAXC) {
      b.tstore = 1;
      for (int j = 0; j < a.n_comp && b.tstore; ++j)
        if (!encode_out_map(&b.umap[j], a.out[j], a, items, C::LPC)) b.tstore = 0;
      if (b.tstore) smem_tstore = C::SMEM_TSTORE_BYTES;
    }
  }
  const int64_t total = tiles * items;
  const int64_t wave = (int64_t)sm_count() * C::MINB;
  const int64_t grid = persist ? (total < wave ? total : wave) : total;
  if (total > 0x7fffffffLL) return fail(EIK_EVALIDATION, "too many column tiles in one launch");
  const size_t smem_bytes = smem_tstore ? smem_tstore : (EIK_DBG_STAGEONLY ? smem_max : C::SMEM_BYTES);
  k<<<(unsigned)grid, C::NT, smem_bytes, st>>>(b);
  CK(cudaGetLastError());
  return EIK_OK;
}

// Even / odd split kernel for the distance group's 4096-point lines (col_eo_kernel);
// EIK_EO=0 at run time keeps the 16-warp four-step kernel (the register-order
// spectrum copies follow the same switch, so it is read once per process)
inline bool use_eo() {
  static const bool on = [] {
    const char* e = std::getenv("EIK_EO");
    return EIK_EO && !(e && e[0] == '0');
  }();
  return on;
}
template <int IN>
int launch_eo(const ColArgs& a, int64_t items, cudaStream_t st) {
  if constexpr (EIK_EO) {
  using C = EoCfg;
  auto k = col_eo_kernel<IN>;
  CK(prep_kernel_attr(k, C::SMEM_BYTES));
  const int64_t tiles = (a.nlines + C::LPC - 1) / C::LPC;
  if (tiles <= 0 || items <= 0) return EIK_OK;
  const int64_t total = tiles * items;
  if (total > 0x7fffffffLL) return fail(EIK_EVALIDATION, "too many column tiles in one launch");
  ColArgs b = a;
  b.tiles = tiles;
  b.items = items;
  b.tstore = 0;
  const int pm = persist_mode();
  const int64_t wave = sm_count();
  const int64_t grid = pm == 0 ? total : (total < wave ? total : wave);
  k<<<(unsigned)grid, C::NT, C::SMEM_BYTES, st>>>(b);
  CK(cudaGetLastError());
  return EIK_OK;
  } else {
    return fail(EIK_EVALIDATION, "even/odd column kernel not built (-DEIK_EO=1)");
  }
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
