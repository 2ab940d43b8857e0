// Shared host-side helpers for the launcher translation units.
#pragma once
#include <cuda_runtime.h>

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

template <int IN, int OUT, bool HALF>
int launch_col(int L, const ColArgs& a, int64_t items, cudaStream_t st);
template <bool INV, bool HALF>
int launch_lines(int L, const LinesArgs& a, int ncomp, cudaStream_t st);
int launch_spectrum_perm(int L, bool sum, const double* re, int64_t ld, int64_t nlines, int odd0, double* kp, int64_t* elems,
                         int* folded, cudaStream_t st);
int launch_row(int LH, const RowArgs& a, int64_t items, cudaStream_t st);
int launch_r2c(int LH, const GenArgs& g, int64_t nrows, double2* out, int64_t out_rs, const double2* tw, int lmax,
               cudaStream_t st);
