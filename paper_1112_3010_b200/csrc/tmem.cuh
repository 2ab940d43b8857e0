// Tensor-memory (TMEM) as per-thread spill space for the column kernels.
//
// The fused column pass keeps the forward spectrum X of its line for all
// output components.  Holding X in registers next to the per-component
// product limits a 4096-point line to one CTA per SM.  Here X lives in TMEM
// (256 KB per SM, tcgen05.st / tcgen05.ld), so the registers hold only the
// product and two CTAs share each SM.
//
// Mapping: warp w addresses TMEM lanes [32*(w%4), 32*(w%4)+32) (the .32x32b
// shape: one lane per thread) and its own block of 4*EPT 32-bit columns at
// column (w/4) * 4*EPT.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace eik {

// One warp allocates `ncols` (power of two >= 32) columns; the base address
// is published through shared memory.  Call from all threads of the CTA.
__device__ __forceinline__ uint32_t tmem_alloc_cta(uint32_t* slot, uint32_t ncols) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  return *reinterpret_cast<volatile uint32_t*>(slot);
}

__device__ __forceinline__ void tmem_free_cta(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(ncols));
}

// This thread's TMEM address for `words_per_thread` consecutive 32-bit columns.
__device__ __forceinline__ uint32_t tmem_thread_addr(uint32_t base, int words_per_thread) {
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t lane0 = 32u * (w & 3u);
  const uint32_t col = (w >> 2) * (uint32_t)words_per_thread;
  return base + (lane0 << 16) + col;
}

__device__ __forceinline__ void tmem_st8(uint32_t a, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(a)
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t a, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// Store / load N complex doubles (4*N 32-bit words) at this thread's TMEM columns.
template <int N>
__device__ __forceinline__ void tmem_put(uint32_t a, const double2 (&v)[N]) {
  static_assert(N % 2 == 0, "whole 8-word chunks");
#pragma unroll
  for (int c = 0; c < N / 2; ++c) {
    uint32_t r[8];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double2 x = v[2 * c + k];
      r[4 * k + 0] = (uint32_t)__double_as_longlong(x.x);
      r[4 * k + 1] = (uint32_t)((unsigned long long)__double_as_longlong(x.x) >> 32);
      r[4 * k + 2] = (uint32_t)__double_as_longlong(x.y);
      r[4 * k + 3] = (uint32_t)((unsigned long long)__double_as_longlong(x.y) >> 32);
    }
    tmem_st8(a + 8 * c, r);
  }
  tmem_wait_st();
}

template <int N>
__device__ __forceinline__ void tmem_get(uint32_t a, double2 (&v)[N]) {
  static_assert(N % 2 == 0, "whole 8-word chunks");
  uint32_t r[4 * N];
#pragma unroll
  for (int c = 0; c < N / 2; ++c) tmem_ld8(a + 8 * c, r + 8 * c);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    v[i].x = __longlong_as_double((long long)(((unsigned long long)r[4 * i + 1] << 32) | r[4 * i + 0]));
    v[i].y = __longlong_as_double((long long)(((unsigned long long)r[4 * i + 3] << 32) | r[4 * i + 2]));
  }
}

}  // namespace eik
