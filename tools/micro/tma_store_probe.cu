// TMA tensor-store throughput for narrow boxes: every CTA (one per SM) stages a
// [rows][W doubles] tile in shared memory and stores it as boxes of W doubles x
// 256 rows into a row-major global tensor whose row stride is 32 KB (the layout
// of the column pass's U_j[row][k1] output, two adjacent lines = 4 doubles).
// Prints bytes / clock / SM and the aggregate rate for W = 4, 8, 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_store_probe tma_store_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W>
__global__ void __launch_bounds__(512) probe(const __grid_constant__ CUtensorMap map, int rows, int iters, long long* clk) {
  extern __shared__ __align__(128) double tile[];
  for (int i = threadIdx.x; i < rows * W; i += blockDim.x) tile[i] = (double)(i + blockIdx.x);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      for (int y = 0; y < rows; y += 256)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                         reinterpret_cast<uint64_t>(&map)),
                     "r"((int)(blockIdx.x * W)), "r"(y), "r"(smem_u32(tile + (size_t)y * W))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
}

template <int W>
void run(PFN_cuTensorMapEncodeTiled_v12000 enc, double* out, int rows, int64_t row_stride_doubles, int ctas) {
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)row_stride_doubles, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)row_stride_doubles * 8};
  const cuuint32_t box[2] = {(cuuint32_t)W, 256u};
  const cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return; }
  long long* clk;
  cudaMalloc(&clk, ctas * sizeof(long long));
  const size_t smem = (size_t)rows * W * 8;
  cudaFuncSetAttribute(probe<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 50;
  probe<W><<<ctas, 512, smem>>>(map, rows, 2, clk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<W><<<ctas, 512, smem>>>(map, rows, iters, clk);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  cudaMemcpy(h, clk, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += (double)h[i];
  mean /= ctas;
  const double bytes = (double)rows * W * 8 * iters;
  printf("W=%2d doubles (%3d B rows) rows=%d: %s  %.1f clk per %zu-byte tile, %.2f B/clk/SM, aggregate %.1f GB/s\n", W, W * 8,
         rows, cudaGetErrorString(err), mean / iters, smem, bytes / mean, bytes * ctas / (ms * 1e-3) / 1e9);
  cudaFree(clk);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaFree(0);
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) { printf("no encode fn\n"); return 1; }
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int rows = 2048, ctas = 148;
  const int64_t stride = 4112;  // doubles per row (2056 complex, C2's U_j)
  double* out;
  cudaMalloc(&out, (size_t)rows * stride * 8);
  run<4>(enc, out, rows, stride, ctas);
  run<8>(enc, out, rows, stride, ctas);
  run<16>(enc, out, rows, stride, ctas);
  return 0;
}
