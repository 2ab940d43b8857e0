// Interior classification on the GPU: nearest-unflagged fill + rounding rule
// (R/sign.py:166-198) and the signed distance (R/sign.py:201-208).
//
// The fill must pick exactly the node scipy.ndimage.distance_transform_edt
// (return_indices=True) picks, ties included, so this is the same separable
// feature transform scipy runs (Voronoi lower envelope along axis 0, then
// axis 1 [, axis 2], in float64 with the same comparisons and the same
// "<=" tie rules), one thread per line.  tests/test_classify_port.py checks
// the algorithm against scipy on CPU; the GPU tests check this kernel
// against scipy.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/eikfld_b200.h"

int eik_fail(int code, const std::string& msg);

namespace {

#define CKC(x)                                                                                    \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) return eik_fail(EIK_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct EdtArgs {
  int rank, d;
  int64_t n[3], stride[3];  // node counts and flat strides per axis
  int32_t* F;               // features: F[a * N + node] (axis-a coordinate), -1 = none
  int32_t* g;               // scratch: stacks [line][n_d], then envelope features [line][n_d][rank]
  int64_t N, nlines;
};

// scipy ni_morphology.c _VoronoiFT along axis d for every line (sampling = None).
__global__ void edt_lines_kernel(const EdtArgs a) {
  const int64_t line = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (line >= a.nlines) return;
  const int d = a.d;
  // fixed coordinates of the line: decompose `line` over the other axes
  int64_t coor[3] = {0, 0, 0};
  int64_t rem = line, base = 0;
  for (int jj = a.rank - 1; jj >= 0; --jj) {
    if (jj == d) continue;
    coor[jj] = rem % a.n[jj];
    rem /= a.n[jj];
    base += coor[jj] * a.stride[jj];
  }
  const int64_t len = a.n[d], st = a.stride[d];
  int32_t* g = a.g + line * len;
  int l = -1;
  for (int ii = 0; ii < len; ++ii) {
    const int64_t node = base + ii * st;
    if (a.F[node] < 0) continue;  // axis-0 feature coordinate < 0 marks "no feature"
    const double fd = (double)a.F[d * a.N + node];
    double wR = 0.0;
    for (int jj = 0; jj < a.rank; ++jj)
      if (jj != d) {
        const double tw = (double)a.F[jj * a.N + node] - (double)coor[jj];
        wR += tw * tw;
      }
    while (l >= 1) {
      const int64_t n1 = base + (int64_t)g[l] * st, n2 = base + (int64_t)g[l - 1] * st;
      const double f1 = (double)a.F[d * a.N + n1];
      const double av = f1 - (double)a.F[d * a.N + n2];
      const double bv = fd - f1;
      const double cv = av + bv;
      double uR = 0.0, vR = 0.0;
      for (int jj = 0; jj < a.rank; ++jj)
        if (jj != d) {
          const double cc = (double)coor[jj];
          const double tu = (double)a.F[jj * a.N + n2] - cc;
          const double tv = (double)a.F[jj * a.N + n1] - cc;
          uR += tu * tu;
          vR += tv * tv;
        }
      if (cv * vR - bv * uR - av * wR - av * bv * cv <= 0.0) break;
      --l;
    }
    ++l;
    g[l] = ii;
  }
  const int maxl = l;
  if (maxl < 0) return;  // no feature on this line: entries stay -1
  // scipy reads the winners from a copy of the line's features (its local f),
  // and this pass overwrites F in place: copy the envelope's features first.
  int32_t* E = a.g + a.nlines * len + line * len * a.rank;
  for (int k = 0; k <= maxl; ++k) {
    const int64_t nd = base + (int64_t)g[k] * st;
    for (int jj = 0; jj < a.rank; ++jj) E[k * a.rank + jj] = a.F[jj * a.N + nd];
  }
  l = 0;
  for (int ii = 0; ii < len; ++ii) {
    double delta1 = 0.0;
    for (int jj = 0; jj < a.rank; ++jj) {
      const double f = (double)E[l * a.rank + jj];
      const double t = (jj == d) ? f - (double)ii : f - (double)coor[jj];
      delta1 += t * t;
    }
    while (l < maxl) {
      double delta2 = 0.0;
      for (int jj = 0; jj < a.rank; ++jj) {
        const double f = (double)E[(l + 1) * a.rank + jj];
        const double t = (jj == d) ? f - (double)ii : f - (double)coor[jj];
        delta2 += t * t;
      }
      if (delta1 <= delta2) break;
      delta1 = delta2;
      ++l;
    }
    const int64_t node = base + ii * st;
    for (int jj = 0; jj < a.rank; ++jj) a.F[jj * a.N + node] = E[l * a.rank + jj];
  }
}

__global__ void edt_init_kernel(const uint8_t* flagged, int rank, const int64_t n1, const int64_t n2, int64_t N,
                                int32_t* F) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (flagged[i]) {
    for (int a = 0; a < rank; ++a) F[a * N + i] = -1;
    return;
  }
  if (rank == 1) {
    F[i] = (int32_t)i;
  } else if (rank == 2) {
    F[i] = (int32_t)(i / n1);
    F[N + i] = (int32_t)(i % n1);
  } else {
    F[i] = (int32_t)(i / (n1 * n2));
    F[N + i] = (int32_t)((i / n2) % n1);
    F[2 * N + i] = (int32_t)(i % n2);
  }
}

__global__ void flag_kernel(const int64_t* idx, int64_t n, int64_t N, uint8_t* flagged, int* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = idx[i];
  if (v < 0 || v >= N) {
    atomicExch(err, 1);
    return;
  }
  flagged[v] = 1;
}

// mask = rule(mu at the node or at its nearest unflagged node); optional signed distance
__global__ void classify_kernel(const double* mu, const uint8_t* flagged, const int32_t* F, int rank, int64_t s0,
                                int64_t s1, int64_t N, int mode, int use_thr, double thr, double* mask,
                                const double* S, double* signed_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int64_t src = i;
  if (flagged && flagged[i]) {
    if (rank == 1) src = F[i];
    else if (rank == 2) src = (int64_t)F[i] * s0 + (int64_t)F[N + i];
    else src = (int64_t)F[i] * s0 + (int64_t)F[N + i] * s1 + (int64_t)F[2 * N + i];
  }
  const double v = mu[src];
  bool inside;
  if (use_thr) inside = v >= thr;
  else if (mode == 1) inside = rint(v) > 0.0;
  else inside = rint(v) >= 1.0;
  const double m = inside ? 1.0 : 0.0;
  if (mask) mask[i] = m;
  if (signed_out) signed_out[i] = (m > 0.5) ? S[i] : -S[i];
}

struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

extern "C" int eik_classify(int dim, const int64_t* counts, const double* mu, const int64_t* flagged_nodes,
                            int64_t n_flagged, int mode, int use_threshold, double threshold, double* out_mask,
                            const double* S, double* out_signed, uint32_t flags, int device, void* stream) {
  if (!counts || !mu || dim < 1 || dim > 3) return eik_fail(EIK_EVALIDATION, "bad arguments");
  if (mode != 1 && mode != 2) return eik_fail(EIK_EVALIDATION, "unknown classification mode");
  if (out_signed && !S) return eik_fail(EIK_EVALIDATION, "signed distance needs S");
  CKC(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t n[3] = {1, 1, 1}, N = 1;
  for (int a = 0; a < dim; ++a) {
    n[a] = counts[a];
    N *= counts[a];
  }
  const bool host = flags & (EIK_HOST_INPUTS | EIK_HOST_OUTPUTS);
  Buf b_mu, b_S, b_fl, b_idx, b_F, b_g, b_mask, b_sd, b_err;
  const double* d_mu = mu;
  const double* d_S = S;
  const int64_t* d_idx = flagged_nodes;
  if (host) {
    CKC(cudaMalloc(&b_mu.p, N * sizeof(double)));
    CKC(cudaMemcpyAsync(b_mu.p, mu, N * sizeof(double), cudaMemcpyHostToDevice, st));
    d_mu = (const double*)b_mu.p;
    if (S) {
      CKC(cudaMalloc(&b_S.p, N * sizeof(double)));
      CKC(cudaMemcpyAsync(b_S.p, S, N * sizeof(double), cudaMemcpyHostToDevice, st));
      d_S = (const double*)b_S.p;
    }
    if (n_flagged > 0) {
      CKC(cudaMalloc(&b_idx.p, n_flagged * sizeof(int64_t)));
      CKC(cudaMemcpyAsync(b_idx.p, flagged_nodes, n_flagged * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      d_idx = (const int64_t*)b_idx.p;
    }
  }
  double* d_mask = out_mask;
  double* d_sd = out_signed;
  if (host) {
    if (out_mask) {
      CKC(cudaMalloc(&b_mask.p, N * sizeof(double)));
      d_mask = (double*)b_mask.p;
    }
    if (out_signed) {
      CKC(cudaMalloc(&b_sd.p, N * sizeof(double)));
      d_sd = (double*)b_sd.p;
    }
  }
  const uint8_t* d_fl = nullptr;
  const int32_t* d_F = nullptr;
  int err = 0;
  if (n_flagged > 0) {
    CKC(cudaMalloc(&b_fl.p, N));
    CKC(cudaMemsetAsync(b_fl.p, 0, N, st));
    CKC(cudaMalloc(&b_err.p, sizeof(int)));
    CKC(cudaMemsetAsync(b_err.p, 0, sizeof(int), st));
    flag_kernel<<<(unsigned)((n_flagged + 255) / 256), 256, 0, st>>>(d_idx, n_flagged, N, (uint8_t*)b_fl.p,
                                                                    (int*)b_err.p);
    CKC(cudaGetLastError());
    CKC(cudaMalloc(&b_F.p, (size_t)dim * N * sizeof(int32_t)));
    edt_init_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>((const uint8_t*)b_fl.p, dim, n[1], n[2], N,
                                                                (int32_t*)b_F.p);
    CKC(cudaGetLastError());
    // per line: stack (len) + envelope feature copies (len * rank); nlines * len = N per phase
    CKC(cudaMalloc(&b_g.p, (size_t)N * (1 + dim) * sizeof(int32_t)));
    int64_t stride[3] = {1, 1, 1};
    for (int a = dim - 2; a >= 0; --a) stride[a] = stride[a + 1] * n[a + 1];
    for (int d = 0; d < dim; ++d) {
      EdtArgs ea{};
      ea.rank = dim;
      ea.d = d;
      for (int a = 0; a < 3; ++a) { ea.n[a] = n[a]; ea.stride[a] = stride[a]; }
      ea.F = (int32_t*)b_F.p;
      ea.g = (int32_t*)b_g.p;
      ea.N = N;
      ea.nlines = N / n[d];
      edt_lines_kernel<<<(unsigned)((ea.nlines + 127) / 128), 128, 0, st>>>(ea);
      CKC(cudaGetLastError());
    }
    d_fl = (const uint8_t*)b_fl.p;
    d_F = (const int32_t*)b_F.p;
  }
  const int64_t s0 = dim == 3 ? n[1] * n[2] : (dim == 2 ? n[1] : 1), s1 = dim == 3 ? n[2] : 1;
  classify_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(d_mu, d_fl, d_F, dim, s0, s1, N, mode, use_threshold,
                                                              threshold, d_mask, d_S, d_sd);
  CKC(cudaGetLastError());
  if (host) {
    if (out_mask) CKC(cudaMemcpyAsync(out_mask, d_mask, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (out_signed) CKC(cudaMemcpyAsync(out_signed, d_sd, N * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  if (b_err.p) CKC(cudaMemcpyAsync(&err, b_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKC(cudaStreamSynchronize(st));  // temporaries are freed on return
  if (err) return eik_fail(EIK_EVALIDATION, "flagged node index out of grid bounds");
  return EIK_OK;
}
