// Interior classification on the GPU: nearest-unflagged fill + rounding rule
// (R/sign.py:166-198) and the signed distance (R/sign.py:201-208).
//
// The fill must pick exactly the node scipy.ndimage.distance_transform_edt
// (return_indices=True) picks, ties included, so this is the same separable
// feature transform scipy runs (Voronoi lower envelope along axis 0, then
// axis 1 [, axis 2], in float64 with the same comparisons and the same
// "<=" tie rules), one thread per line.  tests/test_edt_port.py checks
// the algorithm against scipy on CPU; the GPU tests check this kernel
// against scipy.
//
// Sparse flagged sets (curve / surface nodes: the sign fields' flagged nodes)
// take a per-flagged-node path instead (fill_fix_kernel): with integer
// coordinates every comparison of scipy's envelope pass is exact, and its
// result at a flagged node p of the line along axis d is the pass-(d-1)
// feature of the line member of smallest position among those nearest to p
// (minimisers are never popped from the envelope stack; the query walk stops
// at the first).  Only members with offset^2 <= the best distance so far can
// tie or win, so each flagged node scans a few neighbours per axis.
// tests/fill_rule.py restates the rule and tests/test_fill_rule.py checks it
// against scipy (random, block and curve masks, 1-3-D).
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
    if (err) atomicExch(err, 1);
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

// ---- sparse fill ------------------------------------------------------------

__global__ void fill_bits_kernel(const int64_t* nodes, int64_t K, int64_t N, uint32_t* bits, int* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t v = nodes[i];
  if (v < 0 || v >= N) {
    if (err) atomicExch(err, 1);
    return;
  }
  atomicOr(bits + (v >> 5), 1u << (v & 31));
}

struct FillGeo {
  int n[3];
  int64_t s[3];
  const uint32_t* bits;  // flagged bitmap of planes [e0, e1) (the whole grid unless slab)
  int e0, e1;            // slab fill: planes held locally (own planes + halo)
  int* oob;              // slab fill: set when a search leaves [e0, e1)
};

__device__ __forceinline__ bool is_flagged(const FillGeo& g, const int* c) {
  if (c[0] < g.e0 || c[0] >= g.e1) {  // outside the halo: cannot decide here
    if (g.oob) atomicExch(g.oob, 1);
    return false;
  }
  const int64_t v = (c[0] - g.e0) * g.s[0] + c[1] * g.s[1] + c[2] * g.s[2];
  return (__ldg(g.bits + (v >> 5)) >> (v & 31)) & 1u;
}

// feature of node c after scipy's envelope pass along axis D (D = -1: the
// input features, i.e. the unflagged nodes themselves); false = no feature
template <int D>
__device__ bool fill_feature(const FillGeo& g, const int* c, int* f) {
  if (!is_flagged(g, c)) {
    f[0] = c[0], f[1] = c[1], f[2] = c[2];
    return true;
  }
  if constexpr (D < 0) {
    return false;
  } else {
    const int n = g.n[D], x0 = c[D];
    long long best = 0;
    int bx = 0;
    bool found = false;
    int q[3] = {c[0], c[1], c[2]}, fq[3];
    for (int t = 0;; ++t) {
      if (found && (long long)t * t > best) break;
      if (x0 - t < 0 && x0 + t >= n) break;
      for (int side = 0; side < (t ? 2 : 1); ++side) {
        const int x = side ? x0 + t : x0 - t;  // smaller position first
        if (x < 0 || x >= n) continue;
        q[D] = x;
        if (!fill_feature<D - 1>(g, q, fq)) continue;
        long long dist = 0;
        for (int a = 0; a < 3; ++a) {
          const long long d = fq[a] - c[a];
          dist += d * d;
        }
        if (!found || dist < best || (dist == best && x < bx)) {
          best = dist, bx = x, found = true;
          f[0] = fq[0], f[1] = fq[1], f[2] = fq[2];
        }
      }
    }
    return found;
  }
}

// per flagged node: FROM_MU = apply the rounding / threshold rule to mu at its
// feature (classify); otherwise copy the feature's already-classified mask
// entry (the pipeline's row epilogue classified every node by its own mu)
template <bool FROM_MU, class MaskT>
__global__ void fill_fix_kernel(const int64_t* nodes, int64_t K, int rank, FillGeo g, const double* mu, int mode,
                                int use_thr, double thr, MaskT* mask, const double* S, double* signed_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t v = nodes[i];
  int64_t N = (int64_t)g.n[0] * g.n[1] * g.n[2];
  if (v < 0 || v >= N) return;
  int c[3];
  c[0] = (int)(v / g.s[0]);
  c[1] = (int)((v / g.s[1]) % g.n[1]);
  c[2] = (int)(v % g.n[2]);
  int f[3];
  bool ok;
  if (rank == 1) ok = fill_feature<0>(g, c, f);
  else if (rank == 2) ok = fill_feature<1>(g, c, f);
  else ok = fill_feature<2>(g, c, f);
  if (!ok) return;  // every node flagged: rejected by the callers
  const int64_t src = (f[0] - g.e0) * g.s[0] + f[1] * g.s[1] + f[2] * g.s[2];
  if constexpr (FROM_MU) {
    const double m = mu[src];
    bool inside;
    if (use_thr) inside = m >= thr;
    else if (mode == 1) inside = rint(m) > 0.0;
    else inside = rint(m) >= 1.0;
    if (mask) mask[v] = inside ? MaskT(1) : MaskT(0);
    if (signed_out) signed_out[v] = inside ? S[v] : -S[v];
  } else {
    mask[v] = mask[src];
  }
}

// The search half of the sparse fill: src[i] = flat index of flagged node i's feature (its
// nearest unflagged node under scipy's tie rules), -1 when it has none.  Depends on the
// flagged bitmap only, so the pipeline runs it next to the column passes; the apply half
// (mask[node] = mask[src]) is all that is left after the row pass has classified the nodes.
__global__ void fill_search_kernel(const int64_t* nodes, int64_t K, int rank, FillGeo g, int64_t* src) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t v = nodes[i];
  const int64_t N = (int64_t)g.n[0] * g.n[1] * g.n[2];
  int64_t out = -1;
  if (v >= 0 && v < N) {
    int c[3];
    c[0] = (int)(v / g.s[0]);
    c[1] = (int)((v / g.s[1]) % g.n[1]);
    c[2] = (int)(v % g.n[2]);
    int f[3];
    bool ok;
    if (rank == 1) ok = fill_feature<0>(g, c, f);
    else if (rank == 2) ok = fill_feature<1>(g, c, f);
    else ok = fill_feature<2>(g, c, f);
    if (ok) out = (f[0] - g.e0) * g.s[0] + f[1] * g.s[1] + f[2] * g.s[2];
  }
  src[i] = out;
}
__global__ void fill_apply_kernel(const int64_t* nodes, const int64_t* src, int64_t K, uint8_t* mask) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t s = src[i];
  if (s >= 0) mask[nodes[i]] = mask[s];  // features are unflagged nodes: never written here
}

FillGeo fill_geo(int dim, const int64_t* counts, const uint32_t* bits, int* oob) {
  FillGeo g{};
  g.n[0] = g.n[1] = g.n[2] = 1;
  // rank-r grids use axes [0, r); unused trailing axes have length 1
  for (int a = 0; a < dim; ++a) g.n[a] = (int)counts[a];
  g.s[2] = 1;
  g.s[1] = g.n[2];
  g.s[0] = (int64_t)g.n[1] * g.n[2];
  g.bits = bits;
  g.e0 = 0;
  g.e1 = g.n[0];
  g.oob = oob;
  return g;
}

// slab fill: planes [e0, e1) of a 3-D grid are held (bits, mask); the nodes
// are flat indices relative to plane e0
__global__ void slab_fill_kernel(const int64_t* nodes, int64_t K, FillGeo g, int64_t own0, int64_t own1,
                                 const uint8_t* mask_ext, uint8_t* mask_own) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t v = nodes[i];  // relative to plane e0
  int c[3];
  c[0] = g.e0 + (int)(v / g.s[0]);
  if (c[0] < own0 || c[0] >= own1) return;  // halo nodes belong to the neighbours
  c[1] = (int)((v / g.s[1]) % g.n[1]);
  c[2] = (int)(v % g.n[2]);
  int f[3];
  if (!fill_feature<2>(g, c, f)) return;
  const int64_t src = (f[0] - g.e0) * g.s[0] + f[1] * g.s[1] + f[2] * g.s[2];
  mask_own[(c[0] - own0) * g.s[0] + c[1] * g.s[1] + c[2]] = mask_ext[src];
}

struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
};

// full separable feature transform of a flagged node list: fl (uint8 per node),
// F (features, dim x N int32) and the envelope scratch g are allocated here
int run_edt(int dim, const int64_t* n, const int64_t* d_idx, int64_t K, Buf& fl, Buf& F, Buf& g, int* err,
            cudaStream_t st) {
  const int64_t N = n[0] * n[1] * n[2];
  CKC(cudaMalloc(&fl.p, N));
  CKC(cudaMemsetAsync(fl.p, 0, N, st));
  flag_kernel<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(d_idx, K, N, (uint8_t*)fl.p, err);
  CKC(cudaGetLastError());
  CKC(cudaMalloc(&F.p, (size_t)dim * N * sizeof(int32_t)));
  edt_init_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>((const uint8_t*)fl.p, dim, n[1], n[2], N,
                                                              (int32_t*)F.p);
  CKC(cudaGetLastError());
  // per line: stack (len) + envelope feature copies (len * rank); nlines * len = N per phase
  CKC(cudaMalloc(&g.p, (size_t)N * (1 + dim) * sizeof(int32_t)));
  int64_t stride[3] = {1, 1, 1};
  for (int a = dim - 2; a >= 0; --a) stride[a] = stride[a + 1] * n[a + 1];
  for (int d = 0; d < dim; ++d) {
    EdtArgs ea{};
    ea.rank = dim;
    ea.d = d;
    for (int a = 0; a < 3; ++a) { ea.n[a] = n[a]; ea.stride[a] = stride[a]; }
    ea.F = (int32_t*)F.p;
    ea.g = (int32_t*)g.p;
    ea.N = N;
    ea.nlines = N / n[d];
    edt_lines_kernel<<<(unsigned)((ea.nlines + 127) / 128), 128, 0, st>>>(ea);
    CKC(cudaGetLastError());
  }
  return EIK_OK;
}

// dense fallback of the pipeline's fill: flagged mask entries copied from
// their features (full transform)
__global__ void fill_copy_dense_kernel(const int64_t* nodes, int64_t K, const int32_t* F, int rank, int64_t s0,
                                       int64_t s1, int64_t N, uint8_t* mask) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t v = nodes[i];
  if (v < 0 || v >= N || F[v] < 0) return;
  int64_t src;
  if (rank == 1) src = F[v];
  else if (rank == 2) src = (int64_t)F[v] * s0 + (int64_t)F[N + v];
  else src = (int64_t)F[v] * s0 + (int64_t)F[N + v] * s1 + (int64_t)F[2 * N + v];
  mask[v] = mask[src];
}

}  // namespace

// Pipeline hook (pipeline.cu): flagged-node bitmap of a sorted node list, then
// the per-node fill of an already classified uint8 mask.
int eik_fill_bits(const int64_t* d_nodes, int64_t K, int64_t N, uint32_t* bits, cudaStream_t st) {
  CKC(cudaMemsetAsync(bits, 0, ((N + 31) / 32) * sizeof(uint32_t), st));
  if (K > 0) fill_bits_kernel<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(d_nodes, K, N, bits, nullptr);
  CKC(cudaGetLastError());
  return EIK_OK;
}

// Sparse flagged sets only (the rule eik_fill_mask applies): true when the split fill is used
bool eik_fill_is_sparse(int dim, const int64_t* counts, int64_t K) {
  int64_t N = 1;
  for (int a = 0; a < dim; ++a) N *= counts[a];
  return K > 0 && K <= N / 8;
}
int eik_fill_search(int dim, const int64_t* counts, const int64_t* d_nodes, int64_t K, const uint32_t* bits,
                    int64_t* src, cudaStream_t st) {
  if (K <= 0) return EIK_OK;
  const FillGeo g = fill_geo(dim, counts, bits, nullptr);
  fill_search_kernel<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(d_nodes, K, dim, g, src);
  CKC(cudaGetLastError());
  return EIK_OK;
}
int eik_fill_apply(const int64_t* d_nodes, const int64_t* src, int64_t K, uint8_t* mask, cudaStream_t st) {
  if (K <= 0) return EIK_OK;
  fill_apply_kernel<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(d_nodes, src, K, mask);
  CKC(cudaGetLastError());
  return EIK_OK;
}

int eik_fill_mask(int dim, const int64_t* counts, const int64_t* d_nodes, int64_t K, const uint32_t* bits,
                  uint8_t* mask, cudaStream_t st) {
  if (K <= 0) return EIK_OK;
  int64_t n[3] = {1, 1, 1}, N = 1;
  for (int a = 0; a < dim; ++a) n[a] = counts[a], N *= counts[a];
  if (K > N / 8) {  // dense flagged set: full feature transform (temporaries; synchronous)
    Buf fl, F, g;
    int rc = run_edt(dim, n, d_nodes, K, fl, F, g, nullptr, st);
    if (rc) return rc;
    const int64_t s0 = dim == 3 ? n[1] * n[2] : (dim == 2 ? n[1] : 1), s1 = dim == 3 ? n[2] : 1;
    fill_copy_dense_kernel<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(d_nodes, K, (const int32_t*)F.p, dim, s0, s1,
                                                                        N, mask);
    CKC(cudaGetLastError());
    CKC(cudaStreamSynchronize(st));
    return EIK_OK;
  }
  const FillGeo g = fill_geo(dim, counts, bits, nullptr);
  fill_fix_kernel<false, uint8_t><<<(unsigned)((K + 127) / 128), 128, 0, st>>>(d_nodes, K, dim, g, nullptr, 0, 0, 0.0,
                                                                             mask, nullptr, nullptr);
  CKC(cudaGetLastError());
  return EIK_OK;
}

// Slab ranks (3-D, planes [own0, own0 + c0_local) of counts[0]): fill the own
// planes' flagged mask entries from a halo-extended copy of the mask, planes
// [e0, e1) (own planes plus the neighbours' halo planes).  ext_nodes: every
// flagged node of planes [e0, e1), flat relative to plane e0, device.
// Returns EIK_EVALIDATION when a nearest-unflagged search leaves [e0, e1)
// (the caller widens the halo).  Synchronous.
int eik_slab_fill_mask(const int64_t* counts, const int64_t* ext_nodes, int64_t K, int64_t e0, int64_t e1,
                       int64_t own0, int64_t c0_local, const uint8_t* mask_ext, uint8_t* mask_own, cudaStream_t st) {
  if (K <= 0) return EIK_OK;
  if (e0 < 0 || e1 > counts[0] || own0 < e0 || own0 + c0_local > e1)
    return eik_fail(EIK_EVALIDATION, "slab fill: halo planes do not cover the own planes");
  const int64_t plane = counts[1] * counts[2], n_ext = (e1 - e0) * plane;
  Buf bits, oob;
  CKC(cudaMalloc(&bits.p, ((n_ext + 31) / 32) * sizeof(uint32_t)));
  CKC(cudaMalloc(&oob.p, sizeof(int)));
  CKC(cudaMemsetAsync(oob.p, 0, sizeof(int), st));
  int rc = eik_fill_bits(ext_nodes, K, n_ext, (uint32_t*)bits.p, st);
  if (rc) return rc;
  const int64_t cnt[3] = {counts[0], counts[1], counts[2]};
  FillGeo g = fill_geo(3, cnt, (const uint32_t*)bits.p, (int*)oob.p);
  g.e0 = (int)e0;
  g.e1 = (int)e1;
  // searches may step outside [e0, e1) only where the grid itself continues
  slab_fill_kernel<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(ext_nodes, K, g, own0, own0 + c0_local, mask_ext,
                                                                mask_own);
  CKC(cudaGetLastError());
  int h_oob = 0;
  CKC(cudaMemcpyAsync(&h_oob, oob.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKC(cudaStreamSynchronize(st));
  if (h_oob) return eik_fail(EIK_EVALIDATION, "slab fill: nearest-unflagged search left the halo planes");
  return EIK_OK;
}

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
  // sparse flagged sets: classify every node by its own mu, then fix the
  // flagged ones per node (fill_fix_kernel); dense sets: full feature transform
  const bool sparse = n_flagged > 0 && n_flagged <= N / 8;
  if (sparse) {
    const int64_t nw = (N + 31) / 32;
    CKC(cudaMalloc(&b_fl.p, nw * sizeof(uint32_t)));
    CKC(cudaMemsetAsync(b_fl.p, 0, nw * sizeof(uint32_t), st));
    CKC(cudaMalloc(&b_err.p, sizeof(int)));
    CKC(cudaMemsetAsync(b_err.p, 0, sizeof(int), st));
    fill_bits_kernel<<<(unsigned)((n_flagged + 255) / 256), 256, 0, st>>>(d_idx, n_flagged, N, (uint32_t*)b_fl.p,
                                                                          (int*)b_err.p);
    CKC(cudaGetLastError());
    // every node flagged cannot pass n_flagged <= N / 8
  } else if (n_flagged > 0) {
    CKC(cudaMalloc(&b_err.p, sizeof(int)));
    CKC(cudaMemsetAsync(b_err.p, 0, sizeof(int), st));
    const int rc = run_edt(dim, n, d_idx, n_flagged, b_fl, b_F, b_g, (int*)b_err.p, st);
    if (rc) return rc;
    d_fl = (const uint8_t*)b_fl.p;
    d_F = (const int32_t*)b_F.p;
  }
  const int64_t s0 = dim == 3 ? n[1] * n[2] : (dim == 2 ? n[1] : 1), s1 = dim == 3 ? n[2] : 1;
  classify_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(d_mu, sparse ? nullptr : d_fl, d_F, dim, s0, s1, N,
                                                              mode, use_threshold, threshold, d_mask, d_S, d_sd);
  CKC(cudaGetLastError());
  if (sparse) {
    const FillGeo g = fill_geo(dim, n, (const uint32_t*)b_fl.p, (int*)b_err.p);
    fill_fix_kernel<true, double><<<(unsigned)((n_flagged + 127) / 128), 128, 0, st>>>(
        d_idx, n_flagged, dim, g, d_mu, mode, use_threshold, threshold, d_mask, d_S, d_sd);
    CKC(cudaGetLastError());
  }
  if (host) {
    if (out_mask) CKC(cudaMemcpyAsync(out_mask, d_mask, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (out_signed) CKC(cudaMemcpyAsync(out_signed, d_sd, N * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  if (b_err.p) CKC(cudaMemcpyAsync(&err, b_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKC(cudaStreamSynchronize(st));  // temporaries are freed on return
  if (err) return eik_fail(EIK_EVALIDATION, "flagged node index out of grid bounds");
  return EIK_OK;
}
