// Device kernels of the FFT-convolution distance transform (sm_100a, fp64).
//
// Pipeline (2D, grid c0 x c1, padded M0 x M1, half spectrum H1 = M1/2+1):
//   prep_nodes / rowptr   sorted node list -> per-row CSR (deterministic)
//   col_kernel<SPARSE>    per spectral column k1: impulse DFT along axis 1
//                         straight from the node list (delta_Y never exists
//                         in memory), forward FFT along axis 0, multiply by
//                         the cached kernel spectra, one inverse FFT per
//                         output component, keep rows [0,c0)          (K1-K5)
//   row_kernel            per grid row: c2r along axis 1 (half-length
//                         complex IFFT) fused with the epilogue
//                         S=-tau log phi, S_a=num/phi, Hessian, mu, sign,
//                         underflow flag/count                        (K5-K6)
// 3D adds a plane pass (impulse DFT along axis 2 + FFT along axis 1, stored),
// runs col_kernel<DENSE> along axis 0, and an inverse lines pass along axis 1
// before the row kernel.  Kernel spectra are produced once per plan by
// row_r2c_kernel + lines_kernel + col_kernel<DENSE, SPECTRUM> (K3).
//
// Thread mappings: "column" kernels (col/lines) are line-minor
// (line = tid % LPC) so that a warp touches LPC adjacent lines at the same
// element: every global access is a contiguous run across lines.  Row
// kernels are line-major (a row is contiguous in memory).
#pragma once
#include <cuda.h>  // CUtensorMap (TMA stores of the column outputs)

#include "fft_core.cuh"
#include "tmem.cuh"
#include "bulk.cuh"

#include <type_traits>

namespace eik {

constexpr int MAXC = 8;
constexpr int MAXG = 8;  // ranks of a peer-to-peer slab exchange

enum { IN_SPARSE = 0, IN_DENSE = 1 };
enum { OUT_COMPS = 0, OUT_SUM = 1, OUT_SPECTRUM = 2 };
enum { SPEC_COMPLEX = 0, SPEC_REAL_T = 1, SPEC_IMAG_T = 2, SPEC_COMPLEX_T = 3 };

// Launch shapes.  Column kernels (col/lines): lines of length 2^L, E elements
// per thread, NT threads, LPC lines per CTA, then the line buffers and a
// quarter twiddle table of the line length in dynamic shared memory.  Long
// lines use E = 8 so the forward result and the per-component product both
// stay in registers without spilling at 512 threads.
#ifndef EIK_COL_E_LARGE
#define EIK_COL_E_LARGE 8
#endif
__host__ __device__ constexpr int col_e(int L) { return (L >= 10 && L <= 12) ? EIK_COL_E_LARGE : 16; }
__host__ __device__ constexpr int col_threads(int L) { return L >= 10 ? 512 : 256; }
// Exchange-buffer padding per launch shape, packed as PA | PB << 4 | XT << 8
// (see Line): the bank-conflict-free choices of tools/bank_sim.py for the
// column mapping (line = tid % LPC: col, lines and TMEM kernels) and the row
// mapping (line = tid / TPL).  Shapes not listed are conflict-free already.
__host__ __device__ constexpr int pad_code(int pa, int pb, int xt) { return pa | (pb << 4) | (xt << 8); }
constexpr int PAD_DEFAULT = 3 | (0 << 4) | (2 << 8);
// Column-type kernels interleave the LPC lines of a CTA across its threads
// (line = tid % LPC under __syncthreads), so one warp load/store covers LPC
// adjacent columns of only 32/LPC rows: few 128-byte lines per request.
// EIK_COL_IL = IL < LPC interleaves groups of IL lines over IL*TPL threads,
// each group with its own (warp / named) barrier.  Measured slower: C3 column
// pass 1.88 ms (IL = LPC) vs 2.51 (IL = 2) vs 3.52 (IL = 1, line-major),
// C5 6.98 vs 7.33 vs 7.78 ms; the cache lines touched per warp request cost
// more than the narrower barriers save.
#ifndef EIK_COL_IL
#define EIK_COL_IL 0
#endif
__host__ __device__ constexpr int col_il(int lpc) { return (EIK_COL_IL == 0 || EIK_COL_IL >= lpc) ? lpc : EIK_COL_IL; }
__host__ __device__ constexpr int tpl_of(int L, int E) { return (1 << L) <= E ? 1 : (1 << L) / E; }
// line-major (row) mapping, E = 16 lines, by L (tools/bank_sim.py, mapping "row")
__host__ __device__ constexpr int lm_pad16(int L) {
  return L == 5 ? pad_code(4, 0, 1) : L == 6 ? pad_code(2, 4, 2) : L == 7 ? pad_code(3, 6, 0)
       : L == 8 ? pad_code(4, 0, 0) : L == 9 ? pad_code(3, 4, 0) : L == 10 ? pad_code(4, 0, 0)
       : L == 11 ? pad_code(3, 6, 0) : L == 12 ? pad_code(4, 0, 0) : L == 13 ? pad_code(3, 4, 0) : PAD_DEFAULT;
}
// pair-interleaved (IL = 2 < LPC) pads
__host__ __device__ constexpr int il2_pad(int L, int E) {
  return E == 8 ? (L == 10 ? pad_code(2, 3, 6) : PAD_DEFAULT)
       : L == 7 ? pad_code(3, 5, 2) : L == 8 ? pad_code(4, 0, 5) : (L == 9 || L == 10) ? pad_code(2, 4, 6)
       : PAD_DEFAULT;
}
__host__ __device__ constexpr int col_pad(int L, bool pair) {
  return pair ? il2_pad(L, col_e(L))
       : col_e(L) == 16 ? (L == 13 ? pad_code(3, 4, 0) : PAD_DEFAULT)
       : (L == 10) ? pad_code(3, 0, 3) : (L == 11) ? pad_code(2, 4, 6) : PAD_DEFAULT;
}
// threads per CTA of the TMEM column kernel of 2048-point lines: 256 = two lines per CTA, two
// CTAs per SM (32-byte runs per row); 512 = four lines, one CTA per SM (64-byte runs)
// (measured at 1024^3 with line-major spectra: 914 ms per step at 256, 789 ms at 512).  The
// 3-D instantiations (TmCfg<.., WIDE = true>, selected with the line-major spectra) always run
// 512 threads for 1024- and 2048-point lines: 8 / 4 lines per CTA, 128- / 64-byte runs per row
// of arrays whose rows lie tens of MB apart; the 2-D kernels keep two 256-thread CTAs per SM.
#ifndef EIK_TM11_NT
#define EIK_TM11_NT 256
#endif
#ifndef EIK_TM10_NT
#define EIK_TM10_NT 256  // A/B: 512 = 8 lines per CTA for the 2-D 1024-point column kernels too
#endif
#ifndef EIK_TM9_NT
#define EIK_TM9_NT 256  // A/B: 512 = 16 lines per CTA for 512-point lines
#endif
__host__ __device__ constexpr int tm_pad(int L, bool pair, bool wide = false) {
  return pair ? il2_pad(L, 16)
       : L == 10 ? ((wide || EIK_TM10_NT == 512) ? pad_code(2, 0, 0) : pad_code(2, 4, 0))
       : L == 11 ? ((wide || EIK_TM11_NT == 512) ? pad_code(3, 4, 0) : pad_code(3, 5, 6))
       : L == 12 ? pad_code(4, 0, 0)
       : L == 13 ? pad_code(3, 4, 0) : PAD_DEFAULT;
}
__host__ __device__ constexpr int row_pad(int LH) {
  return LH == 5 ? pad_code(4, 0, 1) : LH == 6 ? pad_code(2, 4, 2) : LH == 7 ? pad_code(3, 6, 0)
       : LH == 8 ? pad_code(4, 0, 0) : PAD_DEFAULT;
}
// barrier covering one group of il interleaved lines (see XBuf)
__host__ __device__ constexpr int group_sync(int il, int lpc, int tpl) {
  return il >= lpc ? 0 : il * tpl <= 32 ? 1 : 2;
}
template <int L, int E, int CODE>
using PaddedLine = Line<L, E, (CODE & 15), ((CODE >> 4) & 15), (CODE >> 8)>;

template <int L>
struct ColCfg {
  static constexpr int TPL0 = tpl_of(L, col_e(L));
  static constexpr int NT = (col_threads(L) > TPL0) ? col_threads(L) : TPL0;
  static constexpr int LPC = NT / TPL0;
  static constexpr int IL = col_il(LPC);
  static constexpr bool PFOLD = false;  // register-order spectra unfolded (see TmCfg::PFOLD)
  static constexpr int NTP = NT;
  using LN = PaddedLine<L, col_e(L), col_pad(L, IL == 2 && LPC > 2)>;
  __device__ static __forceinline__ int line_of(int tid) { return (tid / (IL * TPL0)) * IL + tid % IL; }
  __device__ static __forceinline__ int t_of(int tid) { return (tid % (IL * TPL0)) / IL; }
  static constexpr int M0 = 1 << L;  // transform length the register-order spectrum copy indexes
  __device__ static __forceinline__ int k0_of(int tid, int r) { return LN::out_idx(t_of(tid), r); }
  // ping-pong exchange buffers (one barrier per exchange instead of two) where
  // they were measured to pay off without costing occupancy (C5-sized lines)
  static constexpr int NBUF = ((L == 10 || L == 11) && (2 * LPC * LN::SMEM + LN::TWQ) * 16 <= 200 * 1024) ? 2 : 1;
  using XB = XBuf<NBUF, group_sync(IL, LPC, TPL0), IL * TPL0, false>;
  static constexpr size_t MB_OFF = ((size_t)NBUF * LPC * LN::SMEM + LN::TWQ + LN::ST_SIZE) * sizeof(double2);
  static constexpr size_t SMEM_BYTES = MB_OFF + 128;  // + the split-phase exchange mbarriers
};
// Row kernels (c2r / r2c along the contiguous last axis): complex lines of
// length 2^LH = M_last/2, quarter table at the resolution of M_last.
#ifndef EIK_ROW_E8_MIN
#define EIK_ROW_E8_MIN 7
#endif
__host__ __device__ constexpr int row_e(int LH) { return LH >= EIK_ROW_E8_MIN ? 8 : 16; }
#ifndef EIK_ROW_NBUF2_MAX
#define EIK_ROW_NBUF2_MAX 10
#endif
#ifndef EIK_ROW_FEED
#define EIK_ROW_FEED 1
#endif
// rows of >= 64 threads per line get the TMA row feed (C5 512-point rows:
// 3.69 -> 3.30 ms, trading the ping-pong buffers; C3's 32-thread rows: +12%)
#ifndef EIK_ROW_FEED_MINTPL
#define EIK_ROW_FEED_MINTPL 64
#endif
template <int LH>
struct RowCfg {
  using LN = PaddedLine<LH, row_e(LH), row_pad(LH)>;
  static constexpr int NT = (LN::TPL >= 128) ? LN::TPL : 128;
  static constexpr int LPC = NT / LN::TPL;
  static constexpr int TWQ = tpos_size(1 << (LH > 0 ? LH - 1 : 0));  // (2^(LH+1)) / 4, padded
  // (with EIK_ROW_FEED_MINTPL < 128, multi-line CTAs give up the ping-pong
  // buffers for the row feed where both do not fit next to 4 CTAs)
  static constexpr bool FEED_WANT = EIK_ROW_FEED && LN::TPL >= EIK_ROW_FEED_MINTPL;
  static constexpr int NBUF = (LH <= EIK_ROW_NBUF2_MAX && (2 * LPC * LN::SMEM + TWQ) * 16 <= 110 * 1024 &&
                               !(FEED_WANT && LN::TPL < 128 &&
                                 ((2 * LPC * LN::SMEM + TWQ + LN::ST_SIZE) * 16 + LPC * (LN::M + 1) * 16 + 32) * 4 >
                                     227 * 1024))
                                  ? 2
                                  : 1;
  using XB = XBuf<NBUF, group_sync(1, LPC, LN::TPL), LN::TPL>;  // row kernels are line-major
  static constexpr size_t BASE_BYTES = ((size_t)NBUF * LPC * LN::SMEM + TWQ + LN::ST_SIZE) * sizeof(double2);
  // resident CTAs per SM requested from the register allocator (128 threads:
  // 4 CTAs = 16 warps at <= 128 registers)
#ifndef EIK_ROW_MINB128
#define EIK_ROW_MINB128 4
#endif
  static constexpr int MINB = (NT <= 128 && LN::EPT <= 8) ? EIK_ROW_MINB128 : (NT <= 256 ? 2 : 1);
  // Row prefetch: each line's next spectral row (M/2+1 complex values,
  // contiguous) is bulk-copied into shared memory while the current one is
  // transformed, where it fits next to MINB resident CTAs.
#ifndef EIK_ROW_FEED
#define EIK_ROW_FEED 1
#endif
  static constexpr size_t FEED_BYTES = (size_t)LPC * (LN::M + 1) * sizeof(double2) + LPC * sizeof(uint64_t);
  static constexpr bool FEED = FEED_WANT && (BASE_BYTES + FEED_BYTES + 16) * MINB <= 227 * 1024;
  static constexpr size_t MB_OFF = (BASE_BYTES + (FEED ? FEED_BYTES + 16 : 0) + 15) & ~size_t(15);
  static constexpr size_t SMEM_BYTES = MB_OFF + 128;  // + the split-phase exchange mbarriers
};

// Kernel spectrum reference.  Real/imaginary spectra are stored transposed and
// folded along axis 0: re[k0 * ld + l], k0 in [0, M0/2]; K(M0-k0) = (odd0 ? -1 : 1) * K(k0).
// General complex spectra (arbitrary user kernels): cplx[k0 * ld + l], k0 in [0, M0).
struct KSpec {
  const double* re;
  const double2* cplx;
  int64_t ld;
  int imag;
  int odd0;
  int odd1;  // 3-D: odd along axis 1 (sign of the k1-mirrored lines, see ColArgs::fold_H)
  // Line-major storage (3-D plans): ls > 0 means re[l * ls + k0] (one contiguous run of
  // M0/2 + 1 values per spectral line, ls >= M0/2 + 1), so a column kernel's warp reads
  // consecutive k0 of its lines as whole cache lines; ls == 0 is re[k0 * ld + l].  (At
  // 1024^3 the k0-major layout cost 16 useful bytes per 64-byte DRAM burst: 249 GB read per
  // axis-0 pass against 43 GB needed, profiles/round2/c4prof.)
  int64_t ls;
  // Optional register-order copy (real/imaginary spectra, 2-D plans): the value
  // register r of thread tid of CTA tile b needs, at perm[(b * EPT + r) * NT + tid],
  // unfolded with the axis-0 parity sign applied.  Warp loads are contiguous
  // (a column kernel otherwise touches one cache line per lane).  When set,
  // odd0 is 0 (the sign is baked in).
  const double* perm;
};

struct ColArgs {
  int64_t nlines;  // spectral lines per item
  int n_valid;     // non-zero input elements per line
  int n_out;       // outputs kept per line (inverse)
  int n_in, n_comp;
  // sparse impulse input (rows of the transform axis; last-axis coordinate + weights)
  const int64_t* rowptr;
  const int32_t* cols;
  const double* w[3];
  int64_t rows_per_item;
  int last_shift;  // lmax - log2(M_last)
  int last_mask;   // M_last - 1
  // dense input din[i][item*din_item + e*din_es + l]
  const double2* din[3];
  int64_t din_es, din_item;
  int64_t din_ls;  // line stride of the dense input (1: lines are adjacent columns)
  // kernel spectra (COMPS: one per component; SUM: one per input)
  KSpec ks[MAXC];
  // outputs out[j][item*out_item + n*out_es + l]
  double2* out[MAXC];
  int64_t out_es, out_item;
  // spectrum extraction (OUT_SPECTRUM); SPEC_COMPLEX rows k are split as
  // (k >> out_split_shift) * out_split_stride + (k & (2^shift - 1)) * out_es
  // (slab packing; shift 30 = no split)
  int out_split_shift;
  int64_t out_split_stride;
  int spec_mode;
  double* spec_re[3];
  int64_t spec_ld;
  int64_t spec_ls;  // > 0: line-major real / imaginary spectrum, spec_re[l * spec_ls + k0] (KSpec::ls)
  const double2* tw;
  int lmax;
  // persistent TMEM column kernels (set by the launcher): tiles of LPC lines per item, items
  int64_t tiles, items;
  // 3-D kernel spectra are stored folded along axis 1 (every kernel is even or
  // odd there): line l = (k1 - fold_k1base) * fold_H + k2 of the pass reads the
  // stored line (min(k1, M1 - k1) - fold_f0) * fold_H + k2, negated for odd
  // kernels when k1 > M1/2.  fold_H = 0: lines are read as they are (2-D).
  int fold_H, fold_M1;
  int64_t fold_k1base, fold_f0;
  // TMA output stores (4096-point four-step kernels, set by the launcher): component j
  // leaves through a shared-memory tile [row][LPC lines] as boxes of 2*LPC doubles x 256
  // rows of umap[j], a [item][row][2 * nlines doubles] view of out[j]
  int tstore;
  CUtensorMap umap[MAXC];
  // OUT_COMPS: add the component into its destination instead of overwriting it
  // (streamed 3-D sign group: one flux input at a time, W += IFFT0(K_i FFT0(V_i)))
  int accum;
  // Peer-block outputs (slab exchange fused into the pass, P2P over NVLink):
  // when blk[0] is set, output row n of component j is written to
  // blk[n >> blk_shift] + j * blk_cstride + item * out_item + (n mod 2^blk_shift) * out_es + l,
  // i.e. straight into the receive buffer of the rank that owns row n.
  double2* blk[MAXG];
  int blk_shift;
  int64_t blk_cstride;
};


// Split-phase exchange barriers (XBuf::acquire / release): mbarrier `group` of the
// CTA's block at mbs, one per sync group; call before the kernel's first __syncthreads().
template <class XB>
__device__ __forceinline__ void xb_setup(XB& xb, uint64_t* mbs, int group, int ngroups, int cta_threads) {
  xb.mb = mbs + group;
  xb.par = 0u;
  if constexpr (XB::SPLIT) {
    if ((int)threadIdx.x < ngroups) mbar_init(mbs + threadIdx.x, (uint32_t)XB::group_warps(cta_threads));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
}
constexpr size_t XB_MBAR_BYTES = 128;  // up to 16 sync groups per CTA

// Streaming (evict-first) stores for data written once and read by a later
// kernel (EIK_CS: 1 = component spectra U_j of the TMEM column kernels, 2 = also
// the row pass's outputs)
#ifndef EIK_CS
#define EIK_CS 0
#endif
__device__ __forceinline__ void store_u(double2* dst, double2 x) {
  if constexpr (EIK_CS >= 1) __stcs(dst, x);
  else *dst = x;
}

// Destination of output row n of component j (own buffer or a peer's block).
__device__ __forceinline__ double2* comp_dst(const ColArgs& a, int j, int64_t item, int64_t l, int n) {
  if (a.blk[0])
    return a.blk[n >> a.blk_shift] + j * a.blk_cstride + item * a.out_item +
           (int64_t)(n & ((1 << a.blk_shift) - 1)) * a.out_es + l;
  return a.out[j] + item * a.out_item + (int64_t)n * a.out_es + l;
}

__device__ __forceinline__ double2 kmul(double2 x, const KSpec& k, int64_t l, int k0, int M0) {
  if (k.cplx) return cmul(x, __ldg(k.cplx + (int64_t)k0 * k.ld + l));
  const int half = M0 >> 1;
  const bool hi = k0 > half;
  double v = __ldg(k.re + (int64_t)(hi ? M0 - k0 : k0) * k.ld + l);
  if (hi && k.odd0) v = -v;
  return k.imag ? make_double2(-x.y * v, x.x * v) : make_double2(x.x * v, x.y * v);
}

// Stored kernel-spectrum line of pass line l (ColArgs::fold_H) and whether it is a k1 mirror.
__device__ __forceinline__ int64_t fold_line(const ColArgs& a, int64_t l, bool& mir) {
  mir = false;
  if (!a.fold_H) return l;
  const int64_t q = l / a.fold_H;
  const int64_t k1 = a.fold_k1base + q;
  mir = k1 > (a.fold_M1 >> 1);
  return ((mir ? a.fold_M1 - k1 : k1) - a.fold_f0) * a.fold_H + (l - q * a.fold_H);
}

// Raw folded kernel spectrum value at (k0, l); the fold sign is applied at use
// time (kapply) so a prefetch issued one FFT ahead does not stall on the load.
template <bool LM = false>
__device__ __forceinline__ double kload(const KSpec& k, int64_t l, int k0, int M0) {
  const bool hi = k0 > (M0 >> 1);
  if constexpr (LM) return __ldg(k.re + l * k.ls + (hi ? M0 - k0 : k0));
  else return __ldg(k.re + (int64_t)(hi ? M0 - k0 : k0) * k.ld + l);
}
// All EPT kernel-spectrum values of this thread for a kernel of configuration
// CFG (one uniform branch on the layout, outside the unrolled loads).
// Column of the register-order spectrum copy this thread reads (and whether in
// reversed register order): itself, or its mirror thread under CFG::PFOLD.
template <class CFG>
__device__ __forceinline__ void perm_thread(int& tc, int& rev) {
  tc = threadIdx.x;
  rev = 0;
  if constexpr (CFG::PFOLD) {
    if (tc >= CFG::NTP) {
      const int t = tc >> 1, line = tc & 1, a = t >> 4, b = t & 15;
      tc = 2 * (((16 - a) << 4) | (15 - b)) + line;
      rev = 1;
    }
  }
}
// LM: line-major storage (KSpec::ls), a compile-time property of the 3-D instantiations so
// that the 2-D kernels' code is untouched (a run-time layout select in the unrolled loads
// cost C3's column kernel 16% and C2's 3%)
template <class CFG, bool LM = false>
__device__ __forceinline__ void kload_all(double (&kn)[CFG::LN::EPT], const KSpec& k, int64_t l, int t, int64_t bx) {
  using LN = typename CFG::LN;
  if (!LM && k.perm) {
    int tc, rev;
    perm_thread<CFG>(tc, rev);
    const double* __restrict__ src = k.perm + bx * LN::EPT * CFG::NTP + tc;
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) kn[r] = __ldg(src + (rev ? LN::EPT - 1 - r : r) * CFG::NTP);
  } else {
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) kn[r] = kload<LM>(k, l, LN::out_idx(t, r), LN::M);
  }
}
// Register-resident column kernel (the EIK_TMEM=0 fallback): the layout is a uniform run-time
// branch, and only for the line lengths whose 3-D plans store line-major spectra.
template <class CFG>
__device__ __forceinline__ void kload_rt(double (&kn)[CFG::LN::EPT], const KSpec& k, int64_t l, int t, int64_t bx) {
  if constexpr (CFG::LN::L >= 10) {
    if (k.ls) {
      kload_all<CFG, true>(kn, k, l, t, bx);
      return;
    }
  }
  kload_all<CFG, false>(kn, k, l, t, bx);
}
// L1 prefetch of this thread's EPT kernel-spectrum values (TMEM column kernel).
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
template <class CFG, bool LM = false>
__device__ __forceinline__ void kprefetch_all(const KSpec& k, int64_t l, int t, int64_t bx) {
  using LN = typename CFG::LN;
  if (!LM && k.perm) {
    int tc, rev;
    perm_thread<CFG>(tc, rev);
    const double* src = k.perm + bx * LN::EPT * CFG::NTP + tc;
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) prefetch_l1(src + r * CFG::NTP);
  } else {
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) {
      const int k0 = LN::out_idx(t, r);
      const bool hi = k0 > (LN::M >> 1);
      const int kf = hi ? LN::M - k0 : k0;
      if constexpr (LM) {
        if ((kf & 15) == 0) prefetch_l1(k.re + l * k.ls + kf);  // one request per 128-byte run
      } else {
        prefetch_l1(k.re + (int64_t)kf * k.ld + l);
      }
    }
  }
}
// v[r] *= K (all EPT registers of this thread): the real / imaginary and fold-
// sign cases are uniform per kernel, so they are branched on once, not selected
// per element.
template <class LN>
__device__ __forceinline__ void kapply_all(double2 (&v)[LN::EPT], double (&kv)[LN::EPT], const KSpec& k, int t,
                                           bool mir = false) {
  if (k.odd1 && mir) {
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) kv[r] = -kv[r];
  }
  if (k.odd0) {
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r)
      if (LN::out_idx(t, r) > (LN::M >> 1)) kv[r] = -kv[r];
  }
  if (k.imag) {
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) v[r] = make_double2(-v[r].y * kv[r], v[r].x * kv[r]);
  } else {
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) v[r] = make_double2(v[r].x * kv[r], v[r].y * kv[r]);
  }
}
__device__ __forceinline__ double2 kapply(double2 x, double v, const KSpec& k, int k0, int M0, bool mir = false) {
  if ((k.odd0 && k0 > (M0 >> 1)) != (k.odd1 && mir)) v = -v;
  return k.imag ? make_double2(-x.y * v, x.x * v) : make_double2(x.x * v, x.y * v);
}

// Impulse DFT along the last axis straight from the per-row node lists:
// v[e] = sum_{p in row e} w_p W_{M_last}^{col_p * l}; each row accumulates its
// points in list order (bit-reproducible).  Row bounds for all registers are
// loaded first so their L2 latencies overlap.
constexpr size_t SPARSE_SMEM = 0;
template <class LN, bool HALF>
__device__ __forceinline__ void load_sparse(double2 (&v)[LN::EPT], const ColArgs& a, int t, int64_t l,
                                            int64_t item, int inp, bool valid, const double2* twq) {
  // W_{M_last}^{col*l}: from the shared quarter table when M_last <= M0, else global
  const int llast = a.lmax - a.last_shift;
  const bool shared_tw = llast <= LN::L && LN::L >= 2;
  const int up = LN::L - llast;
  const double* __restrict__ w = a.w[inp];
  const int64_t row0 = item * a.rows_per_item;
  int64_t lo[LN::EPT], hi[LN::EPT];
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    lo[r] = hi[r] = 0;
    if (HALF && LN::L > 0 && LN::upper_in(r)) continue;
    const int e = LN::in_idx(t, r);
    if (valid && e < a.n_valid) {
      lo[r] = __ldg(a.rowptr + row0 + e);
      hi[r] = __ldg(a.rowptr + row0 + e + 1);
    }
  }
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    double2 acc = make_double2(0.0, 0.0);
    if (!(HALF && LN::L > 0 && LN::upper_in(r))) {
      for (int64_t p = lo[r]; p < hi[r]; ++p) {
        const int j = (int)(((int64_t)__ldg(a.cols + p) * l) & a.last_mask);
        const double2 tw = shared_tw ? twq_get(twq, LN::L, j << up) : __ldg(a.tw + (j << a.last_shift));
        const double wt = w ? __ldg(w + p) : 1.0;
        acc.x = fma(wt, tw.x, acc.x);
        acc.y = fma(wt, tw.y, acc.y);
      }
    }
    v[r] = acc;
  }
}

template <class LN, bool HALF>
__device__ __forceinline__ void load_dense(double2 (&v)[LN::EPT], const ColArgs& a, int t, int64_t l,
                                           int64_t item, int inp, bool valid) {
  const double2* __restrict__ src = a.din[inp] + item * a.din_item + l * a.din_ls;
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    if (HALF && LN::L > 0 && LN::upper_in(r)) continue;
    const int e = LN::in_idx(t, r);
    v[r] = (valid && e < a.n_valid) ? src[(int64_t)e * a.din_es] : make_double2(0.0, 0.0);
  }
}

// L2 prefetch of this thread's part of a dense input line (no registers held)
template <class LN, bool HALF>
__device__ __forceinline__ void prefetch_dense_l2(const ColArgs& a, int t, int64_t l, int64_t item, int inp,
                                                  bool valid) {
  if (!valid) return;
  const double2* __restrict__ src = a.din[inp] + item * a.din_item + l * a.din_ls;
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    if (HALF && LN::L > 0 && LN::upper_in(r)) continue;
    const int e = LN::in_idx(t, r);
    if (e < a.n_valid) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + (int64_t)e * a.din_es));
  }
}

// Fused axis-0 column kernel.  blockIdx.x: tile of LPC lines, blockIdx.y: item.
template <int L, int IN, int OUT, bool HALF>
__global__ void __launch_bounds__(ColCfg<L>::NT) col_kernel(const __grid_constant__ ColArgs a) {
  using LN = typename ColCfg<L>::LN;
  constexpr int LPC = ColCfg<L>::LPC;
  extern __shared__ double2 smem[];
  const int line = ColCfg<L>::line_of(threadIdx.x);
  const int t = ColCfg<L>::t_of(threadIdx.x);
  const int64_t l = (int64_t)blockIdx.x * LPC + line;
  const bool valid = l < a.nlines;
  const int64_t item = blockIdx.y;
  using CC = ColCfg<L>;
  typename CC::XB xb{smem + line * LN::SMEM, smem + (LPC + line) * LN::SMEM, 0, 1 + line / CC::IL};
  double2* twq = smem + CC::NBUF * LPC * LN::SMEM;
  double2* sts = twq + LN::TWQ;
  xb_setup(xb, reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + CC::MB_OFF), line / CC::IL, LPC / CC::IL,
           CC::NT);
  if constexpr (L >= 2) twq_fill(twq, L, a.tw, a.lmax);
  st_fill<LN>(sts, a.tw, a.lmax);
  __syncthreads();
  const TwSrc tws{sts, twq, L, 0u};

  double2 v[LN::EPT];
  if constexpr (OUT == OUT_COMPS) {
    if constexpr (IN == IN_SPARSE) load_sparse<LN, HALF>(v, a, t, l, item, 0, valid, twq);
    else load_dense<LN, HALF>(v, a, t, l, item, 0, valid);
    fft_line<LN, false, HALF>(v, t, xb, tws);
    const bool real_ks = a.ks[0].cplx == nullptr;
    bool mir;
    const int64_t lk = fold_line(a, l, mir);
    double kn[LN::EPT];  // next component's kernel spectrum, prefetched
    if (real_ks && valid) {
      kload_rt<ColCfg<L>>(kn, a.ks[0], lk, t, blockIdx.x);
    }
#pragma unroll 1
    for (int j = 0; j < a.n_comp; ++j) {
      double2 y[LN::EPT];
      if (real_ks) {
#pragma unroll
        for (int r = 0; r < LN::EPT; ++r)
          y[r] = valid ? kapply(v[r], kn[r], a.ks[j], LN::out_idx(t, r), LN::M, mir) : v[r];
        if (j + 1 < a.n_comp && valid) {
          kload_rt<ColCfg<L>>(kn, a.ks[j + 1], lk, t, blockIdx.x);
        }
      } else {
#pragma unroll
        for (int r = 0; r < LN::EPT; ++r) y[r] = valid ? kmul(v[r], a.ks[j], l, LN::out_idx(t, r), LN::M) : v[r];
      }
      fft_line<LN, true>(y, t, xb, tws);
#pragma unroll
      for (int r = 0; r < LN::EPT; ++r) {
        if (LN::L > 0 && LN::upper_in(r)) continue;
        const int n = LN::in_idx(t, r);
        if (valid && n < a.n_out) {
          double2* dst = comp_dst(a, j, item, l, n);
          if (a.accum) *dst = cadd(*dst, y[r]);
          else *dst = y[r];
        }
      }
    }
  } else if constexpr (OUT == OUT_SUM) {
    double2 y[LN::EPT];
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) y[r] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int i = 0; i < a.n_in; ++i) {
      const bool real_ks = a.ks[i].cplx == nullptr;
      bool mir;
      const int64_t lk = fold_line(a, l, mir);
      double kn[LN::EPT];  // this input's kernel spectrum, loaded before its transform
      if (real_ks && valid) {
        kload_rt<ColCfg<L>>(kn, a.ks[i], lk, t, blockIdx.x);
      }
      if constexpr (IN == IN_SPARSE) load_sparse<LN, HALF>(v, a, t, l, item, i, valid, twq);
      else load_dense<LN, HALF>(v, a, t, l, item, i, valid);
      fft_line<LN, false, HALF>(v, t, xb, tws);
      if (valid) {
#pragma unroll
        for (int r = 0; r < LN::EPT; ++r)
          y[r] = cadd(y[r], real_ks ? kapply(v[r], kn[r], a.ks[i], LN::out_idx(t, r), LN::M, mir)
                                    : kmul(v[r], a.ks[i], l, LN::out_idx(t, r), LN::M));
      }
    }
    fft_line<LN, true>(y, t, xb, tws);
#pragma unroll
    for (int r = 0; r < LN::EPT; ++r) {
      if (LN::L > 0 && LN::upper_in(r)) continue;
      const int n = LN::in_idx(t, r);
      if (valid && n < a.n_out) *comp_dst(a, 0, item, l, n) = y[r];
    }
  } else {  // OUT_SPECTRUM
#pragma unroll 1
    for (int i = 0; i < a.n_in; ++i) {
      if constexpr (IN == IN_SPARSE) load_sparse<LN, HALF>(v, a, t, l, item, i, valid, twq);
      else load_dense<LN, HALF>(v, a, t, l, item, i, valid);
      fft_line<LN, false, HALF>(v, t, xb, tws);
      if (!valid) continue;
#pragma unroll
      for (int r = 0; r < LN::EPT; ++r) {
        const int k0 = LN::out_idx(t, r);
        if (a.spec_mode == SPEC_COMPLEX) {
          a.out[i][item * a.out_item + (int64_t)(k0 >> a.out_split_shift) * a.out_split_stride +
                   (int64_t)(k0 & ((1 << a.out_split_shift) - 1)) * a.out_es + l] = v[r];
        } else if (a.spec_mode == SPEC_COMPLEX_T) {
          a.out[i][(int64_t)k0 * a.spec_ld + l] = v[r];
        } else if (k0 <= (LN::M >> 1)) {
          const double part = (a.spec_mode == SPEC_REAL_T) ? v[r].x : v[r].y;
          if (a.spec_ls) a.spec_re[i][l * a.spec_ls + k0] = part;
          else a.spec_re[i][(int64_t)k0 * a.spec_ld + l] = part;
        }
      }
    }
  }
}

// Column pass, distance group, with the forward spectrum parked in TMEM.
// Same arithmetic as col_kernel<L, IN, OUT_COMPS, HALF> (bit-identical
// results); E = 16, 256+ threads, two CTAs per SM.
#ifndef EIK_FOUR_STEP
#define EIK_FOUR_STEP 1
#endif
#ifndef EIK_F4K_LPC
#define EIK_F4K_LPC 2
#endif
// Four-step 4096-point lines of the multi-component (COMPS) kernel: EIK_F4K_LPC
// lines per CTA, interleaved by lane parity, so warp loads/stores cover two
// adjacent columns (one CTA per SM).  The SUM kernel (sign group: two forward
// transforms, one inverse) does the same (measured 186 -> 180 us at C2: its
// T reads become whole 32-byte sectors).
#ifndef EIK_F4K_LPC_SUM
#define EIK_F4K_LPC_SUM 2
#endif
__host__ __device__ constexpr int tm_lpcx(int L, int OUT) {
  return (L == 12 && EIK_FOUR_STEP) ? (OUT == OUT_COMPS ? EIK_F4K_LPC : OUT == OUT_SUM ? EIK_F4K_LPC_SUM : 1) : 1;
}
#ifndef EIK_SPF
#define EIK_SPF 1
#endif
#ifndef EIK_PFOLD
#define EIK_PFOLD 0
#endif
#ifndef EIK_TWC
#define EIK_TWC 1
#endif
#ifndef EIK_TWI
#define EIK_TWI 1
#endif
#ifndef EIK_F4K_IL
#define EIK_F4K_IL 2
#endif
// EIK_TM_E = 8: the TMEM column kernels of 1024- to 4096-point lines hold 8
// values per thread (radix-8 Stockham stages) at twice the threads and half the
// registers (64), i.e. 32 resident warps per SM instead of 16 (A/B switch).
#ifndef EIK_TM_E
#define EIK_TM_E 16
#endif
#ifndef EIK_TM_E8_MAXL
#define EIK_TM_E8_MAXL 12
#endif
#ifndef EIK_TM_E8_MINL
#define EIK_TM_E8_MINL 10
#endif
template <int L, int LPCX = 1, bool WIDE = false>
struct TmCfg {
  static constexpr int E = (EIK_TM_E == 8 && L >= EIK_TM_E8_MINL && L <= EIK_TM_E8_MAXL) ? 8 : 16;
  static constexpr int TPL0 = tpl_of(L, E);
  static constexpr bool F4K = (L == 12 && EIK_FOUR_STEP && E == 16);
  static constexpr int NT = F4K ? 256 * LPCX : E == 8 ? (L >= 12 ? 1024 : 512)
                            : (WIDE && E == 16 && (L == 10 || L == 11)) ? 512
                            : (L == 11 && E == 16) ? EIK_TM11_NT
                            : (L == 10 && E == 16) ? EIK_TM10_NT
                            : (L == 9 && E == 16) ? EIK_TM9_NT : (TPL0 > 256 ? TPL0 : 256);
  static constexpr int LPC = NT / TPL0;
  static constexpr int MINB = E == 8 ? (NT >= 1024 ? 1 : 2) : (NT >= 512 ? 1 : 2);
  // four-step lines: EIK_F4K_IL = 1 makes the CTA line-major (warps 0-7 line 0,
  // 8-15 line 1) with one named barrier per line, so the lines drift apart and
  // one line's FP64 phase can overlap the other's exchange
  static constexpr int IL = F4K ? (EIK_F4K_IL < LPC ? EIK_F4K_IL : LPC) : col_il(LPC);
  using LN = std::conditional_t<F4K, Line4K,
                                std::conditional_t<E == 8, PaddedLine<L, 8, col_pad(L, IL == 2 && LPC > 2)>,
                                                   PaddedLine<L, 16, tm_pad(L, IL == 2 && LPC > 2, WIDE)>>>;
  using XB = XBuf<1, group_sync(IL, LPC, TPL0), IL * TPL0>;
  __device__ static __forceinline__ int line_of(int tid) { return (tid / (IL * TPL0)) * IL + tid % IL; }
  __device__ static __forceinline__ int t_of(int tid) { return (tid % (IL * TPL0)) / IL; }
  static constexpr int M0 = 1 << L;
  __device__ static __forceinline__ int k0_of(int tid, int r) { return LN::out_idx(t_of(tid), r); }
  // Folded register-order kernel spectra (four-step lines, two lanes-interleaved
  // lines): thread t = 16 a + b holds k0 = a + 16 b + 256 r, whose mirror
  // M - k0 is held by thread 16 (16 - a) + 15 - b at register 15 - r.  Warps
  // 0-8 (a <= 8) own the stored copy (NTP = 288 of 512 threads per register
  // row); warps 9-15 read their mirror's entries, in reversed lane order
  // (still whole contiguous segments), and the odd-kernel sign of k0 > M/2 is
  // applied at use.  9/16 of the unfolded bytes.
  static constexpr bool PFOLD = EIK_PFOLD && F4K && NT == 512 && IL == 2 && LPC == 2;
  static constexpr int NTP = PFOLD ? 288 : NT;
  static constexpr int WPT = 4 * LN::EPT;  // 32-bit TMEM words per thread (forward spectrum)
  // 4096-point lines: the radix-16 NS=256 stage's twiddles W^{t r} are per-thread
  // constants shared by the forward and every inverse -> cached in TMEM too
  static constexpr bool TWC = EIK_TWC && (L == 12) && LN::INV_SHARES && E == 16;
  // other long lines: the last inverse stage (radix R0 < 16 over NS = M/R0 > 16,
  // quarter-table twiddles otherwise) reads per-thread constants from TMEM
  // (C5 column kernel 5.19 -> 5.01 ms)
  static constexpr bool TWI = []() constexpr {
    if constexpr (F4K) return false;
    // (radix 2 / 8 groups: one TMEM wait per group costs more than it saves, C3 +2.5%)
    else return EIK_TWI && LN::EPT == 16 && LN::NST >= 2 && LN::R0 < 16 && LN::R0 >= 4 &&
                LN::st_quarter(true, LN::NST - 1);
  }();
  static constexpr int WPT_ALL = WPT + (TWC ? 64 : 0) + (TWI ? 64 : 0);
  static constexpr int NEED = (NT / 128) * WPT_ALL;
  static constexpr int COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr size_t MB_OFF = ((size_t)LPC * LN::SMEM + LN::TWQ + LN::ST_SIZE) * sizeof(double2) + 16;
  static constexpr size_t SMEM_BYTES = MB_OFF + 128;  // + the split-phase exchange mbarriers
  // TMA output stores (ColArgs::tstore): the staging tile [M/2 rows][LPC lines] and its
  // hand-over flag after the base layout, 128-byte aligned
  // (A/B switch, default off.  Measured on the B200 with the hand-over built
  // without any extra CTA barrier: distance column kernel 0.330 -> 0.322 ms, but the
  // C2 step 0.829 -> 0.887 ms.  Writing the tile alone costs 15 us of the 61 us the
  // direct stores cost (tools/gpu_ablate.sh), yet the engine reads the tile back in
  // 32-byte rows, a quarter of the shared-memory width per cycle, so the time
  // returns on the shared-memory pipe the exchanges already saturate;
  // tools/micro/tma_store_probe.cu: 2765 clocks per 64 KB tile with the SM idle.)
#ifndef EIK_TSTORE
#define EIK_TSTORE 0
#endif
  static constexpr bool TSTORE = EIK_TSTORE && F4K && LPC == 2;
  static constexpr size_t TSTORE_OFF = (SMEM_BYTES + 127) & ~size_t(127);
  static constexpr size_t TSTORE_TILE = (size_t)(LN::M / 2) * LPC * sizeof(double2);
  static constexpr size_t SMEM_TSTORE_BYTES = TSTORE_OFF + 128 + TSTORE_TILE + 32;
};

#ifndef EIK_SUM_CHUNKED
#define EIK_SUM_CHUNKED 0  // measured: ptxas spills more (132 / 252 bytes against 84 / 120)
#endif
#ifndef EIK_SUM_KCHUNK
#define EIK_SUM_KCHUNK 0  // measured: spill loads 120 -> 100 bytes, but the C2 sign pass 0.217 -> 0.225 ms
#endif
// v[r] *= K, four kernel-spectrum values at a time (sign group: the running sum, the product
// and 16 spectrum values do not fit 128 registers together)
template <class CFG, bool LM>
__device__ __forceinline__ void kmul_chunked(double2 (&v)[16], const KSpec& k, int64_t l, int t, int64_t bx, bool mir) {
  using LN = typename CFG::LN;
  const double* __restrict__ src = k.perm ? k.perm + bx * LN::EPT * CFG::NTP + threadIdx.x : nullptr;
  const bool neg1 = k.odd1 && mir;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double kn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = 4 * c + q;
      kn[q] = (!LM && src) ? __ldg(src + r * CFG::NTP) : kload<LM>(k, l, LN::out_idx(t, r), LN::M);
      if ((k.odd0 && LN::out_idx(t, r) > (LN::M >> 1)) != neg1) kn[q] = -kn[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = 4 * c + q;
      v[r] = k.imag ? make_double2(-v[r].y * kn[q], v[r].x * kn[q]) : make_double2(v[r].x * kn[q], v[r].y * kn[q]);
    }
    asm volatile("" ::: "memory");
  }
}
// v[i] = y[i] + v[i] with the 16 complex values y at TMEM address a, four at a time
__device__ __forceinline__ void tmem_add16(uint32_t a, double2 (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w32[16];
    tmem_ld16(a + 16 * c, w32);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 y = make_double2(
          __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 1] << 32) | w32[4 * q])),
          __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 3] << 32) | w32[4 * q + 2])));
      v[4 * c + q] = cadd(y, v[4 * c + q]);
    }
  }
}

// TMA tensor store (3-D box, shared -> global) and its bulk-group bookkeeping
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// Persistent: the grid is at most one resident wave of CTAs (launch_tmem_t);
// each CTA fills its twiddle tables, allocates its TMEM columns and caches its
// per-thread twiddles once, then walks the (item, tile) list with stride
// gridDim.x, tile index fastest, so concurrently running CTAs work on adjacent
// columns.  a.tiles = tiles per item, a.items = items.
#ifndef EIK_NEXTPF
#define EIK_NEXTPF 0  // next-tile L2 prefetch: measured C2 col 0.361 -> 0.369 ms, C5 5.36 -> 5.48, C3 1.95 -> 2.03
#endif
#ifndef EIK_DBG_NOK
#define EIK_DBG_NOK 0
#endif
// accumulating 3-D passes prefetch their destination rows into L2 before the inverse
// transform (C4 1024^3: sign group 287 -> 276.5 ms)
// Skipping the TMEM round trip component 0 does not need (its spectrum is still in the
// registers the forward transform left) is SLOWER in every kernel: C2 column kernel 0.319 ->
// 0.329 ms, C5 4.68 -> 4.98, C3 1.54 -> 1.56, C4 587 -> 599 ms per step (the branches around
// the tcgen05 instructions cost the schedule more than the two transfers); off.  As a
// compile-time variant for the single-component 3-D passes (no branch, no TMEM traffic at
// all) it is neutral: C4 587.0 -> 585.9 ms, so those transfers are not on the critical path.
#ifndef EIK_TM_SKIP0
#define EIK_TM_SKIP0 0
#endif
#ifndef EIK_ACCUM_PF
#define EIK_ACCUM_PF 1
#endif
// (C4 1024^3: 612.7 -> 602.3 ms in one A/B, within 3 ms of run-to-run noise)
#ifndef EIK_LM_KPF_EARLY
#define EIK_LM_KPF_EARLY 1
#endif
#ifndef EIK_KPF_EARLY_ALL
#define EIK_KPF_EARLY_ALL 0  // the same for the 2-D kernels (6 / 3 components per pass): C2 column kernel 0.318 -> 0.326 ms, C5 4.68 -> 4.73, C3 equal (the early lines do not survive in L1 next to the input loads)
#endif
#ifndef EIK_DBG_NOST
#define EIK_DBG_NOST 0
#endif
#ifndef EIK_DBG_STAGEONLY
#define EIK_DBG_STAGEONLY 0
#endif
template <int L, int IN, int OUT, bool HALF, bool LM = false>
__global__ void __launch_bounds__(TmCfg<L, tm_lpcx(L, OUT), LM>::NT, TmCfg<L, tm_lpcx(L, OUT), LM>::MINB)
    col_tmem_kernel(const __grid_constant__ ColArgs a) {
  using TC = TmCfg<L, tm_lpcx(L, OUT), LM>;
  using LN = typename TC::LN;
  constexpr int LPC = TC::LPC;
  extern __shared__ double2 smem[];
  const int line = TC::line_of(threadIdx.x);
  const int t = TC::t_of(threadIdx.x);
  typename TC::XB xb{smem + line * LN::SMEM, nullptr, 0, 1 + line / TC::IL};
  double2* twq = smem + LPC * LN::SMEM;
  double2* sts = twq + LN::TWQ;
  uint32_t* slot = reinterpret_cast<uint32_t*>(sts + LN::ST_SIZE);
  xb_setup(xb, reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + TC::MB_OFF), line / TC::IL, LPC / TC::IL,
           TC::NT);
  if constexpr (L >= 2) twq_fill(twq, L, a.tw, a.lmax);
  st_fill<LN>(sts, a.tw, a.lmax);
  const uint32_t tbase = tmem_alloc_cta(slot, TC::COLS);  // also publishes the twiddle tables
  const uint32_t ta = tmem_thread_addr(tbase, TC::WPT_ALL);
  uint32_t ttw = 0;
  if constexpr (TC::TWC) {
    ttw = ta + TC::WPT;
    double2 w[16];
    w[0] = make_double2(1.0, 0.0);
#pragma unroll
    for (int r = 1; r < 16; ++r) w[r] = twq_get(twq, L, t * r);  // W_4096^{t r}, k = t at NS = 256
    tmem_put(ttw, w);
  }
  uint32_t ttw2 = 0;
  if constexpr (TC::TWI) {
    ttw2 = ta + TC::WPT;
    tw_last_inv_fill<LN>(ttw2, t, twq, L);
  }
  const TwSrc tws{sts, twq, L, ttw, ttw2};
  const int tiles = (int)a.tiles;
  const int total = tiles * (int)a.items;  // < 2^31 (launcher)
  // TMA output stores: fill counter and the fill thread 0 still has to hand over
  int ts_seq = 0;
  if constexpr (TC::TSTORE && OUT == OUT_COMPS) {
    if (a.tstore && threadIdx.x == 0) {
      char* sbase = reinterpret_cast<char*>(smem);
      const uint32_t mis = smem_u32(sbase + TC::TSTORE_OFF) & 127u;
      volatile int* w = reinterpret_cast<volatile int*>(sbase + TC::TSTORE_OFF + (mis ? 128u - mis : 0u) + TC::TSTORE_TILE);
      w[0] = 0;
      w[1] = 0;
    }
  }

#pragma unroll 1
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const int item = tile / tiles;
    const int bx = tile - item * tiles;
    const int64_t l = (int64_t)bx * LPC + line;
    const bool valid = l < a.nlines;
    bool mir;
    const int64_t lk = fold_line(a, l, mir);
    // the tile this CTA runs next: its dense input lines head for L2 meanwhile
    auto next_prefetch = [&]() {
      if constexpr (EIK_NEXTPF && IN == IN_DENSE) {
        const int ntile = tile + gridDim.x;
        if (ntile < total) {
          const int nitem = ntile / tiles;
          const int64_t nl = (int64_t)(ntile - nitem * tiles) * LPC + line;
          if (nl < a.nlines) prefetch_dense_l2<LN, HALF>(a, t, nl, nitem, 0, true);
        }
      }
    };
    double2 v[LN::EPT];
    if constexpr (OUT == OUT_SUM) {
      // y = sum_i K_i X_i accumulated in TMEM while each input is transformed in registers
#pragma unroll 1
      for (int i = 0; i < a.n_in; ++i) {
        if (valid) kprefetch_all<TC, LM>(a.ks[i], lk, t, bx);  // into L1 while the input is transformed
        if constexpr (IN == IN_SPARSE) {
          load_sparse<LN, HALF>(v, a, t, l, item, i, valid, twq);
        } else {
          load_dense<LN, HALF>(v, a, t, l, item, i, valid);
          // the next input's line heads for L2 while this one is transformed
          if (EIK_SPF && i + 1 < a.n_in) prefetch_dense_l2<LN, HALF>(a, t, l, item, i + 1, valid);
          if (i + 1 == a.n_in) next_prefetch();
        }
        fft_line<LN, false, HALF>(v, t, xb, tws);
        if (valid) {
          if constexpr (EIK_SUM_KCHUNK && LN::EPT == 16 && !TC::PFOLD) {
            kmul_chunked<TC, LM>(v, a.ks[i], lk, t, bx, mir);
          } else {
            double kn[LN::EPT];
            kload_all<TC, LM>(kn, a.ks[i], lk, t, bx);
            kapply_all<LN>(v, kn, a.ks[i], t, mir);
          }
        } else {
#pragma unroll
          for (int r = 0; r < LN::EPT; ++r) v[r] = make_double2(0.0, 0.0);
        }
        if (i > 0) {
          if constexpr (EIK_SUM_CHUNKED && LN::EPT == 16) {
            tmem_add16(ta, v);  // four values at a time: the running sum never sits in 64 registers
          } else {
            double2 y[LN::EPT];
            tmem_get(ta, y);
#pragma unroll
            for (int r = 0; r < LN::EPT; ++r) v[r] = cadd(y[r], v[r]);
          }
        }
        if (i + 1 < a.n_in) tmem_put(ta, v);
      }
      fft_line<LN, true>(v, t, xb, tws);
#pragma unroll
      for (int r = 0; r < LN::EPT; ++r) {
        if (LN::L > 0 && LN::upper_in(r)) continue;
        const int n = LN::in_idx(t, r);
        if (valid && n < a.n_out) store_u(comp_dst(a, 0, item, l, n), v[r]);
      }
    } else if (TC::TSTORE && OUT == OUT_COMPS && a.tstore) {
      // Outputs through shared memory and TMA.  Fill s of the staging tile (one per
      // component) is handed to the TMA engine by thread 0 right after the next
      // CTA-wide barrier (every thread's tile writes precede it), i.e. inside the
      // next transform; before fill s + 1 thread 0 waits until the engine has read
      // fill s and publishes that through a shared flag.  No extra CTA barrier.
      if constexpr (TC::TSTORE && OUT == OUT_COMPS) {
        char* sbase = reinterpret_cast<char*>(smem);
        const uint32_t mis = smem_u32(sbase + TC::TSTORE_OFF) & 127u;
        double2* stg = reinterpret_cast<double2*>(sbase + TC::TSTORE_OFF + (mis ? 128u - mis : 0u));
        // hand-over words after the tile: [0] fills whose tile has been read, [1] a fill
        // is pending, [2..4] its component, tile and item (thread 0's bookkeeping)
        volatile int* freed = reinterpret_cast<volatile int*>(reinterpret_cast<char*>(stg) + TC::TSTORE_TILE);
        auto hook = [&]() {
          if (threadIdx.x == 0 && freed[1]) {
            for (int y = 0; y < a.n_out; y += 256)
              tma_store_3d(&a.umap[freed[2]], stg + y * LPC, freed[3] * LPC * 2, y, freed[4]);
            bulk_commit();
            freed[1] = 0;
          }
        };
        if constexpr (IN == IN_SPARSE) load_sparse<LN, HALF>(v, a, t, l, item, 0, valid, twq);
        else load_dense<LN, HALF>(v, a, t, l, item, 0, valid);
        fft_line<LN, false, HALF>(v, t, xb, tws, hook);
        tmem_put(ta, v);
        if (valid) kprefetch_all<TC, LM>(a.ks[0], lk, t, bx);
#pragma unroll 1
        for (int j = 0; j < a.n_comp; ++j) {
          tmem_get(ta, v);
          if (valid) {
            double kn[LN::EPT];
            kload_all<TC, LM>(kn, a.ks[j], lk, t, bx);
            if (j + 1 < a.n_comp) kprefetch_all<TC, LM>(a.ks[j + 1], lk, t, bx);
            kapply_all<LN>(v, kn, a.ks[j], t, mir);
          }
          fft_line<LN, true>(v, t, xb, tws, hook);
          // the tile is free once the engine has read the previous fill
          ++ts_seq;
          if (threadIdx.x == 0) {
            bulk_wait_read0();
            *freed = ts_seq;
          }
          __syncwarp();
          while (*freed < ts_seq) {
          }
#pragma unroll
          for (int r = 0; r < LN::EPT; ++r) {
            if (LN::L > 0 && LN::upper_in(r)) continue;
            stg[LN::in_idx(t, r) * LPC + line] = v[r];
          }
          fence_proxy_async_smem();
          if (threadIdx.x == 0) {
            freed[1] = 1;
            freed[2] = j;
            freed[3] = bx;
            freed[4] = item;
          }
        }
      }
    } else {
      // 3-D passes often carry one component (streamed schedule): its kernel spectrum heads
      // for L1 before the forward transform, not after it
      constexpr bool KPF_EARLY = (LM && EIK_LM_KPF_EARLY) || EIK_KPF_EARLY_ALL;
      if constexpr (KPF_EARLY) {
        if (valid && !EIK_DBG_NOK) kprefetch_all<TC, LM>(a.ks[0], lk, t, bx);
      }
      if constexpr (IN == IN_SPARSE) load_sparse<LN, HALF>(v, a, t, l, item, 0, valid, twq);
      else load_dense<LN, HALF>(v, a, t, l, item, 0, valid);
      fft_line<LN, false, HALF>(v, t, xb, tws);
      if (!EIK_TM_SKIP0 || a.n_comp > 1) tmem_put(ta, v);  // one component: the spectrum stays in registers
      // kernel spectra: the next component's lines are prefetched into L1 one
      // transform ahead (no registers held across the FFT); loaded at use
      if (!KPF_EARLY && valid && !EIK_DBG_NOK) kprefetch_all<TC, LM>(a.ks[0], lk, t, bx);
      next_prefetch();
#pragma unroll 1
      for (int j = 0; j < a.n_comp; ++j) {
        if (!EIK_TM_SKIP0 || j > 0) tmem_get(ta, v);  // component 0 multiplies the registers the forward left
        if (valid && !EIK_DBG_NOK) {
          double kn[LN::EPT];
          kload_all<TC, LM>(kn, a.ks[j], lk, t, bx);
          if (j + 1 < a.n_comp) kprefetch_all<TC, LM>(a.ks[j + 1], lk, t, bx);
          kapply_all<LN>(v, kn, a.ks[j], t, mir);
        }
        if constexpr (LM && EIK_ACCUM_PF) {
          // accumulating pass: the destination rows head for L2 while the inverse runs
          if (a.accum && valid) {
#pragma unroll
            for (int r = 0; r < LN::EPT; ++r) {
              if (LN::L > 0 && LN::upper_in(r)) continue;
              const int n = LN::in_idx(t, r);
              if (n < a.n_out) asm volatile("prefetch.global.L2 [%0];" ::"l"(comp_dst(a, j, item, l, n)));
            }
          }
        }
        fft_line<LN, true>(v, t, xb, tws);
        if (a.accum) {  // uniform: the streamed sign group adds into W
#pragma unroll
          for (int r = 0; r < LN::EPT; ++r) {
            if (LN::L > 0 && LN::upper_in(r)) continue;
            const int n = LN::in_idx(t, r);
            if (valid && n < a.n_out) {
              double2* dst = comp_dst(a, j, item, l, n);
              *dst = cadd(*dst, v[r]);
            }
          }
        } else {
#if EIK_DBG_STAGEONLY
          // timing probe: the component goes to a shared-memory tile [row][line] only
          double2* stg = reinterpret_cast<double2*>(reinterpret_cast<char*>(smem) + ((TC::SMEM_BYTES + 127) & ~size_t(127)));
#pragma unroll
          for (int r = 0; r < LN::EPT; ++r) {
            if (LN::L > 0 && LN::upper_in(r)) continue;
            const int n = LN::in_idx(t, r);
            if (n < LN::M / 2) stg[n * LPC + line] = v[r];
          }
#else
#pragma unroll
          for (int r = 0; r < LN::EPT; ++r) {
            if (LN::L > 0 && LN::upper_in(r)) continue;
            const int n = LN::in_idx(t, r);
            if (valid && n < a.n_out && !(EIK_DBG_NOST && a.n_comp < 100)) store_u(comp_dst(a, j, item, l, n), v[r]);
          }
#endif
        }
      }
    }
  }
  if constexpr (TC::TSTORE && OUT == OUT_COMPS) {
    if (a.tstore) {  // the last fill leaves after one more barrier; the tile stays valid until it is read
      __syncthreads();
      if (threadIdx.x == 0) {
        char* sbase = reinterpret_cast<char*>(smem);
        const uint32_t mis = smem_u32(sbase + TC::TSTORE_OFF) & 127u;
        double2* stg = reinterpret_cast<double2*>(sbase + TC::TSTORE_OFF + (mis ? 128u - mis : 0u));
        volatile int* w = reinterpret_cast<volatile int*>(reinterpret_cast<char*>(stg) + TC::TSTORE_TILE);
        if (w[1]) {
          for (int y = 0; y < a.n_out; y += 256) tma_store_3d(&a.umap[w[2]], stg + y * LPC, w[3] * LPC * 2, y, w[4]);
          bulk_commit();
        }
        bulk_wait_read0();
      }
    }
  }
  tmem_free_cta(tbase, TC::COLS);
}

// ---------------------------------------------------------------------------
// Even / odd split column kernel for 4096-point lines (distance group).
//
// A half-padded 4096-point forward transform is two independent 2048-point
// transforms of the same input: X[2k] = FFT2048(x)[k], X[2k+1] = FFT2048(x W4096^n)[k],
// and the first 2048 outputs of the inverse are
//   y[n] = IFFT2048(Y_even)[n] + conj(W4096^n) IFFT2048(Y_odd)[n].
// The 512-thread CTA is two groups of 8 warps: group 0 owns the even bins of
// the tile's two lines, group 1 the odd bins.  Each group runs the 2048-point
// Stockham schedule (lines interleaved by lane parity, like the 256-thread TMEM
// kernel of 2048-point lines) on its own exchange buffers under its own named
// barrier, keeps its half of the forward spectrum in TMEM, and multiplies its
// half of every kernel spectrum.  Per component group 1 hands its twiddled
// result to group 0 through a shared-memory buffer, warp to warp (thread
// (line, t) of both groups holds the same n): one mbarrier pair per warp pair,
// no CTA-wide barrier anywhere.  Group 0 adds and stores.  The groups therefore
// run out of phase (group 1 one hand-over ahead): one group's FP64 butterflies
// overlap the other's shared-memory exchange and global stores, which the
// lock-step 16-warp kernel cannot do.
// Measured on the B200 (C2, tools/gpu_eo1.sh, profiles/round2/eo/): parity green, but the
// column kernel takes 0.415 ms against 0.318 ms for the 16-warp four-step kernel, and its
// parts are additive as well (no FP64 -82 us, no exchanges -104, no stores -63, no hand-over
// -28, no spectrum loads -28): eight warps per group do not fill a unit within a phase, so
// the out-of-phase groups hide nothing.  Off by default (-DEIK_EO=1 builds it, EIK_EO=0 at
// run time then selects the four-step kernel).
#ifndef EIK_EO
#define EIK_EO 0
#endif
#ifndef EIK_DBG_NOHAND
#define EIK_DBG_NOHAND 0  // timing probe: no hand-over between the groups (wrong results)
#endif
struct LineEO : PaddedLine<11, 16, pad_code(3, 5, 6)> {
  // only the inverse's NS = 16 stage keeps a stage table (240 entries); every
  // other twiddle comes from the quarter table or this thread's TMEM constants
  static constexpr bool INV_SHARES = false;
  __host__ __device__ static constexpr bool st_quarter(bool inv, int s) { return s >= 1 && !(inv && s == 1); }
  __host__ __device__ static constexpr int st_size(bool inv, int s) { return (inv && s == 1) ? 16 * 15 : 0; }
  __host__ __device__ static constexpr int st_off(bool, int) { return 0; }
  static constexpr int ST_SIZE = 16 * 15;
};
struct EoCfg {
  using LN = LineEO;
  static constexpr int NT = 512, GT = 256, LPC = 2, NTP = 512, M0 = 4096;
  static constexpr bool PFOLD = false;
  using XB = XBuf<1, 2, GT>;
  __device__ static __forceinline__ int group_of(int tid) { return tid >> 8; }
  __device__ static __forceinline__ int line_of(int tid) { return tid & 1; }
  __device__ static __forceinline__ int t_of(int tid) { return (tid & 255) >> 1; }
  __device__ static __forceinline__ int k0_of(int tid, int r) { return 2 * LN::out_idx(t_of(tid), r) + group_of(tid); }
  static constexpr int WPT = 64, WPT_ALL = 128, COLS = 512;  // TMEM words per thread: spectrum half + constants
  static constexpr size_t HB_OFF = (size_t)4 * LN::SMEM * sizeof(double2);
  static constexpr size_t TWQ_OFF = HB_OFF + (size_t)16 * GT * sizeof(double2);
  static constexpr size_t ST_OFF = TWQ_OFF + (size_t)LN::TWQ * sizeof(double2);
  static constexpr size_t SLOT_OFF = ST_OFF + (size_t)LN::ST_SIZE * sizeof(double2);
  static constexpr size_t MB_OFF = SLOT_OFF + 16;  // 2 exchange + 8 full + 8 empty mbarriers
  static constexpr size_t SMEM_BYTES = MB_OFF + 18 * sizeof(uint64_t);
};
static_assert(EoCfg::SMEM_BYTES <= 227 * 1024, "even/odd column kernel: shared memory");

// v[i] *= c[i] (or conj), the 16 per-thread constants at TMEM address a, four at a time
template <bool CONJ>
__device__ __forceinline__ void tmem_cmul16(uint32_t a, double2 (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w32[16];
    tmem_ld16(a + 16 * c, w32);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 w = make_double2(
          __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 1] << 32) | w32[4 * q])),
          __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 3] << 32) | w32[4 * q + 2])));
      v[4 * c + q] = CONJ ? cmulc(v[4 * c + q], w) : cmul(v[4 * c + q], w);
    }
  }
}

template <int IN>
__global__ void __launch_bounds__(EoCfg::NT, 1) col_eo_kernel(const __grid_constant__ ColArgs a) {
  using TC = EoCfg;
  using LN = LineEO;
  extern __shared__ double2 smem[];
  char* sbase = reinterpret_cast<char*>(smem);
  const int tid = threadIdx.x;
  const int g = TC::group_of(tid), line = TC::line_of(tid), t = TC::t_of(tid), tig = tid & (TC::GT - 1);
  const int wp = tig >> 5;  // warp pair of the hand-over
  typename TC::XB xb{smem + (g * 2 + line) * LN::SMEM, nullptr, 0, 1 + g};
  double2* hb = reinterpret_cast<double2*>(sbase + TC::HB_OFF) + tig;  // [register][thread of the group]
  double2* twq = reinterpret_cast<double2*>(sbase + TC::TWQ_OFF);
  double2* sts = reinterpret_cast<double2*>(sbase + TC::ST_OFF);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sbase + TC::SLOT_OFF);
  uint64_t* mbs = reinterpret_cast<uint64_t*>(sbase + TC::MB_OFF);
  uint64_t* mb_full = mbs + 2 + wp;
  uint64_t* mb_empty = mbs + 10 + wp;
  if (tid < 16) mbar_init(mbs + 2 + tid, 1u);
  xb_setup(xb, mbs, g, 2, TC::NT);
  twq_fill(twq, LN::L, a.tw, a.lmax);
  st_fill<LN>(sts, a.tw, a.lmax);
  const uint32_t tbase = tmem_alloc_cta(slot, TC::COLS);  // also publishes the tables and the mbarriers
  const uint32_t ta = tmem_thread_addr(tbase, TC::WPT_ALL);
  const uint32_t tc = ta + TC::WPT;
  if (g) {  // W4096^n of this thread's 16 elements
    double2 w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = __ldg(a.tw + ((int64_t)LN::in_idx(t, i) << (a.lmax - 12)));
    tmem_put(tc, w);
  } else {  // the last inverse stage's twiddles
    tw_last_inv_fill<LN>(tc, t, twq, LN::L);
  }
  const TwSrc tws{sts, twq, LN::L, 0u, g ? 0u : tc};
  const int tiles = (int)a.tiles;
  const int total = tiles * (int)a.items;
  uint32_t seq = 0;  // hand-overs so far (parity of the mbarrier phases)

#pragma unroll 1
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const int item = tile / tiles;
    const int bx = tile - item * tiles;
    const int64_t l = (int64_t)bx * TC::LPC + line;
    const bool valid = l < a.nlines;
    bool mir;
    const int64_t lk = fold_line(a, l, mir);
    double2 v[16];
    if constexpr (IN == IN_SPARSE) load_sparse<LN, false>(v, a, t, l, item, 0, valid, twq);
    else load_dense<LN, false>(v, a, t, l, item, 0, valid);
    if (g) tmem_cmul16<false>(tc, v);
    fft_line<LN, false, false>(v, t, xb, tws);
    tmem_put(ta, v);
    auto kprefetch = [&](const KSpec& k) {  // the next component's values head for L2 (no L1 left next to 226 KB)
      if (!valid) return;
      if (k.perm) {
        const double* src = k.perm + (int64_t)bx * 16 * TC::NTP + tid;
#pragma unroll
        for (int r = 0; r < 16; ++r) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r * TC::NTP));
      } else {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int k0 = TC::k0_of(tid, r);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(k.re + (int64_t)(k0 > 2048 ? 4096 - k0 : k0) * k.ld + lk));
        }
      }
    };
    if (!EIK_DBG_NOK) kprefetch(a.ks[0]);
#pragma unroll 1
    for (int j = 0; j < a.n_comp; ++j) {
      tmem_get(ta, v);
      if (valid && !EIK_DBG_NOK) {
        const KSpec& k = a.ks[j];
        double kn[16];
        if (k.perm) {
          const double* __restrict__ src = k.perm + (int64_t)bx * 16 * TC::NTP + tid;
#pragma unroll
          for (int r = 0; r < 16; ++r) kn[r] = __ldg(src + r * TC::NTP);
        } else {
#pragma unroll
          for (int r = 0; r < 16; ++r) kn[r] = kload(k, lk, TC::k0_of(tid, r), 4096);
        }
        if (j + 1 < a.n_comp) kprefetch(a.ks[j + 1]);
        const bool neg1 = k.odd1 && mir;
        if (k.odd0 || neg1) {
#pragma unroll
          for (int r = 0; r < 16; ++r)
            if ((k.odd0 && TC::k0_of(tid, r) > 2048) != neg1) kn[r] = -kn[r];
        }
        if (k.imag) {
#pragma unroll
          for (int r = 0; r < 16; ++r) v[r] = make_double2(-v[r].y * kn[r], v[r].x * kn[r]);
        } else {
#pragma unroll
          for (int r = 0; r < 16; ++r) v[r] = make_double2(v[r].x * kn[r], v[r].y * kn[r]);
        }
      }
      fft_line<LN, true>(v, t, xb, tws);
      if (g) {
        tmem_cmul16<true>(tc, v);
#if !EIK_DBG_NOHAND
        mbar_wait(mb_empty, (seq & 1u) ^ 1u);  // group 0 has taken the previous hand-over
#pragma unroll
        for (int i = 0; i < 16; ++i) hb[i * TC::GT] = v[i];
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(mb_full);
#endif
      } else {
#if !EIK_DBG_NOHAND
        mbar_wait(mb_full, seq & 1u);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = cadd(v[i], hb[i * TC::GT]);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(mb_empty);
#endif
        if (a.accum) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = LN::in_idx(t, i);
            if (valid && n < a.n_out) {
              double2* dst = comp_dst(a, j, item, l, n);
              *dst = cadd(*dst, v[i]);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = LN::in_idx(t, i);
            if (valid && n < a.n_out && !(EIK_DBG_NOST && a.n_comp < 100)) store_u(comp_dst(a, j, item, l, n), v[i]);
          }
        }
      }
      ++seq;
    }
  }
  tmem_free_cta(tbase, TC::COLS);
}

// Register-order copy of a folded real/imaginary spectrum for the column
// kernel configuration CFG (see KSpec::perm).  One thread per output value.
template <class CFG>
__global__ void spectrum_perm_kernel(const double* __restrict__ re, int64_t ld, int64_t nlines, int odd0,
                                     double* __restrict__ kp, int64_t total) {
  using LN = typename CFG::LN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int tid = (int)(i % CFG::NTP);
    const int64_t rest = i / CFG::NTP;
    const int r = (int)(rest % LN::EPT);
    const int64_t b = rest / LN::EPT;
    const int64_t l = b * CFG::LPC + CFG::line_of(tid);
    const int k0 = CFG::k0_of(tid, r);
    const bool hi = k0 > (CFG::M0 >> 1);
    double v = 0.0;
    if (l < nlines) {
      v = re[(int64_t)(hi ? CFG::M0 - k0 : k0) * ld + l];
      if (odd0 && hi && !CFG::PFOLD) v = -v;  // folded copies: sign applied at use
    }
    kp[i] = v;
  }
}

// Strided batched c2c lines (3D axis 1, both directions).  Line l of component
// blockIdx.y: base = (l / inner) * outer_stride + (l % inner); element stride es.
struct LinesArgs {
  const double2* in[MAXC];
  double2* out[MAXC];
  int64_t nlines, inner, outer_in, outer_out, es_in, es_out;
  // element e -> (e >> shift) * split_stride + (e & (2^shift - 1)) * es, separately for in / out
  int split_shift, split_shift_out;
  int64_t split_stride, split_stride_out;
  int n_valid, n_out;
  double scale;
  const double2* tw;
  int lmax;
  // peer-block outputs (see ColArgs::blk): element n of component c goes to
  // blk[n >> split_shift_out] + c * blk_cstride + o * outer_out + q + (n mod 2^shift) * es_out
  double2* blk[MAXG];
  int64_t blk_cstride;
  // set by the launcher: tiles of LPC lines per component, components
  int64_t tiles;
  int ncomp;
};

// Lines of 1024 to 4096 points: 16 values per thread (two exchanges instead of the three of the
// radix-8 column configuration, which needs its registers for the product as well), 512 threads,
// i.e. 8 / 4 / 2 adjacent lines per CTA (128- / 64- / 32-byte runs per element), persistent CTAs
// (tables filled once per SM instead of once per 2 lines).  EIK_LINES_E16=0: the column configuration.
#ifndef EIK_LINES_E16
#define EIK_LINES_E16 1
#endif
// next-tile L2 prefetch from the persistent loop (C4 1024^3: lines passes 19.0 / 19.7 -> 17.8 /
// 18.5 ms, step 649 -> 638 ms; the same prefetch in the axis-0 column kernel, EIK_NEXTPF, costs
// 7%: 649 -> 696 ms)
#ifndef EIK_LINES16_SPLIT
#define EIK_LINES16_SPLIT 1  // split-phase exchange barriers in the 16-value lines kernels (C4 1024^3: 596 -> 586.5 ms)
#endif
#ifndef EIK_LINES_NEXTPF
#define EIK_LINES_NEXTPF 1
#endif
template <int L>
struct LinesCfg16 {
  static constexpr int TPL0 = (1 << L) / 16;
  static constexpr int NT = 512;
  static constexpr int LPC = NT / TPL0;
  static constexpr int IL = LPC;
  static constexpr bool PERSIST = true;
  using LN = PaddedLine<L, 16, (L == 10 ? pad_code(2, 0, 0) : L == 11 ? pad_code(3, 4, 0) : pad_code(4, 0, 5))>;
  __device__ static __forceinline__ int line_of(int tid) { return tid % LPC; }
  __device__ static __forceinline__ int t_of(int tid) { return tid / LPC; }
  static constexpr int NBUF = 1;
  using XB = XBuf<1, 0, NT, (EIK_LINES16_SPLIT != 0)>;
  static constexpr size_t MB_OFF = ((size_t)LPC * LN::SMEM + LN::TWQ + LN::ST_SIZE) * sizeof(double2);
  static constexpr size_t SMEM_BYTES = MB_OFF + 128;
};
// persistent CTAs (+ next-tile prefetch) for the 512-point lines of C3 as well: lines pass
// 0.812 -> 0.781 ms, step 3.114 -> 3.070 ms
#ifndef EIK_LINES9_PERSIST
#define EIK_LINES9_PERSIST 1
#endif
template <int L>
struct LinesColCfg : ColCfg<L> {
  static constexpr bool PERSIST = (L == 9 && EIK_LINES9_PERSIST);
};
template <int L>
using LinesCfg = std::conditional_t<(EIK_LINES_E16 && L >= 10 && L <= 12), LinesCfg16<L>, LinesColCfg<L>>;

template <int L, bool INV, bool HALF>
__global__ void __launch_bounds__(LinesCfg<L>::NT) lines_kernel(const __grid_constant__ LinesArgs a) {
  using CC = LinesCfg<L>;
  using LN = typename CC::LN;
  constexpr int LPC = CC::LPC;
  extern __shared__ double2 smem[];
  const int line = CC::line_of(threadIdx.x);
  const int t = CC::t_of(threadIdx.x);
  typename CC::XB xb{smem + line * LN::SMEM, smem + (LPC + line) * LN::SMEM, 0, 1 + line / CC::IL};
  double2* twq = smem + CC::NBUF * LPC * LN::SMEM;
  double2* sts = twq + LN::TWQ;
  xb_setup(xb, reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + CC::MB_OFF), line / CC::IL, LPC / CC::IL,
           CC::NT);
  if constexpr (L >= 2) twq_fill(twq, L, a.tw, a.lmax);
  st_fill<LN>(sts, a.tw, a.lmax);
  __syncthreads();
  const TwSrc tws{sts, twq, L, 0u};
  // (component, tile) work items, tile fastest; one per CTA unless the launch is persistent
  const int64_t total = a.tiles * a.ncomp;
#pragma unroll 1
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
  const int c = (int)(w / a.tiles);
  const int64_t l = (w - c * a.tiles) * LPC + line;
  const bool valid = l < a.nlines;
  const int64_t o = valid ? l / a.inner : 0, q = valid ? l % a.inner : 0;
  const double2* src = a.in[c] + o * a.outer_in + q;
  double2* dst = a.out[c] + o * a.outer_out + q;
  double2 v[LN::EPT];
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    if (HALF && LN::L > 0 && LN::upper_in(r)) continue;
    const int e = INV ? LN::out_idx(t, r) : LN::in_idx(t, r);  // inverse input layout = forward output layout
    v[r] = (valid && e < a.n_valid)
               ? src[(int64_t)(e >> a.split_shift) * a.split_stride + (int64_t)(e & ((1 << a.split_shift) - 1)) * a.es_in]
               : make_double2(0.0, 0.0);
  }
  if constexpr (CC::PERSIST && EIK_LINES_NEXTPF) {
    // the tile this CTA runs next heads for L2 while this one is transformed (no registers held)
    const int64_t w2 = w + gridDim.x;
    if (w2 < total) {
      const int c2 = (int)(w2 / a.tiles);
      const int64_t l2 = (w2 - c2 * a.tiles) * LPC + line;
      if (l2 < a.nlines) {
        const double2* src2 = a.in[c2] + (l2 / a.inner) * a.outer_in + (l2 % a.inner);
#pragma unroll
        for (int r = 0; r < LN::EPT; ++r) {
          if (HALF && LN::L > 0 && LN::upper_in(r)) continue;
          const int e = INV ? LN::out_idx(t, r) : LN::in_idx(t, r);
          if (e < a.n_valid)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(src2 + (int64_t)(e >> a.split_shift) * a.split_stride +
                                                         (int64_t)(e & ((1 << a.split_shift) - 1)) * a.es_in));
        }
      }
    }
  }
  fft_line<LN, INV, HALF>(v, t, xb, tws);
  if (!valid) continue;
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    const int n = INV ? LN::in_idx(t, r) : LN::out_idx(t, r);
    if (n < a.n_out) {
      double2 x = v[r];
      if (a.scale != 1.0) { x.x *= a.scale; x.y *= a.scale; }
      const int64_t in_blk = (int64_t)(n & ((1 << a.split_shift_out) - 1)) * a.es_out;
      if (a.blk[0]) a.blk[n >> a.split_shift_out][c * a.blk_cstride + o * a.outer_out + q + in_blk] = x;
      else dst[(int64_t)(n >> a.split_shift_out) * a.split_stride_out + in_blk] = x;
    }
  }
  }
}

// ---------------------------------------------------------------------------
// Kernel sample generation (the reference's sampled kernels, R/distance.py:33-37,
// R/derivatives.py:35-57,139-153, R/sign.py:97-105) on the wrap-around lattice.

enum KType {
  KT_EXP = 0,
  KT_GRAD0 = 1, KT_GRAD1 = 2, KT_GRAD2 = 3,   // (o_a/|o|) * exp
  KT_HXX = 4, KT_HYY = 5, KT_HXY = 6,          // Eq. 40-42 factors * exp (2D)
  KT_RAT2_0 = 7, KT_RAT2_1 = 8,                // o_a/|o|^2 (2D winding)
  KT_RAT3_0 = 9, KT_RAT3_1 = 10, KT_RAT3_2 = 11,  // o_a/|o|^3 (3D degree)
  KT_FIELD = 12,                               // dense user samples (host-provided)
};

struct GenArgs {
  int D;            // internal dimension (2 or 3)
  int c[3];         // grid counts (internal axes)
  int M[3];         // padded lengths
  int ref_axis0;    // first internal axis that is a reference axis (1 for 1-D grids)
  double h, tau, inv_tau, sign;
  int ktype;
  const double* field;   // KT_FIELD: samples; fshape/fstride describe it
  int64_t fcenter[3], fstride[3];
  int field_is_grid;     // 1: field is a grid array (no wrap, rows [0,c)); 0: centred kernel
};

// signed offset of padded index j on an axis with count c and length M, or
// INT_MIN when the index lies outside the kernel support [-(c-1), c-1].
__device__ __forceinline__ int wrap_offset(int j, int c, int M) {
  if (j < c) return j;
  if (j > M - c) return j - M;
  return -0x40000000;
}

__device__ __forceinline__ double sample_kernel(const GenArgs& g, int o0, int o1, int o2) {
  const double h = g.h;
  // offsets of the reference axes (internal axis 0 is a dummy for 1-D grids)
  const double m0 = h * (double)o0, m1 = h * (double)o1, m2 = h * (double)o2;
  const bool centre = (o0 == 0 && o1 == 0 && o2 == 0);
  if (g.ktype == KT_EXP || (g.ktype >= KT_GRAD0 && g.ktype <= KT_HXY)) {
    const long long r2i = (long long)o0 * o0 + (long long)o1 * o1 + (long long)o2 * o2;
    const double base = exp(-(h * sqrt((double)r2i)) / g.tau);
    if (g.ktype == KT_EXP) return base;
    // DirectionalKernels: r = sqrt(sum of squared float offsets), 0 at the centre
    double r;
    if (g.D == 3) r = sqrt((m0 * m0 + m1 * m1) + m2 * m2);
    else if (g.ref_axis0 == 1) r = sqrt(m1 * m1);
    else r = sqrt(m0 * m0 + m1 * m1);
    if (centre) return 0.0 * base;
    const double ir = 1.0 / r;
    double f;
    if (g.ktype <= KT_GRAD2) {
      const int a = g.ktype - KT_GRAD0 + g.ref_axis0;
      const double m = (a == 0) ? m0 : (a == 1 ? m1 : m2);
      f = m / r;
    } else {
      const double fc = m0 / r, fs = m1 / r, it = g.inv_tau;
      if (g.ktype == KT_HXX) f = ((-it) * fc) * fc + (fs * fs) * ir;
      else if (g.ktype == KT_HYY) f = ((-it) * fs) * fs + (fc * fc) * ir;
      else f = ((-(it + ir)) * fc) * fs;
    }
    return f * base;
  }
  // ratio kernels (sign): numerator / r^p with r from the float offsets
  double r = (g.D == 3) ? sqrt((m0 * m0 + m1 * m1) + m2 * m2) : sqrt(m0 * m0 + m1 * m1);
  if (centre) return 0.0;
  double num;
  int p;
  if (g.ktype <= KT_RAT2_1) { num = (g.ktype == KT_RAT2_0) ? m0 : m1; p = 2; }
  else { const int a = g.ktype - KT_RAT3_0; num = (a == 0) ? m0 : (a == 1 ? m1 : m2); p = 3; }
  const double den = (p == 2) ? r * r : pow(r, 3.0);
  return g.sign * (num / den);
}

// Real sample x[j] of padded row `row` (all non-last padded indices flattened).
__device__ __forceinline__ double gen_value(const GenArgs& g, int64_t row, int j) {
  const int D = g.D;
  int jj[3];
  if (D == 3) { jj[0] = (int)(row / g.M[1]); jj[1] = (int)(row % g.M[1]); jj[2] = j; }
  else { jj[0] = (int)row; jj[1] = j; jj[2] = 0; }
  if (g.ktype == KT_FIELD) {
    if (g.field_is_grid) {
      int64_t off = 0;
      for (int a = 0; a < D; ++a) {
        if (jj[a] >= g.c[a]) return 0.0;
        off += (int64_t)jj[a] * g.fstride[a];
      }
      return g.field[off];
    }
    int64_t off = 0;
    for (int a = 0; a < D; ++a) {
      const int o = wrap_offset(jj[a], g.c[a], g.M[a]);
      if (o == -0x40000000) return 0.0;
      off += (int64_t)(o + g.fcenter[a]) * g.fstride[a];
    }
    return g.field[off];
  }
  int o[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) {
    const int oa = wrap_offset(jj[a], g.c[a], g.M[a]);
    if (oa == -0x40000000) return 0.0;
    o[a] = oa;
  }
  return (D == 3) ? sample_kernel(g, o[0], o[1], o[2]) : sample_kernel(g, o[0], o[1], 0);
}

// r2c of padded real rows of length 2*MH: out[row * out_rs + k], k in [0, MH].
template <int LH>
__global__ void __launch_bounds__(RowCfg<LH>::NT) row_r2c_kernel(const __grid_constant__ GenArgs g, int64_t nrows,
                                                                 double2* out, int64_t out_rs,
                                                                 const double2* tw, int lmax) {
  using LN = typename RowCfg<LH>::LN;
  constexpr int LPC = RowCfg<LH>::LPC;
  constexpr int MH = LN::M;
  constexpr int LQ = LH + 1;  // quarter table at the resolution of the real row length
  extern __shared__ double2 smem[];
  const int line = threadIdx.x / LN::TPL;
  const int t = threadIdx.x % LN::TPL;
  const int64_t row = (int64_t)blockIdx.x * LPC + line;
  const bool valid = row < nrows;
  using RC = RowCfg<LH>;
  typename RC::XB xb{smem + line * LN::SMEM, smem + (LPC + line) * LN::SMEM, 0, 1 + line};
  double2* twq = smem + RC::NBUF * LPC * LN::SMEM;
  double2* sts = twq + RC::TWQ;
  xb_setup(xb, reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + RC::MB_OFF), line, LPC, RC::NT);
  twq_fill(twq, LQ, tw, lmax);
  st_fill<LN>(sts, tw, lmax);
  __syncthreads();
  const TwSrc tws{sts, twq, LQ, 0u};
  double2 v[LN::EPT];
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    const int m = LN::in_idx(t, r);
    v[r] = valid ? make_double2(gen_value(g, row, 2 * m), gen_value(g, row, 2 * m + 1)) : make_double2(0.0, 0.0);
  }
  fft_line<LN, false>(v, t, xb, tws);
  // natural-order spectrum Z into shared memory (the buffer the last exchange
  // did not use), then split into X[k], k in [0, MH]
  xb.acquire();
  double2* sm = xb.cur();
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) sm[LN::pad(LN::out_idx(t, r))] = v[r];
  __syncthreads();
  if (!valid) return;
  for (int k = t; k <= MH; k += LN::TPL) {
    const double2 zk = sm[LN::pad(k & (MH - 1))];
    const double2 zc = sm[LN::pad((MH - k) & (MH - 1))];
    const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y - zc.y));   // (Z[k] + conj Z[-k]) / 2
    const double2 d = make_double2(0.5 * (zk.y + zc.y), -0.5 * (zk.x - zc.x));  // (Z[k] - conj Z[-k]) / (2i)
    const double2 w = twq_get(twq, LQ, k);                                     // W_M^k (k = MH -> -1)
    out[row * out_rs + k] = cadd(e, cmul(d, w));
  }
}

// ---------------------------------------------------------------------------
// Row pass: c2r along the last axis fused with the epilogue.

struct RowArgs {
  int64_t rows;        // rows per item
  int64_t row0, row_end, item0;  // this launch covers rows [row0, row_end) of items item0 + blockIdx.y
  int n_out;           // grid count along the last axis
  int64_t rows_a, stride_a, stride_b, comp_item;  // row -> (row / rows_a)*stride_a + b(row % rows_a)
  int split_shift;                                 // b(x) = (x >> shift)*split_stride + (x & (2^shift-1))*stride_b
  int64_t split_stride;
  const double2* comp[MAXC];
  int n_comp;
  int64_t tiles, items;  // persistent row kernel (set by the launcher): tiles of LPC rows per item, items
  int c_phi, c_grad, ngrad, c_hess, c_sign, sign_mode, n_raw;  // component slots (-1 absent)
  double scale, tau, inv_tau;
  double* S;
  double* grad[3];
  double* hess[3];
  double* mu;
  uint8_t* mask;
  uint8_t* uf;
  double* phi_out;
  double* raw[MAXC];
  double raw_tau[MAXC];
  int64_t N;
  unsigned long long* uf_count;
  const double2* tw;
  int lmax;
};

// Per-line prefetch state of the row pass (RowCfg::FEED): xs holds the row
// being consumed / in flight; `bar` completes when it has landed.  The fetch
// sequence runs ahead of the consumption across the tiles of the persistent
// CTA: (tile, component 0..ncomp-1), (tile + gridDim.x, 0..), ...
struct RowFeed {
  double2* xs;
  uint64_t* bar;
  uint32_t phase;
  int ftile;  // tile of the next fetch
  int fcomp;  // component of the next fetch
  int ncomp;  // components per row, in order 0..ncomp-1
  int64_t froff;  // spectral-row offset of the line's row in tile ftile (-1: past the last row)
};

// c2r pre-twist of one half-spectrum row (X[k], k in [0, M]) into the complex
// line z the inverse transform consumes; src is global or a shared-memory copy.
template <class LN>
__device__ __forceinline__ void c2r_twist(double2 (&z)[LN::EPT], const double2* src, int t, const double2* twq,
                                          bool valid) {
  constexpr int MH = LN::M;
  constexpr int LQ = LN::L + 1;
#pragma unroll
  for (int r = 0; r < LN::EPT; ++r) {
    const int k = LN::out_idx(t, r);
    if (valid) {
      const double2 xa = src[k];
      const double2 xb = src[MH - k];  // conj taken below
      const double2 e = make_double2(xa.x + xb.x, xa.y - xb.y);   // X[k] + conj X[MH-k]
      const double2 d = make_double2(xa.x - xb.x, xa.y + xb.y);   // X[k] - conj X[MH-k]
      const double2 o = cmulc(d, twq_get(twq, LQ, k));            // * W_M^{-k}
      z[r] = make_double2(e.x - o.y, e.y + o.x);                  // e + i*o
    } else {
      z[r] = make_double2(0.0, 0.0);
    }
  }
}

// RCP: the ratios u_c / phi are formed as u_c * (scale / phi) (launched for
// plans with the Hessian, five ratios per node: measured C2 row -9%; with only
// the gradient the extra clamp costs more than the two divisions it saves)
template <int LH, bool RCP>
__global__ void __launch_bounds__(RowCfg<LH>::NT, RowCfg<LH>::MINB) row_kernel(const __grid_constant__ RowArgs a) {
  using LN = typename RowCfg<LH>::LN;
  constexpr int LPC = RowCfg<LH>::LPC;
  constexpr int E = LN::EPT;
  extern __shared__ double2 smem[];
  const int line = threadIdx.x / LN::TPL;
  const int t = threadIdx.x % LN::TPL;
  using RC = RowCfg<LH>;
  typename RC::XB xb{smem + line * LN::SMEM, smem + (LPC + line) * LN::SMEM, 0, 1 + line};
  double2* twq = smem + RC::NBUF * LPC * LN::SMEM;
  double2* sts = twq + RC::TWQ;
  xb_setup(xb, reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + RC::MB_OFF), line, LPC, RC::NT);
  // persistent: tiles of LPC rows, tile index fastest, then items (a.tiles per item)
  const int tiles = (int)a.tiles;
  const int total = tiles * (int)a.items;
  // spectral-row offset of this line's row in tile `tl` (false: past the last row)
  auto row_of = [&](int tl, int64_t& row, int64_t& item) -> bool {
    const int it = tl / tiles;
    row = a.row0 + (int64_t)(tl - it * tiles) * LPC + line;
    item = a.item0 + it;
    return row < a.row_end;
  };
  auto roff_of = [&](int64_t row, int64_t item) -> int64_t {
    const int64_t rb = row % a.rows_a;
    return item * a.comp_item + (row / a.rows_a) * a.stride_a + (rb >> a.split_shift) * a.split_stride +
           (rb & ((int64_t(1) << a.split_shift) - 1)) * a.stride_b;
  };
  constexpr uint32_t ROW_BYTES = (LN::M + 1) * sizeof(double2);
  RowFeed fd{nullptr, nullptr, 0u, (int)blockIdx.x, 0, a.n_raw > 0 ? a.n_raw : a.n_comp, -1};
  auto feed_tile = [&]() {  // offset of the fetch tile's row (once per tile: 64-bit divisions)
    int64_t frow, fitem;
    fd.froff = (fd.ftile < total && row_of(fd.ftile, frow, fitem)) ? roff_of(frow, fitem) : -1;
  };
  auto feed_issue = [&]() {  // thread 0 of the line: start the next fetch of the sequence
    if constexpr (RC::FEED) {
      if (fd.ftile < total) {
        if (t == 0 && fd.froff >= 0) {
          fence_proxy_async_smem();
          mbar_expect_tx(fd.bar, ROW_BYTES);
          bulk_g2s(fd.xs, a.comp[fd.fcomp] + fd.froff, ROW_BYTES, fd.bar);
        }
        if (++fd.fcomp == fd.ncomp) {
          fd.fcomp = 0;
          fd.ftile += gridDim.x;
          if (t == 0) feed_tile();
        }
      }
    }
  };
  if constexpr (RC::FEED) {
    char* fb = reinterpret_cast<char*>(smem) + ((RC::BASE_BYTES + 15) & ~size_t(15));
    fd.xs = reinterpret_cast<double2*>(fb) + (size_t)line * (LN::M + 1);
    fd.bar = reinterpret_cast<uint64_t*>(fb + (size_t)LPC * ROW_BYTES) + line;
    if (t == 0) {
      mbar_init(fd.bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (t == 0) feed_tile();
    feed_issue();
  }
  twq_fill(twq, LH + 1, a.tw, a.lmax);
  st_fill<LN>(sts, a.tw, a.lmax);
  __syncthreads();
  const bool even = (a.n_out & 1) == 0;
  unsigned cnt = 0;

#pragma unroll 1
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
  int64_t row, item;
  const bool valid = row_of(tile, row, item);
  const int64_t roff = valid ? roff_of(row, item) : item * a.comp_item;
  // the current component's row: from the prefetch buffer (waits for it) or global
  auto row_src = [&]() -> const double2* {
    if constexpr (RC::FEED) {
      if (valid) {
        mbar_wait(fd.bar, fd.phase);
        fd.phase ^= 1u;
      }
      return fd.xs;
    } else {
      return nullptr;
    }
  };
  // after the twist has read the row: every thread of the line is past it, refill
  auto feed_next = [&]() {
    if constexpr (RC::FEED) {
      xb.sync();
      feed_issue();
    }
  };
  const int64_t obase = item * a.N + row * a.n_out;

#ifndef EIK_DBG_ROW_NOST
#define EIK_DBG_ROW_NOST 0
#endif
  auto put = [&](double* dst, int r, double x0, double x1) {
    const int n = 2 * LN::in_idx(t, r);
    if (!valid || n >= a.n_out || (EIK_DBG_ROW_NOST && a.n_comp < 100)) return;
    if (even) {
      if constexpr (EIK_CS >= 2) __stcs(reinterpret_cast<double2*>(dst + obase + n), make_double2(x0, x1));
      else *reinterpret_cast<double2*>(dst + obase + n) = make_double2(x0, x1);
    } else { dst[obase + n] = x0; if (n + 1 < a.n_out) dst[obase + n + 1] = x1; }
  };
  auto putb = [&](uint8_t* dst, int r, uint8_t x0, uint8_t x1) {
    const int n = 2 * LN::in_idx(t, r);
    if (!valid || n >= a.n_out) return;
    dst[obase + n] = x0;
    if (n + 1 < a.n_out) dst[obase + n + 1] = x1;
  };
  auto active = [&](int r) { return !(LN::L > 0 && LN::upper_in(r)); };

  double2 phi[E], sg[2][E];
  double2 z[E];
  // RCP: after the S epilogue phi[] holds scale / phi (one division per node
  // instead of one per component, no extra registers; <= 1.5 ulp instead of
  // 0.5).  Nodes with phi below ~1e-300 of the scale (deep underflow: noise
  // either way) get a clamped reciprocal.
  auto ratio = [&](double2 u, int r) {
    if constexpr (RCP) return make_double2(u.x * phi[r].x, u.y * phi[r].y);
    else return make_double2((u.x * a.scale) / phi[r].x, (u.y * a.scale) / phi[r].y);
  };
  // inverse real transform of component c's row into z (prefetching the next row)
  auto row_c2r = [&](const double2* X) {
    const double2* xs = row_src();
    c2r_twist<LN>(z, xs ? xs : X, t, twq, valid);
    feed_next();
    fft_line<LN, true>(z, t, xb, TwSrc{sts, twq, LN::L + 1, 0u});
  };
  if (a.c_phi >= 0) {
    row_c2r(a.comp[a.c_phi] + roff);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if (!active(r)) continue;
      phi[r] = make_double2(z[r].x * a.scale, z[r].y * a.scale);
      const int n = 2 * LN::in_idx(t, r);
      if (valid && n < a.n_out) {
        cnt += (phi[r].x <= 0.0);
        if (n + 1 < a.n_out) cnt += (phi[r].y <= 0.0);
      }
      if (a.phi_out) put(a.phi_out, r, phi[r].x, phi[r].y);
      if (a.S) {
        const double s0 = phi[r].x > 0.0 ? (-a.tau) * log(phi[r].x) : __longlong_as_double(0x7ff8000000000000LL);
        const double s1 = phi[r].y > 0.0 ? (-a.tau) * log(phi[r].y) : __longlong_as_double(0x7ff8000000000000LL);
        put(a.S, r, s0, s1);
      }
      if (a.uf) putb(a.uf, r, phi[r].x <= 0.0, phi[r].y <= 0.0);
      if constexpr (RCP)
        phi[r] = make_double2(fmin(fmax(a.scale / phi[r].x, -1e300), 1e300),
                              fmin(fmax(a.scale / phi[r].y, -1e300), 1e300));
    }
  }
  if (a.c_grad >= 0) {
#pragma unroll 1
    for (int d = 0; d < a.ngrad; ++d) {
      row_c2r(a.comp[a.c_grad + d] + roff);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (!active(r)) continue;
        const double2 q = ratio(z[r], r);
        // kept for the Hessian epilogue only (RCP <=> Hessian plan, 2-D): the
        // gradient-only instantiations hold no ratios across components
        if constexpr (RCP) {
          if (d == 0) sg[0][r] = q; else sg[1][r] = q;
        }
        if (a.grad[d]) put(a.grad[d], r, q.x, q.y);
      }
    }
  }
  if (RCP && a.c_hess >= 0) {
#pragma unroll 1
    for (int d = 0; d < 3; ++d) {
      row_c2r(a.comp[a.c_hess + d] + roff);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (!active(r)) continue;
        const double2 tq = ratio(z[r], r);
        // xx: tq + (1/tau) sx sx, yy: tq + (1/tau) sy sy, xy: tq + (1/tau) sx sy (R/derivatives.py:102-106)
        const double2 u = (d == 1) ? sg[1][r] : sg[0][r];
        const double2 pw = (d == 0) ? sg[0][r] : sg[1][r];
        const double2 hv = make_double2(tq.x + (a.inv_tau * u.x) * pw.x, tq.y + (a.inv_tau * u.y) * pw.y);
        put(a.hess[d], r, hv.x, hv.y);
      }
    }
  }
  if (a.c_sign >= 0) {
    row_c2r(a.comp[a.c_sign] + roff);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if (!active(r)) continue;
      const double u0 = z[r].x * a.scale, u1 = z[r].y * a.scale;
      double m0, m1;
      uint8_t b0, b1;
      if (a.sign_mode == 1) {
        m0 = u0 / 6.283185307179586;
        m1 = u1 / 6.283185307179586;
        b0 = rint(m0) > 0.0; b1 = rint(m1) > 0.0;
      } else {
        m0 = -u0 / 12.566370614359172;
        m1 = -u1 / 12.566370614359172;
        b0 = rint(m0) >= 1.0; b1 = rint(m1) >= 1.0;
      }
      if (a.mu) put(a.mu, r, m0, m1);
      if (a.mask) putb(a.mask, r, b0, b1);
    }
  }
#pragma unroll 1
  for (int j = 0; j < a.n_raw; ++j) {
    row_c2r(a.comp[j] + roff);
    const double tj = a.raw_tau[j];  // tau sweep: raw_tau > 0 turns phi_j into S_j = -tau_j log phi_j
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if (!active(r)) continue;
      double x0 = z[r].x * a.scale, x1 = z[r].y * a.scale;
      if (tj > 0.0) {
        const int n = 2 * LN::in_idx(t, r);
        if (valid && n < a.n_out) {
          cnt += (x0 <= 0.0);
          if (n + 1 < a.n_out) cnt += (x1 <= 0.0);
        }
        x0 = x0 > 0.0 ? (-tj) * log(x0) : __longlong_as_double(0x7ff8000000000000LL);
        x1 = x1 > 0.0 ? (-tj) * log(x1) : __longlong_as_double(0x7ff8000000000000LL);
      }
      put(a.raw[j], r, x0, x1);
    }
  }
  }  // tiles
  if (a.uf_count) {
    const unsigned tot = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(a.uf_count, (unsigned long long)tot);
  }
}

// ---------------------------------------------------------------------------
// Impulse DFT along the last axis, one CTA per grid row:
//   T_i[item][row][k] = sum_{p in row} w_i[p] W_{M_last}^{(col_p * k) mod M_last},  k in [0, H)
// The row's points are staged in shared memory (broadcast reads), every
// thread owns a stride of frequencies, and each T value is one thread's
// in-order sum (bit-reproducible).  T then feeds the dense column pass; this
// replaces the per-column re-walk of the node lists inside the column kernel.
struct RowDftArgs {
  const int64_t* rowptr;
  const int32_t* cols;
  const double* w[3];
  int n_in;
  int64_t rows_per_item, H;
  double2* out[3];
  int64_t out_item;  // complex elements per item (rows_per_item * H)
  int64_t out_rs, out_ks;  // element (row, k) at row * out_rs + k * out_ks: (H, 1) row-major, (1, rows) transposed
  int npass;               // frequency passes per CTA (0 = 1)
  int last_shift, last_mask;
  const double2* tw;
};

constexpr int ROWDFT_NT = 256;
// Transposed T ([k1][row]) for the 2-D groups in this mask: 1 = sign, 2 = distance
// (measured: sign column kernel -22%, but one-row-per-CTA transposed writes
// cost the impulse DFT more than that; off)
#ifndef EIK_T_TRANSPOSE
#define EIK_T_TRANSPOSE 0
#endif
#ifndef EIK_T_NPASS
#define EIK_T_NPASS 2
#endif
// Row-fastest lane mapping for the transposed layout (a warp's store of one frequency is one
// run of rpb rows).  Measured with EIK_T_TRANSPOSE=1, EIK_F4K_LPC_SUM=1: C2 sign pass 0.217 ms
// -> 0.258 (4 rows per CTA) / 0.40 (8 rows): the extra frequency passes cost the row DFT more
// than the contiguous column loads save; off.
#ifndef EIK_T_REMAP
#define EIK_T_REMAP 0
#endif
#ifndef EIK_T_NPASS_RM
#define EIK_T_NPASS_RM 4
#endif
#ifndef EIK_T_MINCTA
#define EIK_T_MINCTA (148 * 16)
#endif
#ifndef EIK_ROWDFT_SPLIT
#define EIK_ROWDFT_SPLIT 1
#endif
constexpr int ROWDFT_NF = 16;     // max frequencies per thread (H <= ROWDFT_NF * ROWDFT_NT)
constexpr int ROWDFT_STAGE = 1536;  // staged points per CTA and chunk (<= 42 KB of shared memory)

// Frequencies k in [0, M/2) are spread as k = tl + q * tpr, q < NF, over tpr
// threads per row; the Nyquist term k = M/2 is one extra accumulator of the
// row's thread 0.  NF = 8 (or M/2 below 16 points: 1, 2, 4), so tpr = M/16 <= 256.
__host__ __device__ constexpr int rowdft_nf(int64_t H) { return H - 1 >= 8 ? 8 : (int)(H - 1); }
__host__ __device__ constexpr int rowdft_tpr(int64_t H) { return (int)((H - 1) / rowdft_nf(H)); }

template <int NIN, int NF>
__global__ void __launch_bounds__(ROWDFT_NT) impulse_rows_kernel(const __grid_constant__ RowDftArgs a) {
  extern __shared__ double rowdft_smem[];
  // a.npass passes over the frequencies, NF * tpr of them per pass: more rows
  // per CTA (rpb) for the transposed layout, whose k-th output run is rpb rows
  const int npass = a.npass;
  const int tpr = (int)((a.H - 1) / (NF * npass));
  const int rpb = ROWDFT_NT / tpr;
  // transposed output ([k][row]): the CTA's rows run fastest across lanes, so a warp's store
  // of one frequency is one contiguous run of rpb rows
  const bool tt = a.out_rs == 1 && EIK_T_REMAP;
  const int rl = tt ? threadIdx.x % rpb : threadIdx.x / tpr, tl = tt ? threadIdx.x / rpb : threadIdx.x % tpr;
  const int ROWDFT_CHUNK = ROWDFT_STAGE / rpb;  // per row
  const int64_t item = blockIdx.y;
  const int64_t row = (int64_t)blockIdx.x * rpb + rl;
  const bool valid = row < a.rows_per_item;
  // per-row staging: [rpb][CHUNK] columns + [NIN][rpb][CHUNK] weights
  int32_t* cols = reinterpret_cast<int32_t*>(rowdft_smem + NIN * rpb * ROWDFT_CHUNK);
  double* ws = rowdft_smem;
  const int64_t grow = item * a.rows_per_item + (valid ? row : 0);
  const int64_t p0 = valid ? __ldg(a.rowptr + grow) : 0, p1 = valid ? __ldg(a.rowptr + grow + 1) : 0;
  const int nyq_shift = a.last_shift;  // W^{(col * M/2) mod M}: index 0 or M/2 of the M-point table
  const int64_t half = a.H - 1;
  // rows of one CTA may differ in length: loop to the CTA's longest row
  __shared__ int s_maxlen;
  if (threadIdx.x == 0) s_maxlen = 0;
  __syncthreads();
  if (tl == 0) atomicMax(&s_maxlen, (int)(p1 - p0));
  __syncthreads();
  const int maxlen = s_maxlen;
  double2* dst[NIN];
#pragma unroll
  for (int i = 0; i < NIN; ++i) dst[i] = a.out[i] + item * a.out_item + row * a.out_rs;
#pragma unroll 1
  for (int pass = 0; pass < npass; ++pass) {
    const int64_t kb = (int64_t)pass * NF * tpr + tl;  // this thread's frequencies: kb + q * tpr
    double2 acc[NIN][NF], nyq[NIN];
#pragma unroll
    for (int i = 0; i < NIN; ++i) {
      nyq[i] = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < NF; ++q) acc[i][q] = make_double2(0.0, 0.0);
    }
    const bool do_nyq = tl == 0 && pass == 0;
    for (int cs = 0; cs < maxlen; cs += ROWDFT_CHUNK) {
      const int64_t left = p1 - p0 - cs;
      const int n = left <= 0 ? 0 : (left < ROWDFT_CHUNK ? (int)left : ROWDFT_CHUNK);
      __syncthreads();
      for (int q = tl; q < n; q += tpr) {
        cols[rl * ROWDFT_CHUNK + q] = __ldg(a.cols + p0 + cs + q);
#pragma unroll
        for (int i = 0; i < NIN; ++i)
          ws[(i * rpb + rl) * ROWDFT_CHUNK + q] = a.w[i] ? __ldg(a.w[i] + p0 + cs + q) : 1.0;
      }
      __syncthreads();
      for (int p = 0; p < n; ++p) {
        const int64_t col = cols[rl * ROWDFT_CHUNK + p];
        double wv[NIN];
#pragma unroll
        for (int i = 0; i < NIN; ++i) wv[i] = ws[(i * rpb + rl) * ROWDFT_CHUNK + p];
#if EIK_ROWDFT_SPLIT
        // W^{col k} = W^{col kb} * W^{col q tpr}: one gathered table read per
        // point (lane-dependent) and NF row-uniform (broadcast) reads, instead of
        // NF gathers that touch one cache line per lane
        const double2 wb = __ldg(a.tw + ((int)((col * kb) & a.last_mask) << a.last_shift));
#endif
#pragma unroll
        for (int q = 0; q < NF; ++q) {
#if EIK_ROWDFT_SPLIT
          const double2 t = q == 0 ? wb
                                   : cmul(wb, __ldg(a.tw + ((int)((col * q * tpr) & a.last_mask) << a.last_shift)));
#else
          const int64_t k = kb + (int64_t)q * tpr;
          const double2 t = __ldg(a.tw + ((int)((col * k) & a.last_mask) << a.last_shift));
#endif
#pragma unroll
          for (int i = 0; i < NIN; ++i) {
            acc[i][q].x = fma(wv[i], t.x, acc[i][q].x);
            acc[i][q].y = fma(wv[i], t.y, acc[i][q].y);
          }
        }
        if (do_nyq) {
          const double2 t = __ldg(a.tw + ((int)((col * half) & a.last_mask) << nyq_shift));
#pragma unroll
          for (int i = 0; i < NIN; ++i) {
            nyq[i].x = fma(wv[i], t.x, nyq[i].x);
            nyq[i].y = fma(wv[i], t.y, nyq[i].y);
          }
        }
      }
    }
    if (valid) {
#pragma unroll
      for (int i = 0; i < NIN; ++i) {
#pragma unroll
        for (int q = 0; q < NF; ++q) dst[i][(kb + (int64_t)q * tpr) * a.out_ks] = acc[i][q];
        if (do_nyq) dst[i][half * a.out_ks] = nyq[i];
      }
    }
  }
}

// Launch the impulse DFT for n_in inputs over `rows` rows of `items` items.
inline cudaError_t launch_impulse_rows(const RowDftArgs& ra_in, int n_in, int64_t rows, int64_t items, cudaStream_t st) {
  RowDftArgs ra = ra_in;
  if (ra.out_rs == 0) {  // default layout: row-major [row][k]
    ra.out_rs = ra.H;
    ra.out_ks = 1;
  }
  const int nf = rowdft_nf(ra.H);
  // transposed layout: EIK_T_NPASS passes so that a CTA holds >= 2 rows (whole sectors per k)
  // (row-major layout: up to EIK_T_NPASS_RM passes, i.e. that many times more
  // rows per CTA, whose node lists are staged together, while the launch keeps
  // >= EIK_T_MINCTA CTAs: C5 impulse rows -2.3% of its column pass at 4 passes;
  // C2 with 2048 rows keeps one row per CTA, 4 rows per CTA cost it +8%)
  ra.npass = 1;
  const int want = ra.out_rs == 1 ? EIK_T_NPASS : EIK_T_NPASS_RM;
  auto ctas = [&](int np) {
    const int64_t rp = ROWDFT_NT / ((ra.H - 1) / (nf * np));
    return (rows + rp - 1) / rp * items;
  };
  while (ra.npass < want && (ra.H - 1) % (nf * ra.npass * 2) == 0 && (ra.H - 1) / (nf * ra.npass * 2) >= 1 &&
         (ra.out_rs == 1 || ctas(ra.npass * 2) >= EIK_T_MINCTA))
    ra.npass *= 2;
  const int tpr = (int)((ra.H - 1) / (nf * ra.npass)), rpb = ROWDFT_NT / tpr;
  const size_t smem = (size_t)rpb * (ROWDFT_STAGE / rpb) * (n_in * sizeof(double) + sizeof(int32_t));
  const dim3 grid((unsigned)((rows + rpb - 1) / rpb), (unsigned)items);
#define EIK_ROWDFT_NF(NI, F) \
  if (n_in == NI && nf == F) impulse_rows_kernel<NI, F><<<grid, ROWDFT_NT, smem, st>>>(ra)
#define EIK_ROWDFT_NI(NI) \
  EIK_ROWDFT_NF(NI, 1); else EIK_ROWDFT_NF(NI, 2); else EIK_ROWDFT_NF(NI, 4); else EIK_ROWDFT_NF(NI, 8)
  EIK_ROWDFT_NI(1);
  else EIK_ROWDFT_NI(2);
  else EIK_ROWDFT_NI(3);
  else return cudaErrorInvalidValue;
#undef EIK_ROWDFT_NI
#undef EIK_ROWDFT_NF
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Node-list preparation: validation + per-row CSR, deterministic.

// item_off == nullptr: one item holding all K nodes (no offsets array to upload).
// Also builds the per-row CSR rowptr[r] = first node p with rowid[p] >= r
// (rows_per_item * items + 1 entries), each entry written exactly once for a
// sorted node list: node p writes the rows after its predecessor's row up to
// its own; the item's last node fills the rows after it; an empty item fills
// all of its rows.  Gaps of 32+ rows are written by the whole warp.  (Unsorted
// lists set *err = gen (the caller's run generation) and may leave rows unwritten; the buffer is zeroed at
// allocation, so stale entries stay inside the node range.)
static __global__ void __launch_bounds__(256) prep_nodes_kernel(const int64_t* __restrict__ nodes,
                                                                const int64_t* __restrict__ item_off, int64_t K,
                                                                int64_t clast, int64_t rows_per_item, int64_t N,
                                                                int64_t* __restrict__ rowid, int32_t* __restrict__ cols,
                                                                int64_t* __restrict__ rowptr, int* err, int gen) {
  const int64_t item = blockIdx.y;
  const int64_t p0 = item_off ? item_off[item] : 0, p1 = item_off ? item_off[item + 1] : K;
  const int64_t rbase = item * rows_per_item, rend = rbase + rows_per_item;  // this item's rows [rbase, rend)
  const bool last_item = item + 1 == (int64_t)gridDim.y;
  if (p0 >= p1) {  // empty item
    if (blockIdx.x == 0) {
      for (int64_t r = rbase + threadIdx.x; r < rend; r += blockDim.x) rowptr[r] = p0;
      if (last_item && threadIdx.x == 0) rowptr[rend] = p1;
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  auto row_of = [&](int64_t nd) { return rbase + (nd < 0 ? 0 : (nd >= N ? N - 1 : nd)) / clast; };
  // rows [lo, hi] get value v: short runs by the thread, long ones by the warp
  auto fill = [&](int64_t lo, int64_t hi, int64_t v) {
    const bool lng = hi - lo >= 32;
    if (!lng)
      for (int64_t r = lo; r <= hi; ++r) rowptr[r] = v;
    unsigned m = __ballot_sync(0xffffffffu, lng);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const int64_t lj = __shfl_sync(0xffffffffu, lo, j), hj = __shfl_sync(0xffffffffu, hi, j);
      const int64_t vj = __shfl_sync(0xffffffffu, v, j);
      for (int64_t r = lj + lane; r <= hj; r += 32) rowptr[r] = vj;
    }
  };
  // warp-uniform trip count (p = pw + lane)
  for (int64_t pw = p0 + blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); pw < p1;
       pw += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pw + lane;
    int64_t lo = 0, hi = -1, tlo = 0, thi = -1;
    if (p < p1) {
      const int64_t nd = nodes[p];
      const int64_t prev = p > p0 ? nodes[p - 1] : -1;
      if (nd < 0 || nd >= N || (p > p0 && prev >= nd)) atomicExch(err, gen);
      const int64_t ndc = nd < 0 ? 0 : (nd >= N ? N - 1 : nd);
      const int64_t rr = rbase + ndc / clast;
      rowid[p] = rr;
      cols[p] = (int32_t)(ndc % clast);
      lo = p > p0 ? row_of(prev) + 1 : rbase;
      hi = rr;
      if (p + 1 == p1) {  // rows after the item's last node
        tlo = rr + 1;
        thi = rend - 1;
        if (last_item) rowptr[rend] = p1;
      }
    }
    fill(lo, hi, p);
    fill(tlo, thi, p1);
  }
}

}  // namespace eik
