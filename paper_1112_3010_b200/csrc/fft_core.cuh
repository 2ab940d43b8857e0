// fp64 complex FFT building blocks for sm_100a.
//
// Shape of the engine
// -------------------
// A "line" is one 1-D transform of length M = 2^L.  It is computed by TPL
// threads, each holding EPT = 16 complex values in registers (EPT = M for
// L <= 4).  Stages are Stockham radix-R steps (R in {2,4,8,16}); between
// stages the line is exchanged through a padded shared-memory buffer.  The
// forward schedule is [R0, 16, 16, ...] (R0 absorbs L mod 4); the inverse
// schedule is its reverse, which makes the register layout of a forward
// result identical to the register layout an inverse expects as input: the
// spectral multiply happens in registers with no shared-memory round trip.
//
// Register i of thread t maps to line element
//   fwd input  / inv output : (t + (i / R0) * TPL) + (i % R0) * (M / R0)
//   fwd output / inv input  : (t + (i / RL) * TPL) + (i % RL) * (M / RL)
// (RL = last forward radix).  Zero-padded inputs (only the first M/2
// elements non-zero) and half-length outputs (only the first M/2 needed) are
// pruned inside the first/last radix step.
//
// Twiddles come from one correctly rounded table W_MAX^j = exp(-2 pi i j / MAX)
// per plan (read through the read-only path); inverse transforms use its
// conjugate.  No normalisation is applied anywhere: callers fold the exact
// power-of-two scale into their epilogue.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "bulk.cuh"
#include "tmem.cuh"

namespace eik {

#ifndef EIK_TW_POW
#define EIK_TW_POW 1
#endif
// Timing-only debug switches (results are wrong with any of them on; used by
// tools/ablate.sh to split a kernel's time into its FP64 / exchange / memory parts)
#ifndef EIK_DBG_NODFT
#define EIK_DBG_NODFT 0
#endif
#ifndef EIK_DBG_NOTW
#define EIK_DBG_NOTW 0
#endif
#ifndef EIK_DBG_NOXCHG
#define EIK_DBG_NOXCHG 0
#endif

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// a * w
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
// a * conj(w)
__device__ __forceinline__ double2 cmulc(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
}

constexpr double kC1 = 0.92387953251128675613;  // cos(pi/8)
constexpr double kS1 = 0.38268343236508977173;  // sin(pi/8)
constexpr double kR2 = 0.70710678118654752440;  // 1/sqrt(2)

// a * W16^q   (forward W16 = exp(-2 pi i/16); inverse uses the conjugate)
template <bool INV>
__device__ __forceinline__ double2 w16(double2 a, int q) {
  const double sg = INV ? -1.0 : 1.0;  // sign of the imaginary part of conj-ness
  switch (q) {
    case 0: return a;
    case 4: return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
    case 2: return INV ? make_double2((a.x - a.y) * kR2, (a.x + a.y) * kR2)
                       : make_double2((a.x + a.y) * kR2, (a.y - a.x) * kR2);
    case 6: return INV ? make_double2(-(a.x + a.y) * kR2, (a.x - a.y) * kR2)
                       : make_double2((a.y - a.x) * kR2, -(a.x + a.y) * kR2);
    default: {
      double c, s;  // W16^q = c - i*s (forward)
      if (q == 1) { c = kC1; s = kS1; }
      else if (q == 3) { c = kS1; s = kC1; }
      else if (q == 5) { c = -kS1; s = kC1; }
      else { c = -kC1; s = kS1; }  // q == 7
      s *= sg;
      return make_double2(fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s));
    }
  }
}

// Butterfly (u, x) -> (u + W16^Q x, u - W16^Q x) with the constant twiddle
// folded into FMAs: the product W16^Q x is never formed, its scale factor
// multiplies inside the final fused add (6 DP instructions instead of 8 for
// Q = 1, 2, 3, 5, 6, 7; the compiler does not contract a product used twice).
// Odd Q: W = c - i s = f (1 - i t) with f = c, t = s/c (|c| >= |s|) or
// f = s, t = c/s, |t| = tan(pi/8).
#ifndef EIK_FMA_BFLY
#define EIK_FMA_BFLY 1
#endif
constexpr double kT1 = 0.41421356237309504880;  // tan(pi/8)
template <bool INV, int Q>
__device__ __forceinline__ void bfly16(double2& a, double2& b) {
  const double2 u = a, x = b;
  if constexpr (Q == 0) {
    a = cadd(u, x);
    b = csub(u, x);
  } else if constexpr (Q == 4) {
    const double2 w = INV ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
    a = cadd(u, w);
    b = csub(u, w);
  } else if constexpr (Q == 2 || Q == 6) {
    double p, q;  // W x = kR2 * (p, q)
    if constexpr (Q == 2 && !INV) { p = x.x + x.y; q = x.y - x.x; }
    else if constexpr (Q == 2) { p = x.x - x.y; q = x.x + x.y; }
    else if constexpr (!INV) { p = x.y - x.x; q = -(x.x + x.y); }
    else { p = -(x.x + x.y); q = x.x - x.y; }
    a = make_double2(fma(p, kR2, u.x), fma(q, kR2, u.y));
    b = make_double2(fma(-p, kR2, u.x), fma(-q, kR2, u.y));
  } else {
    constexpr double c = (Q == 1) ? kC1 : (Q == 3) ? kS1 : (Q == 5) ? -kS1 : -kC1;
    constexpr double s0 = (Q == 1) ? kS1 : (Q == 3) ? kC1 : (Q == 5) ? kC1 : kS1;
    constexpr double s = INV ? -s0 : s0;
    constexpr bool bigc = (c < 0 ? -c : c) >= (s < 0 ? -s : s);
    constexpr double f = bigc ? c : s;
    constexpr double t = (c * s > 0) ? kT1 : -kT1;
    double2 y;  // W x = f * y
    if constexpr (bigc) y = make_double2(fma(t, x.y, x.x), fma(-t, x.x, x.y));
    else y = make_double2(fma(t, x.x, x.y), fma(t, x.y, -x.x));
    a = make_double2(fma(f, y.x, u.x), fma(f, y.y, u.y));
    b = make_double2(fma(-f, y.x, u.x), fma(-f, y.y, u.y));
  }
}

__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

// Compile-time bit reversal (a template constant, so register indices stay static).
template <int N, int BITS>
struct BitRev {
  static constexpr int value = BITS == 0 ? 0 : (((N & 1) << (BITS - 1)) | BitRev<(N >> 1), (BITS > 0 ? BITS - 1 : 0)>::value);
};
template <int N>
struct BitRev<N, 0> {
  static constexpr int value = 0;
};

template <int R, int N, bool HALF_IN>
__device__ __forceinline__ void perm_load(double2* x, const double2* a) {
  if constexpr (N < R) {
    if constexpr (!(HALF_IN && (N & 1))) x[N] = a[BitRev<N, ilog2c(R)>::value];
    perm_load<R, N + 1, HALF_IN>(x, a);
  }
}

// One radix-2 level of length LEN over the R registers (compile-time indices).
template <int R, int LEN, int S, int K, bool INV, bool HALF_IN>
__device__ __forceinline__ void bfly_level(double2* x) {
  if constexpr (S < R) {
    if constexpr (K < LEN / 2) {
      if constexpr (HALF_IN && LEN == 2) {
        x[S + 1] = x[S];
      } else if constexpr (EIK_FMA_BFLY) {
        bfly16<INV, K * (16 / LEN)>(x[S + K], x[S + K + LEN / 2]);
      } else {
        const double2 u = x[S + K];
        const double2 w = w16<INV>(x[S + K + LEN / 2], K * (16 / LEN));
        x[S + K] = cadd(u, w);
        x[S + K + LEN / 2] = csub(u, w);
      }
      bfly_level<R, LEN, S, K + 1, INV, HALF_IN>(x);
    } else {
      bfly_level<R, LEN, S + LEN, 0, INV, HALF_IN>(x);
    }
  }
}

template <int R, int LEN, bool INV, bool HALF_IN>
__device__ __forceinline__ void bfly_levels(double2* x) {
  if constexpr (LEN <= R) {
    bfly_level<R, LEN, 0, 0, INV, HALF_IN>(x);
    bfly_levels<R, LEN * 2, INV, HALF_IN>(x);
  }
}

// In-register R-point DFT (natural order in/out), radix-2 DIT, R <= 16.
// HALF_IN: a[R/2..R) are known zero (not read).
template <int R, bool INV, bool HALF_IN>
__device__ __forceinline__ void dft(double2* a) {
  if constexpr (EIK_DBG_NODFT) return;
  if constexpr (R > 1) {
    double2 x[R];
    perm_load<R, 0, HALF_IN>(x, a);
    bfly_levels<R, 2, INV, HALF_IN>(x);
#pragma unroll
    for (int n = 0; n < R; ++n) a[n] = x[n];
  }
}

// Quarter-wave twiddle table in shared memory: q[k] = W_Q^k = exp(-2 pi i k / Q),
// k in [0, Q/4), Q = 2^lq.  Any W_Q^j is one table read plus a quadrant rotation,
// so the table for a 4096-point line is ~19 KB instead of 64 KB.  Stage
// twiddles are read at power-of-two strides; the multi-level padding tpos()
// spreads such strides over distinct 16-byte bank groups.
__device__ __forceinline__ int tpos(int k) { return k + (k >> 3) + (k >> 6) + (k >> 9) + (k >> 12); }
__host__ __device__ constexpr int tpos_size(int n) { return n + (n >> 3) + (n >> 6) + (n >> 9) + (n >> 12) + 1; }

__device__ __forceinline__ double2 twq_get(const double2* q, int lq, int j) {
  const int qb = lq - 2;
  const int quad = (j >> qb) & 3;
  const double2 w = q[tpos(j & ((1 << qb) - 1))];
  const double2 r = (quad & 1) ? make_double2(w.y, -w.x) : w;  // * W_Q^{Q/4} = -i
  return (quad & 2) ? make_double2(-r.x, -r.y) : r;
}

// Fill the quarter table from the plan's global table W_MAX^j (MAX = 2^lmax); call
// from every thread of the block, followed by __syncthreads().
__device__ __forceinline__ void twq_fill(double2* q, int lq, const double2* __restrict__ gtw, int lmax) {
  const int n = 1 << (lq - 2);
  for (int k = threadIdx.x; k < n; k += blockDim.x) q[tpos(k)] = __ldg(gtw + ((int64_t)k << (lmax - lq)));
}

// Compile-time description of a length-2^L line transform with at most E
// elements (and radix) per thread.
// Exchange-buffer padding: element i of a line lives at slot
// i + (i >> PA) + (i >> PB) (PB = 0: no second term) and consecutive lines of a
// CTA are SMEM = pad(M-1) + 1 + XT slots apart.  The defaults suit line-major
// lines; the kernel configurations pick (PA, PB, XT) per shape so that every
// exchange store and load is free of bank conflicts (tools/bank_sim.py).
template <int L_, int E_ = 16, int PA = 3, int PB = 0, int XT = 2>
struct Line {
  static constexpr bool FOUR_STEP = false;
  static constexpr int L = L_;
  static constexpr int E = E_;
  static constexpr int LE = ilog2c(E_);
  static constexpr int M = 1 << L;
  static constexpr int EPT = (M <= E) ? M : E;
  static constexpr int TPL = M / EPT;
  static constexpr int NST = (L == 0) ? 0 : ((L <= LE) ? 1 : (L + LE - 1) / LE);
  static constexpr int R0 = (L <= LE) ? M : ((L % LE) ? (1 << (L % LE)) : E);
  static constexpr int RL = (NST <= 1) ? R0 : E;
  __host__ __device__ static constexpr int pad(int i) { return i + (i >> PA) + (PB ? (i >> PB) : 0); }
  static constexpr int SMEM = pad(M - 1) + 1 + XT;  // padded double2 slots per line
  static constexpr int TWQ = tpos_size((L >= 2) ? (M >> 2) : 1);  // quarter-table slots (own resolution)
  __host__ __device__ static constexpr int frad(int s) { return s == 0 ? R0 : E; }
  __host__ __device__ static constexpr int rad(bool inv, int s) { return inv ? frad(NST - 1 - s) : frad(s); }
  __host__ __device__ static constexpr int ns(bool inv, int s) { return s == 0 ? 1 : ns(inv, s - 1) * rad(inv, s - 1); }
  // element index held by register i of thread t
  __device__ static __forceinline__ int in_idx(int t, int i) {   // forward input / inverse output
    return (t + (i / R0) * TPL) + (i % R0) * (M / R0);
  }
  __device__ static __forceinline__ int out_idx(int t, int i) {  // forward output / inverse input
    return (t + (i / RL) * TPL) + (i % RL) * (M / RL);
  }
  // register i is a structurally-zero input of a half-padded forward transform
  __device__ static __forceinline__ constexpr bool upper_in(int i) { return (i % R0) >= (R0 / 2); }

  // Per-stage twiddle tables (shared memory).  Stage (NS, R) needs
  // W_{NS*R}^{k*r}, k < NS, 1 <= r < R.  With k = 16*k_hi + k_lo the table
  // holds lo[k_lo][r] = W^{k_lo*r} and hi[k_hi][r] = W^{16*k_hi*r}; a twiddle
  // is lo * hi (one product) or lo alone when NS <= 16.  Consecutive threads
  // differ in k_lo and read rows R-1 entries apart (odd stride: no bank
  // conflicts); k_hi is shared by 16 threads (broadcast).  The inverse
  // schedule reuses the forward tables when it has the same stage types.
  static constexpr bool INV_SHARES = (R0 == E);
  __host__ __device__ static constexpr int st_lo(bool inv, int s) { return ns(inv, s) < 16 ? ns(inv, s) : 16; }
  // two-level (lo * hi) tables for radix <= 8 lines; radix-16 stages with NS > 16
  // read the quarter-wave table instead (measured faster: 15 extra products per
  // butterfly cost more than one rotated table read)
  static constexpr bool TWO_LEVEL = (E <= 8);
  __host__ __device__ static constexpr bool st_quarter(bool inv, int s) { return !TWO_LEVEL && ns(inv, s) > 16; }
  __host__ __device__ static constexpr int st_hi(bool inv, int s) {
    return (ns(inv, s) > 16 && TWO_LEVEL) ? ns(inv, s) / 16 : 0;
  }
  __host__ __device__ static constexpr int st_size(bool inv, int s) {
    return (s == 0 || st_quarter(inv, s)) ? 0 : (st_lo(inv, s) + st_hi(inv, s)) * (rad(inv, s) - 1);
  }
  __host__ __device__ static constexpr int st_off(bool inv, int s) {
    int o = 0;
    if (inv && INV_SHARES) inv = false;
    if (inv)
      for (int j = 1; j < NST; ++j) o += st_size(false, j);
    for (int j = 1; j < s; ++j) o += st_size(inv, j);
    return o;
  }
  __host__ __device__ static constexpr int st_total() {
    int o = 0;
    for (int j = 1; j < NST; ++j) o += st_size(false, j) + (INV_SHARES ? 0 : st_size(true, j));
    return o < 1 ? 1 : o;
  }
  static constexpr int ST_SIZE = st_total();  // double2 slots of all stage tables
};

// Fill the stage tables of line type LN from the global table W_MAX^j.
template <class LN, bool INV, int S>
__device__ __forceinline__ void st_fill_stage(double2* sts, const double2* __restrict__ gtw, int lmax) {
  if constexpr (S < LN::NST) {
    if constexpr (S >= 1 && !(INV && LN::INV_SHARES)) {
      constexpr int NS = LN::ns(INV, S), R = LN::rad(INV, S);
      constexpr int NLO = LN::st_lo(INV, S), SZ = LN::st_size(INV, S), OFF = LN::st_off(INV, S);
      const int sh = lmax - ilog2c(NS * R);
      for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
        const int row = i / (R - 1), r = i % (R - 1) + 1;
        const int m = row < NLO ? row * r : 16 * (row - NLO) * r;
        sts[OFF + i] = __ldg(gtw + ((int64_t)m << sh));
      }
    }
    st_fill_stage<LN, INV, S + 1>(sts, gtw, lmax);
  }
}
template <class LN>
__device__ __forceinline__ void st_fill(double2* sts, const double2* __restrict__ gtw, int lmax) {
  if constexpr (LN::FOUR_STEP) {
    for (int i = threadIdx.x; i < LN::ST_SIZE; i += blockDim.x) {  // W_256^{j a}, row j, column a-1
      const int j = i / 15, a = i % 15 + 1;
      sts[i] = __ldg(gtw + ((int64_t)(j * a) << (lmax - 8)));
    }
  } else {
    st_fill_stage<LN, false, 0>(sts, gtw, lmax);
    st_fill_stage<LN, true, 0>(sts, gtw, lmax);
  }
}

// Twiddle sources of a line: stage tables + the quarter-wave table (resolution 2^lq >= M).
struct TwSrc {
  const double2* st;
  const double2* q;
  int lq;
  uint32_t tm;  // TMEM address of this thread's cached radix-16 quarter-stage twiddles (0 = none)
  uint32_t tm2 = 0;  // TMEM address of the last inverse stage's twiddles (radix < 16, NS > 16; 0 = none)
};

template <class LN, bool INV, int S>
__device__ __forceinline__ double2 st_tw(const TwSrc& tw, int k, int r) {
  constexpr int NS = LN::ns(INV, S), R = LN::rad(INV, S);
  constexpr int NLO = LN::st_lo(INV, S), OFF = LN::st_off(INV, S);
  const double2* sts = tw.st;
  if constexpr (LN::st_quarter(INV, S)) {
    return twq_get(tw.q, tw.lq, (k * r) << (tw.lq - ilog2c(NS * R)));
  } else if constexpr (NS <= 16) {
    return sts[OFF + k * (R - 1) + (r - 1)];
  } else {
    const double2 lo = sts[OFF + (k & 15) * (R - 1) + (r - 1)];
    const double2 hi = sts[OFF + (NLO + (k >> 4)) * (R - 1) + (r - 1)];
    return cmul(lo, hi);
  }
}

// Exchange buffers of one line.  With NBUF = 2 consecutive exchanges alternate
// between two buffers, so a stage needs one barrier (between its writes and
// its reads): writes of exchange k+2 cannot overtake reads of exchange k
// because every thread passed the barrier of exchange k+1.
// SYNC selects the barrier that covers exactly the threads of one line:
// 0 = the CTA (__syncthreads), 1 = the warp (lines of <= 32 threads, whole
// lines per warp), 2 = named barrier `bar` over the NTH threads of the line
// (line-major CTAs holding several lines), so lines of a CTA do not wait on
// each other.
// With NBUF = 1 the second barrier of an exchange ("every thread has read the
// buffer, it may be written again") is split-phase (EIK_XSPLIT): release()
// after a thread's reads is one mbarrier arrival per warp and does not block;
// acquire() before its next write into the buffer waits for that phase, which
// by then (a radix stage of FP64 work later) has normally completed, so warps
// start their butterflies as their own loads return instead of after the
// slowest warp's.  `mb` is the line group's mbarrier (count = its warps).
// Measured (B200): C2 step 0.819 -> 0.805 ms (column kernel 0.3225 -> 0.3176,
// sign column kernel 0.2226 -> 0.2173, row 0.2601 -> 0.2564), C5 8.077 -> 8.021 ms,
// TS 1.009 -> 0.994 ms; the register-resident col / lines kernels (ColCfg) keep
// the blocking barrier (C3's axis-1 inverse measured 0.812 -> 0.829 ms with it).
#ifndef EIK_XSPLIT
#define EIK_XSPLIT 1
#endif
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
template <int NBUF, int SYNC = 0, int NTH = 0, bool SPLIT_OK = true>
struct XBuf {
  double2* b0;
  double2* b1;
  int ph;
  int bar;
  uint64_t* mb;
  uint32_t par;
  static constexpr bool SPLIT = EIK_XSPLIT && SPLIT_OK && NBUF == 1 && SYNC != 1;
  __device__ __forceinline__ double2* cur() const { return (NBUF == 2 && ph) ? b1 : b0; }
  __device__ __forceinline__ void sync() const {
    if constexpr (SYNC == 1) __syncwarp();
    else if constexpr (SYNC == 2) asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "n"(NTH) : "memory");
    else __syncthreads();
  }
  // this thread has finished reading the buffer
  __device__ __forceinline__ void release() {
    if constexpr (NBUF == 2) {
      ph ^= 1;
    } else if constexpr (SPLIT) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(mb);
    } else {
      sync();
    }
  }
  // before this thread's next write into the buffer
  __device__ __forceinline__ void acquire() {
    if constexpr (SPLIT) {
      mbar_wait(mb, par ^ 1u);
      par ^= 1u;
    }
  }
  __device__ __forceinline__ void done() { release(); }
  // threads of one sync group's mbarrier (its warps arrive once per release)
  __host__ __device__ static constexpr int group_warps(int cta_threads) { return (SYNC == 2 ? NTH : cta_threads) / 32; }
};

// One Stockham stage S of direction INV, followed (if not last) by the
// shared-memory exchange into the next stage's register layout.
// twq: shared quarter table at resolution 2^lq (lq >= L).
template <class LN, bool INV, int S, bool HALF_IN, class XB>
__device__ __forceinline__ void stage(double2 (&v)[LN::EPT], int t, XB& xb, const TwSrc& tw) {
  constexpr int R = LN::rad(INV, S);
  constexpr int NS = LN::ns(INV, S);
  constexpr int G = LN::EPT / R;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int b = t + g * LN::TPL;
    if constexpr (NS > 1 && !EIK_DBG_NOTW) {
      const int k = b & (NS - 1);
      bool done = false;
      if constexpr (LN::st_quarter(INV, S) && G == 1 && R == 16) {
        if (tw.tm) {  // per-thread constants cached in TMEM: 4 x (16-word load, wait), no table math
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t w32[16];
            tmem_ld16(tw.tm + 16 * c, w32);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int r = 4 * c + q;  // TMEM holds W^{k r} at complex slot r (slot 0 unused)
              if (r >= 1) {
                const double2 w = make_double2(
                    __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 1] << 32) | w32[4 * q])),
                    __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 3] << 32) | w32[4 * q + 2])));
                v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
              }
            }
          }
          done = true;
        }
      }
      if constexpr (INV && S == LN::NST - 1 && S > 0 && LN::st_quarter(INV, S) && R < 16 && R * G == 16) {
        if (tw.tm2) {  // per-thread constants W^{k r}, group g at R complex slots (slot 0 unused)
          double2 w[R];
          tmem_get<R>(tw.tm2 + 4 * R * g, w);
#pragma unroll
          for (int r = 1; r < R; ++r) v[g * R + r] = cmulc(v[g * R + r], w[r]);
          done = true;
        }
      }
      if (!done) {
        if constexpr (EIK_TW_POW && LN::TWO_LEVEL && R > 2) {
          // radix <= 8 lines: W^{k r} as powers of W^k (one table lookup per
          // group instead of R-1, or 2(R-1) for two-level stages); products in
          // registers trade shared-memory wavefronts for FP64 issue
          const double2 w1 = st_tw<LN, INV, S>(tw, k, 1);
          double2 w = w1;
#pragma unroll
          for (int r = 1; r < R; ++r) {
            if (r > 1) w = cmul(w, w1);
            v[g * R + r] = INV ? cmulc(v[g * R + r], w) : cmul(v[g * R + r], w);
          }
        } else {
#pragma unroll
          for (int r = 1; r < R; ++r) {
            const double2 w = st_tw<LN, INV, S>(tw, k, r);
            v[g * R + r] = INV ? cmulc(v[g * R + r], w) : cmul(v[g * R + r], w);
          }
        }
      }
    }
    dft<R, INV, HALF_IN && S == 0>(&v[g * R]);
  }
  if constexpr (S + 1 < LN::NST && !EIK_DBG_NOXCHG) {
    xb.acquire();
    double2* sm = xb.cur();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int b = t + g * LN::TPL;
      const int o = (b / NS) * NS * R + (b & (NS - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) sm[LN::pad(o + r * NS)] = v[g * R + r];
    }
    xb.sync();
    constexpr int R2 = LN::rad(INV, S + 1);
    constexpr int G2 = LN::EPT / R2;
#pragma unroll
    for (int g = 0; g < G2; ++g) {
      const int b = t + g * LN::TPL;
#pragma unroll
      for (int r = 0; r < R2; ++r) v[g * R2 + r] = sm[LN::pad(b + r * (LN::M / R2))];
    }
    xb.done();
  }
}

// Fill this thread's TMEM copy of the last inverse stage's twiddles (TwSrc::tm2).
template <class LN>
__device__ __forceinline__ void tw_last_inv_fill(uint32_t tm2, int t, const double2* q, int lq) {
  constexpr int S = LN::NST - 1;
  constexpr int R = LN::rad(true, S), NS = LN::ns(true, S), G = LN::EPT / R;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int k = (t + g * LN::TPL) & (NS - 1);
    double2 w[R];
    w[0] = make_double2(1.0, 0.0);
#pragma unroll
    for (int r = 1; r < R; ++r) w[r] = twq_get(q, lq, (k * r) << (lq - ilog2c(NS * R)));
    tmem_put<R>(tm2 + 4 * R * g, w);
  }
}

template <class LN, bool INV, int S, bool HALF_IN, class XB>
__device__ __forceinline__ void stages_from(double2 (&v)[LN::EPT], int t, XB& xb, const TwSrc& tw) {
  if constexpr (S < LN::NST) {
    stage<LN, INV, S, HALF_IN>(v, t, xb, tw);
    stages_from<LN, INV, S + 1, HALF_IN>(v, t, xb, tw);
  }
}

// ---------------------------------------------------------------------------
// 4096-point lines as 16 x 256 ("four-step"), 256 threads per line.
//
// The Stockham schedule exchanges the whole line through shared memory twice
// per transform, each time with CTA-wide barriers, so the 8 warps of a CTA
// move in lock-step between the FP64 and the shared-memory phases.  Here
// n = n2 + 256 n1 and k = k1 + 16 k2: a 16-point DFT over n1 in registers
// (thread t = n2), the twiddle W_4096^{n2 k1} (per-thread constants), ONE
// CTA-wide exchange that hands row k1 to half-warp k1, then the 256-point DFT
// of that row inside its half-warp (16 x 16, exchange through the row's own
// buffer with __syncwarp only).  Forward output / inverse input layout:
//   register i of thread t holds k = (t >> 4) + 16 (t & 15) + 256 i
// Forward input / inverse output: n = t + 256 i (as the Stockham layout).
// Exchange buffer: 16 rows of PITCH slots; the in-row 16 x 16 transpose uses
// a stride of 17 so both sides are free of bank conflicts.
struct Line4K {
  static constexpr bool FOUR_STEP = true;
  static constexpr int L = 12, E = 16, M = 4096, EPT = 16, TPL = 256, R0 = 16, RL = 16, NST = 3;
  static constexpr int PITCH = 272;
  static constexpr int SMEM = 16 * PITCH + 4;  // line stride: == 4 (mod 8) so lane-interleaved lines miss each other's banks
  static constexpr int TWQ = tpos_size(M >> 2);
  static constexpr bool INV_SHARES = true;
  static constexpr int ST_SIZE = 16 * 15;  // W_256^{j a}, j < 16, 1 <= a < 16
  __device__ static __forceinline__ int in_idx(int t, int i) { return t + 256 * i; }
  __device__ static __forceinline__ int out_idx(int t, int i) { return (t >> 4) + 16 * (t & 15) + 256 * i; }
  __device__ static __forceinline__ constexpr bool upper_in(int i) { return i >= 8; }
};

// v[r] *= W_4096^{t r} (or its conjugate), r = 1..15: TMEM cache or quarter table
template <bool INV>
__device__ __forceinline__ void f4k_twiddle_t(double2 (&v)[16], int t, const TwSrc& tw) {
  if constexpr (EIK_DBG_NOTW) return;
  if (tw.tm) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t w32[16];
      tmem_ld16(tw.tm + 16 * c, w32);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = 4 * c + q;
        if (r >= 1) {
          const double2 w = make_double2(
              __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 1] << 32) | w32[4 * q])),
              __longlong_as_double((long long)(((unsigned long long)w32[4 * q + 3] << 32) | w32[4 * q + 2])));
          v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
        }
      }
    }
  } else {
#pragma unroll
    for (int r = 1; r < 16; ++r) {
      const double2 w = twq_get(tw.q, tw.lq, (t * r) << (tw.lq - 12));
      v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
    }
  }
}

// v[r] *= W_256^{x r} (or conjugate), x = t & 15, from the stage table
template <bool INV>
__device__ __forceinline__ void f4k_twiddle_row(double2 (&v)[16], int x, const TwSrc& tw) {
  if constexpr (EIK_DBG_NOTW) return;
  const double2* row = tw.st + x * 15 - 1;
#pragma unroll
  for (int r = 1; r < 16; ++r) v[r] = INV ? cmulc(v[r], row[r]) : cmul(v[r], row[r]);
}

// XB::sync() is the barrier over the threads of this line: the CTA when its
// lines are interleaved across all warps, a named barrier for line-major CTAs
// HOOK: called by every thread right after the transform's first CTA-wide
// barrier (the column kernels issue their pending TMA output stores there).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

template <bool HALF_IN, class XB, class HOOK = NoHook>
__device__ __forceinline__ void f4k_forward(double2 (&v)[16], int t, XB& xb, const TwSrc& tw,
                                            const HOOK& hook = HOOK()) {
  constexpr int P = Line4K::PITCH;
  double2* sm = xb.b0;
  const int g = t >> 4, x = t & 15;
  double2* row = sm + g * P;
  dft<16, false, HALF_IN>(v);  // over n1: v[k1], thread t = n2
  f4k_twiddle_t<false>(v, t, tw);
  if constexpr (!EIK_DBG_NOXCHG) {
  xb.acquire();  // every thread is done with the buffer (previous transform)
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[r * P + t] = v[r];
  xb.sync();
  hook();
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = row[x + 16 * m];  // row k1 = g, n2 = x + 16 m
  }
  dft<16, false, false>(v);                             // over m: v[a], lane x = j
  f4k_twiddle_row<false>(v, x, tw);
  if constexpr (!EIK_DBG_NOXCHG) {
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 16; ++a) row[a * 17 + x] = v[a];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = row[x * 17 + j];  // lane x = a
  xb.release();  // (the next transform may write any row once every warp is here)
  }
  dft<16, false, false>(v);                             // over j: v[b] = X[g + 16 x + 256 b]
}

template <class XB, class HOOK = NoHook>
__device__ __forceinline__ void f4k_inverse(double2 (&v)[16], int t, XB& xb, const TwSrc& tw,
                                            const HOOK& hook = HOOK()) {
  constexpr int P = Line4K::PITCH;
  double2* sm = xb.b0;
  const int g = t >> 4, x = t & 15;
  double2* row = sm + g * P;
  dft<16, true, false>(v);  // over b: v[j], lane x = a
  f4k_twiddle_row<true>(v, x, tw);
  if constexpr (!EIK_DBG_NOXCHG) {
  xb.acquire();  // the previous transform's CTA-wide reads of this row are done
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) row[x * 17 + j] = v[j];
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 16; ++a) v[a] = row[a * 17 + x];  // lane x = j
  }
  dft<16, true, false>(v);                              // over a: v[m] = z[x + 16 m]
  if constexpr (!EIK_DBG_NOXCHG) {
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 16; ++m) row[x + 16 * m] = v[m];
  xb.sync();
  hook();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = sm[r * P + t];  // thread t = n2: v[k1]
  xb.release();  // buffer free again once every warp is here: the next transform may write any row
  }
  f4k_twiddle_t<true>(v, t, tw);
  dft<16, true, false>(v);  // over k1: v[i] = x[t + 256 i]
}

// Full transform of the line held in v (layouts documented above).
// HALF_IN (forward only): input elements >= M/2 are zero and their registers are not read.
template <class LN, bool INV, bool HALF_IN = false, class XB, class HOOK = NoHook>
__device__ __forceinline__ void fft_line(double2 (&v)[LN::EPT], int t, XB& xb, const TwSrc& tw,
                                         const HOOK& hook = HOOK()) {
  static_assert(!(INV && HALF_IN), "input pruning is a forward-transform feature");
  if constexpr (LN::FOUR_STEP) {
    if constexpr (INV) f4k_inverse(v, t, xb, tw, hook);
    else f4k_forward<HALF_IN>(v, t, xb, tw, hook);
  } else {
    stages_from<LN, INV, 0, HALF_IN && (LN::L > 0)>(v, t, xb, tw);
  }
}

}  // namespace eik
