/* eikfld_b200 — C ABI of the B200-native FFT-convolution distance transform.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `eikfld` (/root/reference/pkg/src/eikfld).  The reference is pure Python and
 * has no FFI of its own; its "operator API" for this path is the module API
 * listed below.  Each entry point names the reference functions whose work it
 * replaces (file:line, R/ = /root/reference/pkg/src/eikfld/).  The Python
 * package `paper_1112_3010_b200` binds these with ctypes and re-exposes the
 * reference signatures (see INTEGRATION.md for the binding a maintainer of the
 * reference would add).
 *
 * Conventions
 *   - plain pointers and sizes only; no exceptions cross the ABI;
 *   - fields are float64, row-major (last axis fastest), N = prod(counts) per grid;
 *   - node lists are flat indices (np.ravel_multi_index order), strictly
 *     increasing within each item (np.unique order, R/grid.py:112-114);
 *   - by default every pointer is a device pointer and work is queued on
 *     `stream` (a cudaStream_t, NULL = legacy default stream) without a host
 *     sync; EIK_HOST_INPUTS / EIK_HOST_OUTPUTS make the library stage host
 *     buffers itself (pinned host memory gives the best copy rate);
 *   - status codes: 0 ok, 1 validation, 2 underflow (phi <= 0 somewhere;
 *     only reported when EIK_CHECK_UNDERFLOW is set), 3 CUDA/OOM;
 *   - device-resident asynchronous eik_run calls (no EIK_HOST_*, EIK_SYNC,
 *     EIK_CHECK_UNDERFLOW, EIK_PROFILE, n_underflow) repeated with identical
 *     arguments are replayed as one CUDA graph from the second call on (the
 *     buffers' contents may change between calls, their addresses may not;
 *     environment EIK_GRAPH=0 disables this);
 *   - a plan is reentrant for calls on one stream at a time; distinct plans are
 *     independent.  No floating-point atomics are used on value paths, so
 *     results are bit-reproducible run to run.
 */
#ifndef EIKFLD_B200_H
#define EIKFLD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIK_OK 0
#define EIK_EVALIDATION 1
#define EIK_EUNDERFLOW 2
#define EIK_ECUDA 3

/* plan field bits: which kernel spectra a plan caches */
#define EIK_FIELD_PHI 0x1u     /* phi = exp(-|x|/tau) * delta_Y      R/distance.py:63-86   */
#define EIK_FIELD_S 0x2u       /* S = -tau log phi                   R/distance.py:89-122  */
#define EIK_FIELD_GRAD 0x4u    /* grad S ratios                      R/derivatives.py:64-79,156-172 */
#define EIK_FIELD_HESS 0x8u    /* (S_xx, S_yy, S_xy), 2-D only       R/derivatives.py:82-112 */
#define EIK_FIELD_WINDING 0x10u /* winding number mu, 2-D           R/sign.py:108-132 */
#define EIK_FIELD_DEGREE 0x20u /* topological degree mu, 3-D        R/sign.py:135-163 */

/* run flags */
#define EIK_HOST_INPUTS 0x1u
#define EIK_HOST_OUTPUTS 0x2u
#define EIK_SYNC 0x4u              /* synchronize the stream before returning */
#define EIK_CHECK_UNDERFLOW 0x8u   /* sync, and return EIK_EUNDERFLOW if any phi <= 0
                                      (R/convolution.py:378-388 assert_positive) */
#define EIK_PROFILE 0x10u          /* record CUDA events around each pass (see eik_pass_times) */
#define EIK_SLAB_P2P 0x20u         /* slab passes: exchange through peer arenas (eik_slab_p2p_*) */
#define EIK_ASYNC 0x40u            /* host outputs: return once queued (no host sync, no result checks);
                                      the outputs are complete when the stream is; consecutive calls on
                                      one plan overlap the next column passes with this D2H */

/* pass ids reported by eik_pass_times */
#define EIK_PASS_PREP 0     /* node validation + per-row CSR */
#define EIK_PASS_COL 1      /* fused column kernel, distance group (impulse DFT, fwd, multiply, inverses) */
#define EIK_PASS_COL_SIGN 2 /* fused column kernel, sign group */
#define EIK_PASS_LINES 3    /* 3-D inverse along axis 1 */
#define EIK_PASS_ROW 4      /* c2r along the last axis + epilogue */
#define EIK_PASS_COL_KERNEL 5 /* the distance group's column / axis-0 kernel alone (inside EIK_PASS_COL) */
#define EIK_NPASS 6

typedef struct eik_plan eik_plan;

typedef struct {
  /* unit impulses delta_Y (R/distance.py:50-60): sorted distinct flat nodes */
  const int64_t* nodes;
  const int64_t* item_offsets; /* batch+1 offsets into nodes; NULL when batch == 1 */
  int64_t n_nodes;             /* total nodes over all items */
  int64_t batch;               /* independent grids sharing this plan (>= 1) */
  /* weighted impulses for the sign field: sorted distinct flat nodes and
     dim weight rows (weights[a*n_sign_nodes + p]); 2-D: chord tangents
     accumulated per node (R/sign.py:42-57); 3-D: area-weighted normals
     accumulated per node (R/sign.py:68-86).  Batch 1 only. */
  const int64_t* sign_nodes;
  int64_t n_sign_nodes;
  const double* sign_weights;
} eik_inputs;

typedef struct {
  /* every pointer may be NULL (not computed); sizes are batch * N */
  double* phi;        /* raw convolution phi */
  double* S;          /* -tau log phi, NaN where phi <= 0 */
  double* grad[3];    /* S_a = (f_a exp * delta)/(exp * delta), reference axis order */
  double* hess[3];    /* S_xx, S_yy, S_xy (2-D) */
  double* mu;         /* winding (2-D) or degree (3-D) field */
  uint8_t* mask;      /* classify(mu) of R/sign.py:166-198: rint(mu) > 0 (2-D) / rint(mu) >= 1 (3-D), the
                         flagged (sign) nodes taking their nearest unflagged node's class with
                         scipy's EDT ties (eik_run; slab ranks: eik_slab_fill) */
  uint8_t* underflow; /* 1 where phi <= 0 */
  int64_t* n_underflow;        /* host scalar, written when the call synchronizes */
  unsigned long long* d_underflow_count; /* optional device counter (accumulated) */
} eik_outputs;

/* Build a plan for a grid: padded lengths, twiddles and the cached kernel
 * spectra for `fields` (replaces the per-call kernel sampling + forward FFTs of
 * R/distance.py:22-47, R/derivatives.py:26-57,139-153, R/sign.py:97-105 and
 * FftConvolver.__init__/kernel_hat, R/convolution.py:220-251). */
int eik_plan_create(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields,
                    int device, eik_plan** out);
/* Same, but the cached kernel spectra cover only the spectral planes
 * k1 in [k1_begin, k1_begin + k1_count) (3-D slab ranks; k1_count < 0 = all). */
int eik_plan_create_slab(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields,
                         int device, int64_t k1_begin, int64_t k1_count, eik_plan** out);
int eik_plan_destroy(eik_plan* plan);
/* padded[3], spectral lines per item, device bytes held */
int eik_plan_info(const eik_plan* plan, int64_t* padded, int64_t* lines, int64_t* device_bytes);

/* One pass of the hot path over a batch: phi, S, gradient, Hessian from one
 * shared transform of delta_Y plus the sign field (R/distance.py:114-122,
 * R/derivatives.py:64-112, R/sign.py:108-163).
 * 3-D plans keep their kernel spectra folded along all three axes (every
 * kernel is even or odd per axis).  A 3-D run of one item whose fused buffers
 * (one spectrum per input, one per component) would not fit the device runs
 * the streamed schedule instead: one spectrum slot and one component slot,
 * one axis-0 pass per component, the epilogue applied elementwise at the end
 * (same arithmetic per node; C4 at 1024^3 on one 180 GB GPU).  EIK_STREAM3D=1/0
 * in the environment forces / forbids it. */
int eik_run(eik_plan* plan, const eik_inputs* in, const eik_outputs* out, uint32_t flags, void* stream);

/* Engine-level linear convolution of n_kernels centred kernels (each of shape
 * kshape, odd, >= 2c-1 per axis) with one dense field on the grid
 * (FftConvolver.convolve/convolve_many, R/convolution.py:317-366).  kernels:
 * n_kernels * prod(kshape) doubles; field: N doubles; out: n_kernels * N. */
int eik_convolve(int dim, const int64_t* counts, const double* kernels, int64_t n_kernels,
                 const int64_t* kshape, const double* field, double* out, uint32_t flags, int device,
                 void* stream);

/* Slab-decomposed 3-D pipeline.  A rank owns the
 * real-space planes [i0_begin, i0_begin + c0_local) (c0 = G * c0_local) and the
 * spectral planes k1 in [k1_begin, k1_begin + ks) (M1 = G * ks).  Device
 * pointers only; complex buffers are interleaved double pairs.  Between the
 * three passes the caller runs one all-to-all (NCCL) per buffer:
 *   eik_slab_planes   impulse DFT along axis 2 + FFT along axis 1 of the owned
 *                     planes (node indices relative to the slab, sorted).  Writes
 *                     V[i] packed by destination k1-slab: [G][c0_local][ks][H2]
 *                     (H2 = M2/2+1); group 0: delta_Y (1 buffer), group 1: the
 *                     three flux components (weights[3 * n_nodes]).
 *   eik_slab_axis0    after the exchange, V[i] = [c0][ks][H2] for this rank's
 *                     k1-slab: fused axis-0 FFT, kernel-spectrum multiply and
 *                     inverse; writes W_j = [c0][ks][H2] per component (group 0:
 *                     phi + 3 gradient numerators; group 1: the degree sum).
 *   eik_slab_finish   after the exchange back, W_j = [G][c0_local][ks][H2]:
 *                     inverse along axis 1, c2r along axis 2 and the epilogue
 *                     for the owned planes (outputs sized c0_local * c1 * c2).
 * eik_run on a 3-D plan is exactly these passes with G = 1 and no exchange. */
int eik_slab_planes(eik_plan* plan, int group, const int64_t* nodes, int64_t n_nodes, const double* weights,
                    int64_t c0_local, int64_t ks, double* const* v_out, uint32_t flags, void* stream);
int eik_slab_axis0(eik_plan* plan, int group, double* const* v_in, int64_t k1_begin, int64_t ks,
                   double* const* w_out, uint32_t flags, void* stream);
int eik_slab_finish(eik_plan* plan, double* const* w, int64_t c0_local, int64_t ks, const eik_outputs* out,
                    uint32_t flags, void* stream);

/* Peer-to-peer slab exchange: the two all-to-alls fused into the passes.
 * Each rank's plan owns one device arena of (4 + n_comp) slots, each slot
 * G * c0_local * ks * H2 complex in the receive layout [G src][c0_local][ks][H2]
 * (V slots: 0 = delta_Y, 1..3 = flux fields; then one W slot per component).
 * With EIK_SLAB_P2P, eik_slab_planes stores its k1-slab blocks straight into
 * the owning rank's V slots and eik_slab_axis0 stores its rows straight into
 * the owning rank's W slots (NVLink stores through peer pointers, overlapped
 * with the transforms); both read / eik_slab_finish reads the own arena and
 * ignore their buffer arguments.  No data collective remains: the caller
 * orders the ranks with a stream-ordered barrier after each planes pass and
 * after the last axis-0 pass (replacing the reference-free NCCL schedule's
 * one all-to-all per buffer).  c0_local must be a power of two; G <= 8.
 *   eik_slab_p2p_init     allocate the arena; return its device pointer, size
 *                         and (ipc_handle != NULL) its 64-byte CUDA IPC handle.
 *   eik_slab_p2p_connect  peer arenas by device pointer (same process: the
 *                         single-GPU emulation) or by IPC handle (world * 64
 *                         bytes, one process per GPU); the own entry is ignored. */
int eik_slab_p2p_init(eik_plan* plan, int world, int rank, int64_t c0_local, int64_t ks, void** arena,
                      int64_t* arena_bytes, void* ipc_handle);
int eik_slab_p2p_connect(eik_plan* plan, void* const* peer_arenas, const void* ipc_handles);

/* Streamed slab schedule: one input and one component at a time, so a rank
 * holds one V and one W buffer pair instead of one per input and component
 * (C4 at 1024^3 on 2 GPUs; eik_run does the same on one GPU).  eik_slab_planes_one:
 * the planes pass of the distance input (group 0) or of flux input `input` in
 * 0..2 (group 1; weights is the full [3][n_nodes] array).  eik_slab_axis0_one:
 * W (+)= IFFT0(K FFT0(V)) for one kernel (0 exp, 1..3 gradient, 4..6 degree);
 * accumulate != 0 adds into W (the degree sums its three inputs).
 * eik_slab_finish_raw: inverse along axis 1 + c2r of ONE component into the
 * scaled real-space field raw_out (no epilogue).  eik_slab_epilogue: the
 * elementwise epilogue over the rank's n_local nodes: S = -tau log phi_raw,
 * out->grad[a] (holding the raw numerators) /= phi_raw, mu = -mu_raw / 4 pi,
 * mask = rint(mu) >= 1 -- the operations of the fused row epilogue. */
int eik_slab_planes_one(eik_plan* plan, int group, int input, const int64_t* nodes, int64_t n_nodes,
                        const double* weights, int64_t c0_local, int64_t ks, double* v_out, void* stream);
int eik_slab_axis0_one(eik_plan* plan, int kernel, const double* v_in, int64_t k1_begin, int64_t ks, double* w_out,
                       int accumulate, void* stream);
int eik_slab_finish_raw(eik_plan* plan, double* w, int64_t c0_local, int64_t ks, double* raw_out, void* stream);
int eik_slab_epilogue(eik_plan* plan, int64_t n_local, const double* phi_raw, const double* mu_raw,
                      const eik_outputs* out, void* stream);

/* Flagged-node fill of a slab rank's sign mask (the classify step of
 * R/sign.py:179-195, which eik_run performs internally): eik_slab_finish
 * classifies every owned node by its own mu; this call then gives each owned
 * flagged node the class of its nearest unflagged node, with scipy EDT ties.
 * The nearest node may lie on a neighbour's planes, so the caller passes a
 * halo-extended copy of the mask, planes [e0, e1) (own planes
 * [own0, own0 + c0_local) plus neighbour planes), and every flagged node of
 * those planes (ext_nodes: sorted flat indices relative to plane e0).  Device
 * buffers; synchronous.  Returns EIK_EVALIDATION if a search needs a plane
 * outside [e0, e1) (widen the halo and call again). */
int eik_slab_fill(eik_plan* plan, const int64_t* ext_nodes, int64_t n_ext, int64_t e0, int64_t e1, int64_t own0,
                  int64_t c0_local, const uint8_t* mask_ext, uint8_t* mask_own, void* stream);

/* Extended-precision (double-double, ~106-bit) convolution (SURVEY.md §8(f)
 * rank 4): the big-float path of R/convolution.py:67-143 with p = 106, used by
 * the drop-in API for PrecisionConfig.bigfloat(tau, bits <= 106).  Fields:
 * EIK_FIELD_PHI | EIK_FIELD_S [| EIK_FIELD_GRAD | EIK_FIELD_HESS (2-D)];
 * axes up to 2048 nodes.  phi is returned as its (hi, lo) double pair; S,
 * gradient and Hessian as float64 (the reference converts big-float ratios to
 * float64, R/derivatives.py:165-170).  Host or device buffers (flags
 * EIK_HOST_INPUTS / EIK_HOST_OUTPUTS); synchronous; EIK_CHECK_UNDERFLOW
 * returns EIK_EUNDERFLOW when any phi <= 0. */
typedef struct eik_dd_plan eik_dd_plan;
typedef struct {
  double* phi_hi;
  double* phi_lo;
  double* S;
  double* grad[3];
  double* hess[3];
  uint8_t* underflow;
  int64_t* n_underflow; /* host */
} eik_dd_outputs;
int eik_dd_plan_create(int dim, const int64_t* counts, double spacing, double tau, uint32_t fields, int device,
                       eik_dd_plan** out);
int eik_dd_plan_destroy(eik_dd_plan* plan);
int eik_dd_run(eik_dd_plan* plan, const int64_t* nodes, int64_t n_nodes, const eik_dd_outputs* out, uint32_t flags,
               void* stream);

/* tau sweep (the kernel-reuse of R/experiments.py:74-109):
 * one plan caches exp(-|x|/tau_i) spectra for n_taus values; eik_run_sweep
 * transforms delta_Y once and writes S_i = -tau_i log phi_i for every tau
 * (NaN where phi_i <= 0; n_underflow counts those over all taus).  1-D, 2-D
 * and 3-D grids (3-D: the planes pass is shared, the axis-0 pass runs in
 * chunks of four tau values). */
int eik_plan_create_sweep(int dim, const int64_t* counts, double spacing, const double* taus, int n_taus,
                          int device, eik_plan** out);
int eik_run_sweep(eik_plan* plan, const int64_t* nodes, int64_t n_nodes, double* const* S, int64_t* n_underflow,
                  uint32_t flags, void* stream);

/* Interior mask from a winding / degree field (R/sign.py:166-198): flagged
 * nodes take mu from their nearest unflagged node with exactly the ties of
 * scipy.ndimage.distance_transform_edt(return_indices=True) (same separable
 * feature transform), then rint(mu) > 0 (mode 1, 2-D winding) / rint(mu) >= 1
 * (mode 2, 3-D degree), or mu >= threshold when use_threshold.  out_mask is
 * float64 0/1 as in the reference; with S given, out_signed = +S inside, -S
 * outside (R/sign.py:201-208).  EIK_HOST_INPUTS|EIK_HOST_OUTPUTS for host buffers. */
int eik_classify(int dim, const int64_t* counts, const double* mu, const int64_t* flagged_nodes, int64_t n_flagged,
                 int mode, int use_threshold, double threshold, double* out_mask, const double* S,
                 double* out_signed, uint32_t flags, int device, void* stream);

/* Engine-level spectral API (R/convolution.py:164-313), for callers of the
 * reference's FftConvolver building blocks.  Arrays of any shape (each axis
 * >= 1; mixed-radix Stockham transforms, Bluestein for prime factors > 31);
 * complex arrays are interleaved (re, im) float64, row-major.  Host or device
 * buffers (EIK_HOST_INPUTS / EIK_HOST_OUTPUTS); synchronous when host buffers
 * are used.  The reference's 2^31-element cap (_check_sizes) is lifted.
 *   eik_fftn         unnormalised forward DFT over every axis (fft_forward,
 *                    164-169), or the 1/P-normalised inverse (fft_inverse,
 *                    172-177); in_real: `in` is real float64.
 *   eik_fft_pair     forward_pair (264-286): the spectra of two real arrays
 *                    zero-padded to pshape, from one complex transform
 *                    (a or b may be NULL = zeros).
 *   eik_ifft_window  inverse_to_grid / inverse_pair_to_grid (288-307): inverse
 *                    of hat_a (+ i hat_b), window [start, start + counts) per
 *                    axis, real (and imaginary) parts.
 *   eik_cmul         product (309-313): elementwise complex multiply. */
int eik_fftn(int ndim, const int64_t* shape, const double* in, int in_real, double* out, int inverse, uint32_t flags,
             int device, void* stream);
int eik_fft_pair(int ndim, const int64_t* pshape, const double* a, const int64_t* ashape, const double* b,
                 const int64_t* bshape, double* a_hat, double* b_hat, uint32_t flags, int device, void* stream);
int eik_ifft_window(int ndim, const int64_t* pshape, const double* hat_a, const double* hat_b,
                    const int64_t* window_start, const int64_t* window_counts, double* out_re, double* out_im,
                    uint32_t flags, int device, void* stream);
int eik_cmul(int64_t n, const double* a, const double* b, double* out, uint32_t flags, int device, void* stream);

/* Device milliseconds of each pass of the last eik_run issued with
 * EIK_PROFILE (synchronizes on its events); -1 for passes that did not run. */
int eik_pass_times(eik_plan* plan, double* ms, int n);

const char* eik_last_error(void);
int eik_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EIKFLD_B200_H */
