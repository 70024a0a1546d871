/*
 * fsld_b200.h -- C ABI of the B200 (sm_100a) Fourier-slice project/adjoint path.
 *
 * Drop-in boundary for the hot path of the reference package `fsld`
 * (/root/reference/pkg/src/fsld).  The reference has no native ABI of its
 * own: its "native" layer is the numba kernel module kernels.py, called from
 * Python (Projector / DatasetOperator / optim).  Each entry point below names
 * the reference interface it replaces.  INTEGRATION.md shows the ctypes
 * binding a maintainer would add on the reference side.
 *
 * Conventions (all entry points):
 *  - every pointer argument is a DEVICE pointer unless documented otherwise;
 *  - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default
 *    stream) and is stream-ordered; nothing synchronises the host;
 *  - outputs are caller-allocated (mirrors the numba output-parameter style,
 *    kernels.py:138-302); accumulating outputs ("acc") are ADDED to, so the
 *    caller zeroes them (as Projector.backproject_batch does, forward.py:326-328);
 *  - return value: FSLD_OK (0) or a negative status; nothing throws across
 *    the ABI.  fsld_status_string() gives a message.
 *
 * Layouts (reference layout contract, grid.py:9-31):
 *  - volume: M^3 complex64 (interleaved re, im float32), linear index
 *    j = (z_index*M + y_index)*M + x_index, x/y centred (k + ceil(M/2)),
 *    z in FFT order (kz < 0 -> kz + M);
 *  - masked pixels: `pix` is (n_mask, 2) int16 (kx, ky) in ascending pixel
 *    index order (disk_mask, grid.py:185-189);
 *  - images: (rows, n_mask) complex64, compact masked (DatasetOperator.x,
 *    forward.py:527);
 *  - batch: `idx` (B,) int32 row numbers into the per-image records and the
 *    image rows (DatasetOperator.project(values, idx), forward.py:540-545);
 *    idx may be NULL, meaning batch entry b uses record (and image row) b.
 */
#ifndef FSLD_B200_H
#define FSLD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSLD_ABI_VERSION 2

/* status codes */
#define FSLD_OK 0
#define FSLD_EINVAL (-1)     /* invalid argument (reference: ValueError) */
#define FSLD_ECUDA (-2)      /* CUDA launch / runtime error */
#define FSLD_ENODEV (-3)     /* no sm_100 device */

/* interpolation modes (forward.py:35 MODES = ("nn", "tri")) */
#define FSLD_MODE_NN 0
#define FSLD_MODE_TRI 1

/* flags */
#define FSLD_DETERMINISTIC 1u /* accumulate in int64 fixed point: bitwise repeatable */
#define FSLD_TILE_PATH 2u     /* force the per-pixel tile kernel (global atomics) instead of bricks */
#define FSLD_NN_BRICK 8u      /* nn mode with dataset tables: the brick kernel instead of the per-pixel
                                 tile kernel (one global RED per pixel is cheaper for nn at every
                                 measured M, so the tile kernel is the default there) */
#define FSLD_REUSE_BINS 4u    /* reuse the brick work items the previous sorted call on the same scratch
                                 built for the same (recs, idx, B): skips the per-step binning */

/* fsld_image_rec.flags */
#define FSLD_REC_CTF 1u
#define FSLD_REC_SHIFT 2u

/*
 * Per-image parameter record, 128 bytes, read with one coalesced load per
 * image.  Replaces the reference's per-(image, pixel) tables rots/phases/
 * ctf_vals (forward.py:296-312, 524-527): phase and CTF are evaluated
 * in-kernel, so nothing of size (N, n_mask) but the images themselves lives
 * in HBM.
 *   rot   : R[0][0..2], R[1][0..2] (kernels.py:42-47 reads rows 0 and 1 only)
 *   shift : phase(kx,ky) = exp(i*pi*(shift[0]*kx + shift[1]*ky)), i.e.
 *           shift = -2 t / M (forward.py:299-303)
 *   gamma : CTF phase g = gamma[0]*(kx^2+ky^2) + gamma[1]*(kx^2-ky^2)
 *                        + gamma[2]*(2 kx ky) + gamma[3]*(kx^2+ky^2)^2
 *   env   : envelope exp(-env*(kx^2+ky^2))
 *   C(kx,ky) = -(wsin*sin g + wcos*cos g) * envelope     (if FSLD_REC_CTF)
 * The reference's radial toy CTF (forward.py:93-111) is the special case
 * gamma = {pi*defocus/r_max^2, 0, 0, 0}, env = b_factor/r_max^2,
 * wsin = 1-w, wcos = w; the physical astigmatic CTF of the BASELINE configs
 * fills all four gamma terms with wsin = sqrt(1-A^2), wcos = A.
 */
typedef struct fsld_image_rec {
    double rot[6];
    double shift[2];
    double gamma[4];
    double env;
    float wsin, wcos;
    uint32_t flags;
    float xmax;        /* >= max |x(p)| over this image's masked pixels (bounds the
                          fixed-point brick accumulator; set when images are uploaded) */
    uint32_t pad[2];
} fsld_image_rec;

int fsld_abi_version(void);
const char* fsld_status_string(int status);
/* number of visible devices with compute capability 10.x (host call) */
int fsld_device_count(int* count);
/* Page-locked host buffers for the host-buffer entry points (fsld_loss_grad_host): cudaHostAlloc
 * memory, which the copy engines stream at full PCIe rate in both directions at once. */
int fsld_host_alloc(size_t bytes, void** out);
int fsld_host_free(void* p);

/*
 * Scratch bytes needed by the reducing entry points for batches of up to B
 * images: prepared geometry (pixel lookup, mask rows), brick binning work
 * space and per-CTA partial sums (reduced in a fixed order).
 */
size_t fsld_scratch_bytes(int M, int n_mask, int B);

/*
 * Stamp `scratch` for a grid/mask (once per scratch buffer, like a plan
 * handle).  Kept for ABI stability; the current kernels need no precomputed
 * geometry in scratch.
 */
int fsld_prepare(int M, int n_mask, const int16_t* pix, void* scratch, size_t scratch_bytes, void* stream);

/*
 * Fused slice -> CTF/shift -> residual -> |r|^2 -> adjoint scatter.
 * Replaces optim._resid_pass(want_grad=True) (optim.py:147-162), i.e.
 * kernels.project_{tri,nn} (kernels.py:138-190) + residual numpy +
 * kernels.backproject_{tri,nn} (kernels.py:193-248) + fold_chunks.
 *   sq_out   : device double, receives sum over batch of |P v - x|^2
 *   grad_acc : += sum_i P_i^* conj(f_i) r_i   (unscaled; see fsld_grad_finalize)
 *              complex64 M^3, or int64 pairs M^3 when FSLD_DETERMINISTIC
 *   fx_scale : device double fixed-point scale (FSLD_DETERMINISTIC only,
 *              from fsld_fixed_scale), else NULL
 */
int fsld_loss_grad(int M, int mode, int n_mask, const int16_t* pix,
                   const fsld_image_rec* recs, const int32_t* idx, int B,
                   const void* v, const void* x, void* grad_acc, double* sq_out,
                   unsigned flags, const double* fx_scale,
                   void* scratch, size_t scratch_bytes, void* stream);

/* Loss only (Armijo trials): optim._resid_pass(want_grad=False) (optim.py:193-207). */
int fsld_loss(int M, int mode, int n_mask, const int16_t* pix,
              const fsld_image_rec* recs, const int32_t* idx, int B,
              const void* v, const void* x, double* sq_out,
              void* scratch, size_t scratch_bytes, void* stream);

/* Projection out[b, p] = f_b(p) * (P_b v)(p), (B, n_mask) complex64.
 * Replaces Projector.project_batch / DatasetOperator.project (forward.py:316-324, 540-545). */
int fsld_project(int M, int mode, int n_mask, const int16_t* pix,
                 const fsld_image_rec* recs, const int32_t* idx, int B,
                 const void* v, void* out, void* stream);

/* Adjoint acc += sum_b P_b^* conj(f_b) img[b]; img is (B, n_mask) complex64 (batch-local rows).
 * Replaces Projector.backproject_batch / DatasetOperator.backproject (forward.py:326-335, 547-552). */
int fsld_backproject(int M, int mode, int n_mask, const int16_t* pix,
                     const fsld_image_rec* recs, const int32_t* idx, int B,
                     const void* img, void* acc, unsigned flags, const double* fx_scale,
                     void* stream);

/* Normal operator acc += sum_b P_b^* C_b^2 P_b z (z complex64 M^3); the shift phase cancels.
 * Replaces the loop body of DatasetOperator.hvp (forward.py:554-570). */
int fsld_hvp(int M, int mode, int n_mask, const int16_t* pix,
             const fsld_image_rec* recs, const int32_t* idx, int B,
             const void* z, void* acc, unsigned flags, const double* fx_scale,
             void* stream);

/*
 * Hutchinson probe batcher: k Rademacher probes bit-packed as zbits
 * (M^3, words) uint32, words = ceil(k/32), bit p of word w = probe 32w+p
 * (1 -> +1, 0 -> -1, as optim.rademacher, optim.py:142-144).  Accumulates the
 * probe-folded sample  acc[j] += sum_p z_p[j] * (sum_b P_b^* C_b^2 P_b z_p)[j]
 * (float32 M^3, or int64 M^3 when FSLD_DETERMINISTIC) in one pass over the
 * batch; hutchinson_update (optim.py:210-229) then needs only
 * scale/k * acc + lam.
 */
int fsld_hutch_fold(int M, int mode, int n_mask, const int16_t* pix,
                    const fsld_image_rec* recs, const int32_t* idx, int B,
                    const uint32_t* zbits, int k, void* acc, unsigned flags,
                    const double* fx_scale, void* stream);

/* Pack k real probe vectors z ((k, n) float64, entries +-1, probe-major) into zbits
 * (n, ceil(k/32)) uint32; unused bits of the last word are zero.  Sets *bad (device
 * int, may be NULL) to 1 if an entry is not exactly +-1. */
int fsld_pack_probes(int64_t n, int k, const double* z, uint32_t* zbits, int* bad, void* stream);

/* Generate k counter-based Rademacher probes in place (no host RNG, no z bytes read):
 * bit = hash(seed, voxel, word).  For throughput runs; parity runs pack the
 * reference's numpy stream with fsld_pack_probes. */
int fsld_gen_probes(int64_t n, int k, uint64_t seed, uint32_t* zbits, void* stream);

/* Exact diagonal of sum_b P_b^* C_b^2 P_b: tri: acc[j] += C^2 w_j^2, nn: acc[j] += C^2
 * (kernels.scatter_sq_tri kernels.py:251-294; nn bincount forward.py:341-349, hessian.py:62-107). */
int fsld_exact_diag(int M, int mode, int n_mask, const int16_t* pix,
                    const fsld_image_rec* recs, const int32_t* idx, int B,
                    void* acc, unsigned flags, const double* fx_scale, void* stream);

/* fsld_exact_diag on the table-driven brick kernel (trilinear; the dataset's sorted layout and
 * tables, fsld_sorted_tables): acc[j] += sum_b,p C^2 w_pj^2 for the B images idx (no volume, no
 * images read).  acc is fp32, or with FSLD_DETERMINISTIC int64 at *fx_scale -- then bitwise the
 * same for any launch grid and batch order, and B <= 1024 per call.  scratch as fsld_scratch_bytes(B).
 * Replaces kernels.scatter_sq_tri (kernels.py:251-294) as called by hessian.exact_diag
 * (hessian.py:62-107). */
int fsld_exact_diag_sorted_tab(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                               const int8_t* pc, const void* ptab, const int32_t* seg_off, const int32_t* segs,
                               void* acc, unsigned flags, const double* fx_scale, void* scratch, size_t scratch_bytes,
                               void* stream);

/* Nearest-neighbour voxel index per (image, pixel), int32 (B, n_mask); bit-exact with
 * kernels.assign_nn (kernels.py:123-135). */
int fsld_assign_nn(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                   const int32_t* idx, int B, int32_t* out, void* stream);

/*
 * Table-driven variants with the numba kernel signatures (kernels.py:138-294):
 * the caller supplies the per-(image, pixel) factor table instead of the
 * in-kernel CTF/shift model.  Batch entry b uses record b (no idx).
 *   ftab : (B, n_mask) complex64, f = phase * ctf  (project: out = f * P v;
 *          adjoint: acc += P^* conj(f) img, the numba `img*conj(phase)*ctf`)
 *   wtab : (B, n_mask) complex64 whose real part is the per-pixel weight
 *          (scatter_sq_tri `weights`; nn mode: the bincount weights)
 */
int fsld_project_tab(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int B,
                     const void* v, const void* ftab, void* out, void* stream);
int fsld_backproject_tab(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int B,
                         const void* img, const void* ftab, void* acc, unsigned flags,
                         const double* fx_scale, void* stream);
int fsld_scatter_sq_tab(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int B,
                        const void* wtab, void* acc, unsigned flags, const double* fx_scale, void* stream);

/*
 * Brick-sorted dataset layout (M <= 256, n_mask <= 65535).  Poses are fixed
 * for a refinement run, so each image's masked pixels are stored once grouped
 * by the 8^3 volume brick that owns their trilinear footprint (floor corner
 * of R^T k, kernels.py:42-60, 147-170):
 *   xs     : (N, n_mask) complex64, images in sorted pixel order
 *   pc     : (N, n_mask, 2) int8, (kx, ky) of each sorted pixel
 *   seg_off: (N+1) int32 CSR offsets; segs: (S, 2) int32 = (brick, start | count << 16)
 * Build: fsld_sorted_count (writes seg_off; read seg_off[N] to size segs), then
 * fsld_sorted_fill (x_in in mask order -> xs; x_in may be NULL to build pc/segs only).
 */
int fsld_sorted_count(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int N,
                      int32_t* seg_off, void* stream);
int fsld_sorted_fill(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int N,
                     const void* x_in, void* x_out, int8_t* pc_out, const int32_t* seg_off,
                     int32_t* segs, void* stream);

/*
 * Per-pixel invariants of a brick-sorted dataset (poses, shifts and CTFs are fixed for a
 * refinement run; the reference likewise keeps per-(image, pixel) phase and CTF tables,
 * forward.py:524-527).  ptab: fsld_sorted_tables_bytes(N, n_mask) bytes (24 per pixel + a
 * header), 256-byte aligned, opaque; per pixel in the sorted order:
 *   f = C * phase (fp32 complex, evaluated in fp64; forward.py:93-111, 299-312), and the
 *   trilinear footprint of the clamped rotated pixel (fp64, kernels.py:42-60, 147-170) in
 *   the frame of its brick: weights (wx, wy, wz) as fp32 and the corner index in the 9^3 brick.
 * Passing ptab to the brick entry points below selects the table-driven brick kernel
 * (24 bytes loaded per pixel instead of evaluating geometry, CTF and phase per pixel);
 * ptab = NULL runs the compute path from pc and the records.  mode FSLD_MODE_NN stores the
 * reference's nearest-neighbour voxel (bit-exact, kernels.py:69-120) instead of the trilinear
 * footprint: fsld_loss_grad_sorted with FSLD_NN_BRICK / fsld_hvp_sorted then run the brick kernel
 * in nn mode (one gather, one complex shared-memory add per pixel).  Rebuild after changing poses
 * or CTFs (the images themselves are not part of the table).
 */
size_t fsld_sorted_tables_bytes(int N, int n_mask);
int fsld_sorted_tables(int M, int mode, int n_mask, const fsld_image_rec* recs, int N, const int8_t* pc,
                       const int32_t* seg_off, const int32_t* segs, void* ptab, void* stream);

/* Fused loss + gradient over a brick-sorted dataset (optim.py:147-190 hot loop):
 * tri mode runs the brick kernel (smem-staged bricks, one global reduction per
 * touched voxel per work item); nn / deterministic / FSLD_TILE_PATH fall back to
 * the per-pixel tile kernel reading coordinates from pc. */
int fsld_loss_grad_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx,
                          int B, const void* v, const void* xs, const int8_t* pc, const void* ptab,
                          const int32_t* seg_off, const int32_t* segs, void* grad_acc, double* sq_out,
                          unsigned flags, const double* fx_scale, void* scratch, size_t scratch_bytes,
                          void* stream);
/* fsld_loss_grad_sorted fused with the k = 1 Hutchinson probe of the same batch (tri, brick path):
 *   grad_acc += sum_b P_b^* conj(f_b) r_b,  *sq_out = sum |r|^2          (optim.py:147-162)
 *   fold[j]  += z_j (sum_b P_b^* C_b^2 P_b z)_j                           (optim.py:210-229 numerator)
 * z = +-1 from bit 0 of zbits[j] (M^3 words, fsld_pack_probes / fsld_gen_probes with k = 1).
 * One pass over the batch: the probe rides along with the gradient (one more gather from
 * shared memory and 8 more shared-memory adds per pixel).  FSLD_DETERMINISTIC / FSLD_TILE_PATH
 * are rejected (use fsld_loss_grad_sorted + fsld_hutch_fold). */
int fsld_loss_grad_hutch_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                                const void* v, const void* xs, const int8_t* pc, const void* ptab,
                                const int32_t* seg_off,
                                const int32_t* segs, const uint32_t* zbits, void* grad_acc, float* fold,
                                double* sq_out, unsigned flags, void* scratch, size_t scratch_bytes, void* stream);

/* Hessian data term on the brick-sorted layout (tri, fp32 accumulation; replaces fsld_hvp,
 * forward.py:554-570 / hessian.py:110-118, for datasets laid out by fsld_sorted_fill):
 *   acc += sum_b P_b^* C_b^2 P_b z,   *sq_out = sum_b ||C_b P_b z||^2 = ||A z||^2
 * The brick loss+grad pass with zero images: r = f P z, conj(f) r = |f|^2 P z.  The caller applies
 * the n_total/|B| scale and lam (forward.py:567-570).  Deterministic / tile-path flags are rejected
 * (use fsld_hvp). */
int fsld_hvp_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                    const void* z, const int8_t* pc, const void* ptab, const int32_t* seg_off, const int32_t* segs, void* acc,
                    double* sq_out, unsigned flags, void* scratch, size_t scratch_bytes, void* stream);

/* Loss only over a brick-sorted dataset (Armijo trials, optim.py:193-207). */
int fsld_loss_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                     const void* v, const void* xs, const int8_t* pc, double* sq_out, void* scratch,
                     size_t scratch_bytes, void* stream);
/* fsld_loss_sorted over a table-built dataset (ptab from fsld_sorted_tables; seg_off / segs the
 * dataset's segment list): the brick binning and the table-driven kernel's projection pass alone
 * (optim.py:193-207 data term); ptab = NULL or nn mode fall back to fsld_loss_sorted. */
int fsld_loss_sorted_tab(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                         const void* v, const void* xs, const int8_t* pc, const void* ptab, const int32_t* seg_off,
                         const int32_t* segs, double* sq_out, void* scratch, size_t scratch_bytes, void* stream);
/* Projection of dataset rows idx into their sorted pixel order: out (B, n_mask). */
int fsld_project_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                        const void* v, const int8_t* pc, void* out, void* stream);
/* acc += sum_b P^* conj(f) xs[idx[b]] (b_vector, forward.py:572-579). */
int fsld_backproject_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx,
                            int B, const void* xs, const int8_t* pc, void* acc, unsigned flags,
                            const double* fx_scale, void* stream);

/*
 * Fixed-point scale for FSLD_DETERMINISTIC accumulation: writes
 * 2^floor(61 - log2(bound)) to *fx_scale, bound = mult * (max_i |data_i| + add),
 * data complex64 of n elements (data may be NULL -> max = 0).
 */
int fsld_fixed_scale(const void* data, int64_t n, double mult, double add, double* fx_scale,
                     void* stream);

/*
 * Finalize an accumulator into complex64:
 *   out = scale * acc_value + lam * v      (v may be NULL -> 0)
 * acc_value = acc (complex64) or int64 pairs / fx_scale when FSLD_DETERMINISTIC.
 * The loss_and_grad epilogue (optim.py:186-189) and hvp's (forward.py:570).
 */
int fsld_grad_finalize(int64_t nvox, const void* acc, unsigned flags, const double* fx_scale,
                       const void* v, double scale, double lam, void* out, void* stream);

/* Real-accumulator variant (Hutchinson fold / exact diag): out = scale*acc + add, float32. */
int fsld_real_finalize(int64_t nvox, const void* acc, unsigned flags, const double* fx_scale,
                       double scale, double add, float* out, void* stream);

/*
 * Fused loss_and_grad epilogue (optim.py:186-189), one pass over the volume:
 *   grad = scale * acc + lam * v  (complex64);  acc is zeroed for the next step;
 *   *loss = 0.5 * scale * (*sq) + 0.5 * lam * ||v||^2  (device doubles; loss / norm2 may be NULL).
 * scratch: >= 1184 doubles of per-block partials (fixed reduction order).
 */
int fsld_grad_epilogue(int64_t nvox, void* acc, const void* v, double scale, double lam, void* grad,
                       const double* sq, double* loss, double* norm2, void* scratch, size_t scratch_bytes,
                       void* stream);

/* sum |v|^2 over complex64 M^3 in a fixed order (fp64), for the lam/2 ||v||^2 term. */
int fsld_norm2(int64_t n, const void* v, double* out, void* scratch, size_t scratch_bytes,
               void* stream);

/*
 * ---- Algorithm-1 step on the device -------------------
 *
 * One preconditioned SGD step of optim.run (optim.py:362-382) without host
 * round trips:  loss_grad pass (acc, sq) [+ hutch_fold pass (fold)] ->
 * fsld_precond_step (grad, Hutchinson average, EMA, threshold, direction and
 * the line-search volume terms, one pass) -> fsld_armijo_terms (one projection
 * of the direction) -> fsld_armijo_select (closed-form backtracking) ->
 * fsld_apply_step.  The loss is quadratic in v, so
 *   batch_loss(v - eta d) - f0 = 1/2 s (eta^2 |q|^2 - 2 eta Re<r, q>)
 *                              + 1/2 lam (eta^2 ||d||^2 - 2 eta Re<v, d>)
 * with r = f P v - x and q = f P d over the batch: (1 + backtracks) loss
 * passes (optim.py:269-306) become one projection.
 */
typedef struct fsld_step_params {
    double scale;        /* N / |batch| (optim.py:183) */
    double lam;
    double beta;         /* EMA weight (optim.py:244) */
    double floor;        /* alpha, or 1e-12 for the unthresholded variant (optim.py:246) */
    double w_old, w_new; /* d_avg <- w_old d_avg + w_new sample: k_old/k, k_new/k (optim.py:226-229) */
    double hutch_scale;  /* sample = hutch_scale * fold + lam, hutch_scale = scale / k_new */
    int estimating;      /* 1: Hutchinson/EMA/threshold from fold; 0: dhat = dhat_fixed (or 1) */
    int pad;
} fsld_step_params;

typedef struct fsld_armijo_state {
    double eta;          /* carried step size, in/out (optim.py:362, 372-376) */
    double f0;           /* 1/2 s sq + 1/2 lam ||v||^2 of the step */
    double f_next;       /* accepted loss */
    double eta_applied;  /* step applied by fsld_apply_step (0 when decrease == 0) */
    double decrease;     /* ||grad||^2 in the dhat^-1 norm */
    int backtracks;
    int status;          /* 0 ok; 1 = more than max_halvings halvings (NumericalError) */
    int n_steps;         /* steps selected so far (hist row index) */
    int pad;
} fsld_armijo_state;

/* One pass over the volume (complex64 acc / v / dir, float32 state):
 *   grad = scale*acc + lam*v;  acc <- 0
 *   estimating: sample = hutch_scale*fold + lam; fold <- 0;
 *               d_avg <- w_old*d_avg + w_new*sample; d <- beta*d + (1-beta)*d_avg;
 *               dhat = max(|d|, floor)            (optim.py:210-247)
 *   else        dhat = dhat_fixed[i] (or 1 when NULL: the plain variant)
 *   dir = grad / dhat                             (optim.py:292)
 *   out5 = {sum |grad|^2/dhat, ||v||^2, Re<v, dir>, ||dir||^2, Re<acc, dir>}  (fp64, fixed order);
 *   the last is Re<r, A dir> of the line search (acc = A^* r), so only ||A dir||^2 needs a pass.
 * grad_out / dhat_out may be NULL.  All vectors 16-byte aligned.  scratch >= 5 * 2368 doubles. */
int fsld_precond_step(int64_t nvox, void* acc, const void* v, float* fold, float* d_avg, float* d,
                      const float* dhat_fixed, const fsld_step_params* params, void* dir, void* grad_out,
                      float* dhat_out, double* out5, void* scratch, size_t scratch_bytes, void* stream);

/* Line-search terms of the direction d over the batch (r = f P v - x, q = f P d), tile kernel:
 *   out3 = {sum |r|^2, sum Re(conj(r) q), sum |q|^2}  (fp64, fixed order).
 * Coordinates from pc (brick-sorted dataset: xs and pc in the sorted layout) or, when pc
 * is NULL, from the mask table pix. */
int fsld_armijo_terms(int M, int mode, int n_mask, const int16_t* pix, const int8_t* pc,
                      const fsld_image_rec* recs, const int32_t* idx, int B, const void* v, const void* d,
                      const void* xs, double* out3, void* scratch, size_t scratch_bytes, void* stream);

/* Hutchinson probe batcher on the brick-sorted layout (tri, k <= 256): same result as
 * fsld_hutch_fold (float32 fold += sum_p z_p * (sum_b P_b^* C_b^2 P_b z_p)), per brick work item
 * with the probe words staged in shared memory and a shared fixed-point accumulator. */
int fsld_hutch_fold_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                           const int8_t* pc, const int32_t* seg_off, const int32_t* segs, const uint32_t* zbits,
                           int k, float* fold, void* scratch, size_t scratch_bytes, void* stream);

/* ||A d||^2 = sum_b sum_p C^2 |P d|^2 over the batch on the brick-sorted layout (tri mode):
 * a gather-only pass (no images) for the closed-form line search.  *out = device double.
 * flags: 0 or FSLD_REUSE_BINS: reuse the work items the last sorted call on this scratch binned
 * (the loss+grad call of the same step).  EINVAL if that call was for another recs / idx pointer /
 * B; the rows themselves are compared on the device with the copy the binning stored, and if the
 * caller rewrote idx in place since, the batch is binned again (never stale work items). */
int fsld_proj_energy_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                            const void* d, const int8_t* pc, const int32_t* seg_off, const int32_t* segs,
                            double* out, unsigned flags, void* scratch, size_t scratch_bytes, void* stream);

/* Closed-form Armijo backtracking (optim.py:269-306) on the device, one thread:
 * sq = the step's loss-pass sum |r|^2 (f0), rq = Re<r, A d>, qq = ||A d||^2, vol = the first four
 * outputs of fsld_precond_step.  Halves st->eta until delta(eta) <= -c eta decrease (at most
 * max_halvings times); records (f0, eta, f_next, backtracks, decrease) into
 * hist[5 * st->n_steps ...] when st->n_steps < hist_cap. */
int fsld_armijo_select(const double* sq, const double* rq, const double* qq, const double* vol, double scale,
                       double lam, double c, int max_halvings, fsld_armijo_state* st, double* hist, int hist_cap,
                       void* stream);

/* v <- v - st->eta_applied * dir  (complex64). */
int fsld_apply_step(int64_t nvox, void* v, const void* dir, const fsld_armijo_state* st, void* stream);

/*
 * Multi-batch binning plans.  The batches of an epoch are known in advance (optim.py:133-139),
 * so the per-step brick binning (count -> scan -> fill of the batch's segment records) can be done
 * for K batches of B images at once; each step then only runs the work-item kernel.
 *   idx         : (K, B) int32 dataset rows, batch k = idx[k*B .. k*B+B)
 *   total_pairs : sum over the K batches of the images' segment counts
 *                 (sum_k sum_b seg_off[row+1] - seg_off[row]); sizes the plan
 * A plan is read-only after fsld_plan_build; batch k can be run any number of times.
 * fsld_loss_grad_planned = fsld_loss_grad_sorted (zbits == NULL) or fsld_loss_grad_hutch_sorted
 * (zbits != NULL) for batch k; fsld_proj_energy_planned = fsld_proj_energy_sorted for batch k.
 * scratch: fsld_scratch_bytes(M, n_mask, B) (per-CTA partial sums).
 */
size_t fsld_plan_bytes(int M, int n_mask, int B, int K, int64_t total_pairs);
int fsld_plan_build(int M, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int K, int B,
                    const int32_t* seg_off, const int32_t* segs, int64_t total_pairs, void* plan, size_t plan_bytes,
                    void* stream);
int fsld_loss_grad_planned(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan, int B, int k,
                           const void* v, const void* xs, const int8_t* pc, const void* ptab, const uint32_t* zbits,
                           void* grad_acc,
                           float* fold, double* sq_out, void* scratch, size_t scratch_bytes, void* stream);
/* The complete loss+grad step of batch k of a plan, epilogue fused around the brick pass
 * (optim.py:165-190 with loss_and_grad's scale / lam applied on the device):
 *   grad  = scale * sum_b P_b^* conj(f_b) r_b + lam v        (overwritten; v != grad)
 *   *sq_out = sum |r|^2,   *loss = 0.5 scale sq + 0.5 lam ||v||^2
 * grad is set to lam v first and the brick pass adds its scaled contributions into it, so no
 * separate accumulator is read back or cleared.  scratch: fsld_scratch_bytes(M, n_mask, B);
 * norm_scratch: >= 148 * 8 doubles. */
int fsld_loss_grad_step_planned(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan, int B,
                                int k, const void* v, const void* xs, const int8_t* pc, const void* ptab, double scale,
                                double lam,
                                void* grad, double* sq_out, double* loss, void* scratch, size_t scratch_bytes,
                                void* norm_scratch, size_t norm_scratch_bytes, void* stream);
/* Host-buffer loss + gradient: the call a host caller makes with numpy-style buffers
 * (optim.loss_and_grad, optim.py:165-190, whose v / grad are host arrays), tri mode, brick path.
 * HOST pointers (page-locked, cudaHostAlloc / cudaHostRegister):
 *   idx_host  : (B,) int32 dataset rows          v_host : M^3 complex64
 *   grad_host : M^3 complex64, overwritten with  scale * sum_b P_b^* conj(f_b) r_b + lam v
 *   out_host  : 2 doubles, {sum |r|^2, loss = 0.5 scale sq + 0.5 lam ||v||^2}
 * DEVICE staging: v_dev, grad_dev (M^3 complex64 each, distinct), idx_dev (B int32);
 * scratch: fsld_scratch_bytes(M, n_mask, B), prepared.
 * The volume moves in n_slabs (1..16) z-slabs of brick layers: slab g's host->device copy, its
 * lam v initialisation, its brick pass and its device->host copy of the finished gradient are
 * pipelined on two internal copy streams (forked from / joined back into `stream`), so the
 * PCIe transfers in both directions overlap each other and the kernels.  Everything is enqueued
 * on `stream`: the outputs are valid once `stream` has been synchronised.
 * Host-side blocking: the step of a given call shape is one cached CUDA graph whose batch rows come
 * from a pinned staging buffer it owns, so a call first waits (host) until the previous replay of
 * the same shape has read its rows; calls from several host threads are serialised.
 * Buffer lifetime: a cached graph's copies hold v_host / grad_host / out_host as captured.
 * fsld_host_free drops the graphs that use the buffer it frees; before freeing host buffers that
 * came from another allocator, call fsld_host_step_reset() (drops every cached graph). */
int fsld_host_step_reset(void);
int fsld_loss_grad_host(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host, int B,
                        const void* v_host, const void* xs, const int8_t* pc, const void* ptab,
                        const int32_t* seg_off, const int32_t* segs, double scale, double lam, void* grad_host, double* out_host,
                        void* v_dev, void* grad_dev, int32_t* idx_dev, int n_slabs, void* scratch,
                        size_t scratch_bytes, void* stream);
/* fsld_loss_grad_host with the gradient delivered as complex128 (the reference's dtype, optim.py:190):
 * grad_host_c128 is a page-locked M^3 complex128 host buffer; each finished slab is cast on the device
 * into grad_dev128 (device staging, M^3 complex128) and copied out from there, so the host never casts
 * the gradient.  v_host stays complex64. */
int fsld_loss_grad_host_c128(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host, int B,
                             const void* v_host, const void* xs, const int8_t* pc, const void* ptab,
                             const int32_t* seg_off, const int32_t* segs, double scale, double lam,
                             void* grad_host_c128, double* out_host, void* v_dev, void* grad_dev, void* grad_dev128,
                             int32_t* idx_dev, int n_slabs, void* scratch, size_t scratch_bytes, void* stream);
/* The reference's call shape end to end: optim.loss_and_grad(op, v, batch, lam) with a numpy complex128
 * volume in and a complex128 gradient out (optim.py:165-190).  v128_host / grad128_host: M^3 complex128
 * host arrays (any host memory, 16-byte aligned).  The library casts v to complex64 on its host thread
 * pool (streaming stores) into its own page-locked staging and runs the slab-pipelined host step; a
 * page-locked grad128_host is written by the copy engine (each finished slab cast to complex128 on the
 * device), any other memory receives the complex64 gradient cast back by the host threads.  Blocking:
 * returns once grad128_host and out_host = [sum|r|^2, loss] are written. */
int fsld_loss_grad_host_np(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host, int B,
                           const double* v128_host, const void* xs, const int8_t* pc, const void* ptab,
                           const int32_t* seg_off, const int32_t* segs, double scale, double lam, double* grad128_host,
                           double* out_host, void* v_dev, void* grad_dev, int32_t* idx_dev, int n_slabs,
                           void* scratch, size_t scratch_bytes, void* stream);
/* The same call moving only the touched ball (grid.touched_ball): the data term
 * only reaches voxels within touch_radius = max |k| over the mask + sqrt(3) of the origin.  With
 * touch_radius > 0 only those voxels cross PCIe, packed row by row as complex64 -- one contiguous range per
 * z-slab in each direction (fsld_ball_voxels(M, touch_radius) voxels: ~58 % of the cube at M=128) -- and
 * the host threads cast each finished gradient slab to complex128 into grad128_host (any host memory)
 * while later slabs are in flight; off the ball they write grad = lam v in fp64 while the device works,
 * and ||v||^2 in the loss is summed on the host in fp64.  touch_radius <= 0: fsld_loss_grad_host_np. */
int fsld_loss_grad_host_np_ball(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host,
                                int B, const double* v128_host, const void* xs, const int8_t* pc, const void* ptab,
                                const int32_t* seg_off, const int32_t* segs, double scale, double lam,
                                double* grad128_host, double* out_host, void* v_dev, void* grad_dev, int32_t* idx_dev,
                                int n_slabs, void* scratch, size_t scratch_bytes, void* stream, double touch_radius);
/* Voxels of the packed ball of fsld_loss_grad_host_np_ball (M^3 when touch_radius <= 0). */
int64_t fsld_ball_voxels(int M, double touch_radius);
int fsld_proj_energy_planned(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan, int B, int k,
                             const void* d, const int8_t* pc, double* out, void* scratch, size_t scratch_bytes,
                             void* stream);

/*
 * Per-epoch metric and ingest on the device.
 * fsld_fsc: Fourier shell correlation of complex64 volumes u, v (metrics.py:38-63):
 *   out[r] = sum_{shell r} Re(u conj(v)),  out[R+1+r] = sum |u|^2,  out[2(R+1)+r] = sum |v|^2
 *   for r = 0..max_radius (rounded |k|), fp64; the caller forms num / sqrt(pu pv).
 *   scratch: fsld_fsc_scratch_bytes(M, max_radius) (per-CTA partial rows, added in a fixed order).
 * fsld_mask_images: x[i, p] = (complex64) images[i, mask[p]] for N full M^2 complex128 images
 *   (the FSD1 payload, io.py:91-125) -> the compact masked rows of the dataset (forward.py:527).
 */
size_t fsld_fsc_scratch_bytes(int M, int max_radius);
/* out[i] = mean over the n_ring pixels (kx, ky) of ring of C_i(k)^2 (fp64; 1 without a CTF): the
 * per-image term of threshold_alpha for a non-radial CTF (optim.py:250-266). */
int fsld_ctf_ring_power(const fsld_image_rec* recs, int N, const int16_t* ring, int n_ring, double* out, void* stream);
int fsld_fsc(int M, int max_radius, const void* u, const void* v, double* out, void* scratch, size_t scratch_bytes,
             void* stream);
int fsld_mask_images(int M, int n_mask, const int32_t* mask, int N, const void* images, void* x, void* stream);

/*
 * Host-side casts for the numpy (reference-signature) calls: dst = (float) src / (double) src over
 * n reals (2 per complex) with non-temporal stores, so a page-locked staging buffer is not left
 * dirty in the CPU caches before the copy engine reads it.  Host pointers; synchronous; thread-safe
 * (callers split large ranges over their own threads).
 */
int fsld_host_cast_f64_to_f32(const double* src, float* dst, int64_t n);
int fsld_host_cast_f32_to_f64(const float* src, double* dst, int64_t n);

/*
 * Touched-ball compaction for the data-parallel all-reduce: a scatter can only reach
 * voxels within radius R + 1/2 + sqrt(3) of the origin (mask radius R; Appendix A item 7), ~54 %
 * of the cube at M=128, so ranks all-reduce the compacted vector.  idx: (n,) int32 voxel indices
 * (ascending); elements of elem_bytes = 8 (complex64) or 4 (float32).
 *   gather : dst[i] = src[idx[i]]        scatter: dst[idx[i]] = src[i]   (other dst entries untouched)
 */
int fsld_ball_gather(int64_t n, const int32_t* idx, const void* src, void* dst, int elem_bytes, void* stream);
int fsld_ball_scatter(int64_t n, const int32_t* idx, const void* src, void* dst, int elem_bytes, void* stream);

/*
 * Data-parallel gradient exchange through NVSwitch multicast (NVLS), fused into the brick pass.
 * The loss is a sum over images (optim.py:186-189; the per-rank partial sums of a sharded dataset
 * add), so every rank maps one multicast object over its own copy of the gradient accumulator and
 * the brick kernel's per-item flush reduces into the multicast address (multimem.red): NVSwitch
 * applies each flush to every copy while the pass runs, and after fsld_nvls_barrier each rank's copy
 * holds the sum over all ranks -- no all-reduce after the pass.  Replaces the NCCL all-reduce of
 * the touched-ball vector (fsld_ball_gather / fsld_ball_scatter) on NVSwitch systems.
 *   rank 0       : fsld_nvls_create -> size, fd (a POSIX fd for n_ranks > 1, else -1)
 *   rank r > 0   : receive the fd (fsld_fd_listen before rank 0 sends, fsld_fd_send, fsld_fd_recv),
 *                  fsld_nvls_import(fd, n_ranks, r, data_bytes, size)
 *   every rank   : fsld_nvls_add_device (current device) ; [all ranks] ; fsld_nvls_bind -> uc, mc
 *   per step     : fsld_nvls_barrier(NULL, NULL)  -- every copy zeroed by its rank's epilogue
 *                  fsld_loss_grad_planned_mc(..., mc, ...)  -- the pass, flushing into the multicast
 *                  fsld_nvls_barrier(sq, sq_total)  -- all flushes landed; |r|^2 summed in rank order
 *                  fsld_grad_epilogue on uc (grad = scale uc + lam v, uc <- 0)
 * data_bytes: the accumulator (M^3 complex64); the bound range also holds the barrier word and the
 * per-rank |r|^2 slots at fsld_nvls_ctl_offset(data_bytes).  A barrier that waits > 20 s for a peer
 * gives up and fsld_nvls_status returns FSLD_ECUDA.  fsld_nvls_supported: the driver reports
 * multicast support for the device AND creates a one-device multicast object (0 without a driver,
 * on systems without NVSwitch multicast, or where the fabric's multicast service is not reachable).
 */
typedef struct fsld_nvls fsld_nvls;
int fsld_nvls_supported(int device);
size_t fsld_nvls_ctl_offset(size_t data_bytes);
int fsld_nvls_create(int n_ranks, size_t data_bytes, size_t* size_out, int* fd_out, fsld_nvls** out);
int fsld_nvls_import(int fd, int n_ranks, int rank, size_t data_bytes, size_t size, fsld_nvls** out);
int fsld_nvls_add_device(fsld_nvls* g);
int fsld_nvls_bind(fsld_nvls* g, void** uc_ptr, void** mc_ptr);
int fsld_nvls_barrier(fsld_nvls* g, const double* sq_in, double* sq_out, void* stream);
int fsld_nvls_status(fsld_nvls* g);
int fsld_nvls_destroy(fsld_nvls* g);
/* fd passing between processes of one node: SCM_RIGHTS over an abstract unix socket `name`.
 * fsld_fd_listen binds (before the sender connects); fsld_fd_recv accepts one fd and closes the
 * socket; fsld_fd_send connects (retrying for ~10 s) and sends. */
int fsld_fd_listen(const char* name, int* sock_out);
int fsld_fd_recv(int sock, int* fd_out);
int fsld_fd_send(const char* name, int fd);
/* fsld_loss_grad_planned (trilinear, tables, no probe) with grad_acc a MULTICAST address from
 * fsld_nvls_bind: the flush reduces into every rank's copy.  sq_out: this rank's |r|^2. */
int fsld_loss_grad_planned_mc(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan, int B, int k,
                              const void* v, const void* xs, const int8_t* pc, const void* ptab, void* grad_acc_mc,
                              double* sq_out, void* scratch, size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FSLD_B200_H */
