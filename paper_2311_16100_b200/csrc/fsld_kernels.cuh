// fsld_kernels.cuh -- launch interface between the C ABI (fsld_capi.cu) and the kernels.
#pragma once

#include "fsld_common.cuh"

namespace fsld {

enum Op { OP_PROJECT = 0, OP_LOSS, OP_LOSS_GRAD, OP_BACKPROJECT, OP_HVP, OP_DIAG, OP_ARMIJO };

struct SliceArgs {
    int M, c2, n_mask;
    int tiles;  // CTAs per image
    int ppt;    // pixels per thread
    double bnd;
    const short2* pix;
    const fsld_image_rec* recs;
    const int32_t* idx;
    const float2* v;       // volume / probe (complex64)
    const float2* x;       // image rows (complex64)
    int x_by_idx;          // x row = idx[b] (dataset) or b (batch-local)
    float2* out;           // projection output (B, n_mask)
    void* acc;             // scatter accumulator
    double* partials;      // per-CTA loss partials
    const double* fx;      // fixed-point scale (deterministic)
    const float2* ftab;    // optional (B, n_mask) factor table f = phase*ctf (numba-style calls)
    const char2* pc;       // optional per-(row, p) pixel coordinates (brick-sorted dataset layout)
    const float2* v2;      // OP_ARMIJO: the search direction d
    int nparts;            // OP_ARMIJO: column stride of the 3 partial columns
};

// ---------------------------------------------------------------------------
// Brick-sorted path (fsld_brick.cu).  Poses are fixed for the whole run, so
// each image's masked pixels are stored once in HBM grouped by the 8^3 volume
// brick that owns their trilinear footprint (floor corner), with per-pixel
// (kx, ky) as int8 pairs and a per-image segment list (brick, start, count).
// Per step the batch's segments are binned by brick (count -> scan -> fill)
// into work items (brick, <= BC segments); one CTA per item gathers from /
// scatters into a shared-memory copy of the brick (+1 halo), so the adjoint
// costs one global reduction per touched brick voxel per item instead of 8
// per pixel.
// ---------------------------------------------------------------------------
constexpr int BT = 8;                 // brick edge (voxels)
constexpr int BH = BT + 1;            // + halo for the floor+1 corners
constexpr int BH3 = BH * BH * BH;     // 729
#ifndef FSLD_BC
#define FSLD_BC 64
#endif
constexpr int BC = FSLD_BC;           // segments (images) per work item (tools/build_exp.sh -DFSLD_BC=..)
constexpr int BW = 8;                 // warps per CTA
constexpr int kSegMax = 128;          // pixels per (image, brick) segment (larger runs are split)
constexpr int BTHREADS = BW * 32;
constexpr uint32_t kGeomMagic = 0xF51DB200u;

struct GeomHeader {   // at the start of the scratch buffer (256-byte slot)
    uint32_t magic;
    int M, n_mask, pad0;
    const void* pix;
    int pad1[10];
};

// Per binned (image, brick) segment, written by the per-step fill pass from the
// image's fsld_image_rec: everything the main kernel needs per pixel, in six
// 16-byte words.  The CTF defocus phase and the shift phase are carried as
// 64-bit fixed-point "turns" coefficients (frac(coef / 2pi) * 2^64), so the
// kernel evaluates gamma mod 2pi exactly with wrapping 32-bit integer
// multiplies on small non-negative integer monomials of (kx, ky) instead of
// fp64 arithmetic (see seg_factor in fsld_brick_main.cuh).
struct __align__(16) SegRec {
    long long gofs;       // row * n_mask + start (element offset of the segment in xs / pc)
    int count, row;
    float frame[6];       // fp32 rotation rows 0, 1 (floor_corner)
    float wsin, wcos;     // CTF = -(wsin sin(gamma) + wcos cos(gamma)) * 2^(-envl k^2)
    float envl;
    uint32_t gc;          // gamma constant term, turns * 2^32
    uint32_t sc;          // shift constant term, turns * 2^32
    uint32_t start;
    uint32_t glo[4], ghi[4];  // gamma: k2, c2 + 2^15, s2 + 2^16, k2^2
    uint32_t slo[2], shi[2];  // shift: kx + 128, ky + 128
    uint32_t pad[4];
};
static_assert(sizeof(SegRec) == 128, "SegRec is 8 x 16 B");

// Shared-memory slot of a SegRec in the brick kernels: 8 + FSLD_SEG_PAD 16-byte words.  With a
// 128-byte stride every segment's copy of a field sits in the same bank, so a warp whose pixels
// span several segments replays each record load once per segment; the pad staggers them.
#ifndef FSLD_SEG_PAD
#define FSLD_SEG_PAD 1
#endif
constexpr int SEG_W = 8 + FSLD_SEG_PAD;

// Per binned segment in global memory (16 B): the brick kernels assemble a SegRec in shared
// memory from it and the per-image template (the SegRec fields that depend only on the image).
struct __align__(16) PairRec {
    long long gofs;  // row * n_mask + start
    int count;
    int tslot;       // index of the image's SegRec template in SortedArgs::tmpl
};
static_assert(sizeof(PairRec) == 16, "PairRec is one 16-byte word");

// Slab-pipelined host step (fsld_loss_grad_host): at most kMaxSlabs z-slabs of brick layers, each
// with its own work-item list, control block and partial sums.
constexpr int kMaxSlabs = 16;
constexpr int kSlabCtas = 148 * 8;     // >= the persistent brick grid (CTAs per SM x SMs)
constexpr int kInitParts = 148 * 2;    // grad_init partial sums per contiguous volume piece

struct ScratchLayout {
    size_t hdr, cnt, off, fill, pairs, tmpl, items, ctl, part, gitems, gctl, gpart, npart, hout, bidx, gate, total;
    int nb, nbr, cap_pairs, cap_items, cap_part;
};

ScratchLayout scratch_layout(int M, int n_mask, int B);

// Multi-batch binning plan (fsld_plan_*): K batches of B images binned at once.
struct PlanLayout {
    size_t hdr, cnt, off, fill, ctl, seg_tot, items, pairs, tmpl, total;
    int nbr, K, B;
    long long total_pairs, cap_items;
};
PlanLayout plan_layout(int M, int B, int K, long long total_pairs);

struct SortedArgs {
    int M, c, nb, nbr, n_mask, B;
    float bnd;
    const fsld_image_rec* recs;
    const int32_t* idx;
    const float2* v;
    const float2* xs;        // (N, n_mask) brick-sorted images
    const char2* pc;         // (N, n_mask) (kx, ky) of each sorted pixel
    const void* ptab;        // optional (N, n_mask) PixTab (f, footprint): the table-driven brick kernel
    int nn;                  // nearest-neighbour slicing (table-driven kernel only; 0 = trilinear)
    const int32_t* seg_off;  // (N+1) CSR offsets into segs
    const int2* segs;        // (brick, start | count << 16)
    float2* acc;
    const uint32_t* zbits;   // optional k = 1 Rademacher probe (bit 0 of word j, M^3 words): fused Hutchinson
    float* fold;             // fold[j] += z_j (sum_b P^* C^2 P z)_j
    int* cnt;
    int* off;
    int* fill;
    PairRec* pairs;          // per binned segment, item-contiguous
    SegRec* tmpl;            // per batch image: its SegRec template (tslot = batch position)
    int4* items;             // (brick, first pair, n pairs, 0)
    int* ctl;
    double* part;
    int32_t* bidx;           // the batch rows the work items in scratch were binned for (reuse check)
    int* gate;               // non-NULL: the binning kernels run only if *gate != 0 (set by the check)
    int cap_pairs, cap_items;
    float out_scale;         // the flush adds out_scale * (sum of contributions) to acc (1 = plain accumulator)
    int mc;                  // acc is a multicast address (fsld_nvls): the flush is multimem.red (table kernel)
    // fused step (table-driven kernel, fsld_loss_grad_step_planned): acc = lam v first (each CTA a
    // slice, ||v||^2 partials in fnorm), the flushes wait until every slice is written (ctl[6]), and
    // the last CTA to finish (ctl[7]) forms *fsq / *floss and re-arms both counters -- the whole
    // step in one kernel launch (+ the claim-counter reset)
    int fuse;
    // deterministic mode (table-driven kernel): work items in brick order with their segments
    // sorted by dataset offset, the flush converts each item's int32 sums to int64 fixed point at
    // the caller's scale *fxp (order-free integer adds), and the loss is summed per item in item order
    int det;
    const double* fxp;
    float flam;
    double fscale;
    double* fnorm;
    double* fsq;
    double* floss;
};

cudaError_t launch_sorted_count(int M, int n_mask, const short2* pix, const fsld_image_rec* recs, int N,
                                int32_t* seg_off, cudaStream_t s);
cudaError_t launch_sorted_fill(int M, int n_mask, const short2* pix, const fsld_image_rec* recs, int N,
                               const float2* x_in, float2* x_out, char2* pc_out, const int32_t* seg_off,
                               int2* segs, cudaStream_t s);
size_t sorted_tables_bytes(long long npx);
cudaError_t launch_sorted_tables(int M, int n_mask, int mode, const fsld_image_rec* recs, int N, const char2* pc,
                                 const int32_t* seg_off, const int2* segs, void* ptab, cudaStream_t s);
cudaError_t launch_sorted_loss_grad(const SortedArgs& a, double* sq_out, cudaStream_t s);
cudaError_t launch_sorted_loss_grad_det(const SortedArgs& a, double* sq_out, cudaStream_t s);
cudaError_t launch_sorted_loss_tab(const SortedArgs& a, double* sq_out, cudaStream_t s);
cudaError_t launch_sorted_diag(const SortedArgs& a, cudaStream_t s);
constexpr int kDetMaxBatch = 1024;  // deterministic brick path: <= 2 segments per image and brick -> 2048 per sort
cudaError_t launch_planned_loss_grad(const SortedArgs& a, double* sq_out, cudaStream_t s);
cudaError_t launch_sorted_bin(const SortedArgs& a, cudaStream_t s);
struct SlabMap {                 // brick z-layer -> slab of the host step (nb <= 32 for M <= 256)
    unsigned char of_layer[32];
};
cudaError_t launch_slab_items(const SortedArgs& a, const SlabMap& map, int G, int4* gitems, int* gctl, cudaStream_t s);
cudaError_t launch_sorted_pass(const SortedArgs& a, cudaStream_t s, int* grid);
cudaError_t prepare_host_step(int* grid_out);  // per device; grid of the slab passes
cudaError_t launch_plan_build(SortedArgs a, const PlanLayout& P, char* plan, cudaStream_t s);  // + hutch if a.zbits
cudaError_t set_phase_profile(unsigned long long* buf);

cudaError_t launch_slice(int op, int mode, bool det, const SliceArgs& a, int nblocks, cudaStream_t s);
cudaError_t launch_reduce(const double* part, int n, double* out, cudaStream_t s);
cudaError_t launch_ball(bool gather, int64_t n, const int32_t* idx, const void* src, void* dst, int elem_bytes,
                        cudaStream_t s);
cudaError_t launch_reduce_cols(const double* part, int n, int ncols, double* out, cudaStream_t s);
cudaError_t launch_grad_init(int64_t nvox, const float2* v, double lam, float2* grad, double* part, int nparts,
                             cudaStream_t s);
cudaError_t launch_loss_finalize(const double* part_sq, int n_sq, const double* part_norm, int n_norm, double scale,
                                 double lam, double* sq_out, double* loss, cudaStream_t s);
cudaError_t launch_planned_loss_grad_step(SortedArgs a, int64_t nvox, double scale, double lam, double* sq_out,
                                          double* loss, double* norm_part, int n_norm, cudaStream_t s);

// Algorithm-1 step kernels (fsld_step.cu)
cudaError_t launch_precond_step(int64_t nvox, float2* acc, const float2* v, float* fold, float* d_avg, float* d,
                                const float* dhat_fixed, const fsld_step_params& p, float2* dir, float2* grad_out,
                                float* dhat_out, double* out4, double* part, int nparts, cudaStream_t s);
cudaError_t launch_armijo_select(const double* sq, const double* rq, const double* qq, const double* vol,
                                 double scale, double lam, double c, int max_halvings, fsld_armijo_state* st,
                                 double* hist, int hist_cap, cudaStream_t s);
cudaError_t launch_sorted_energy(const SortedArgs& a, double* out, bool rebin, cudaStream_t s);
cudaError_t launch_sorted_hutch(const SortedArgs& a, int k, cudaStream_t s);
cudaError_t launch_apply_step(int64_t nvox, float2* v, const float2* dir, const fsld_armijo_state* st,
                              cudaStream_t s);
cudaError_t launch_assign_nn(const SliceArgs& a, int nblocks, int32_t* out, cudaStream_t s);
cudaError_t launch_hutch(int mode, bool det, const SliceArgs& a, int nblocks, const uint32_t* zbits,
                         int words, int k, cudaStream_t s);
cudaError_t launch_pack_probes(int64_t n, int k, const double* z, uint32_t* zbits, int* bad, cudaStream_t s);
cudaError_t launch_gen_probes(int64_t n, int k, uint64_t seed, uint32_t* zbits, cudaStream_t s);
cudaError_t launch_fixed_scale(const float2* data, int64_t n, double mult, double add, double* fx,
                               cudaStream_t s);
cudaError_t launch_grad_finalize(int64_t nvox, const void* acc, bool det, const double* fx,
                                 const float2* v, double scale, double lam, float2* out, cudaStream_t s);
cudaError_t launch_real_finalize(int64_t nvox, const void* acc, bool det, const double* fx, double scale,
                                 double add, float* out, cudaStream_t s);
int fsc_grid();
cudaError_t launch_cast_c64_c128(int64_t n, const void* src, void* dst, cudaStream_t s);
// rows of the touched ball: volume -> packed (pack) or packed -> volume; rows[r] = (voxel offset, length, packed offset, -)
cudaError_t launch_ball_rows(bool pack, const int4* rows, int nrows, const void* src, void* dst, cudaStream_t s);
cudaError_t launch_ctf_ring_power(const fsld_image_rec* recs, int N, const short2* ring, int n_ring, double* out,
                                  cudaStream_t s);
cudaError_t launch_fsc(int M, int R, const float2* u, const float2* v, double* part, double* out, cudaStream_t s);
cudaError_t launch_mask_images(int M, int n_mask, const int32_t* mask, int N, const void* in, void* out,
                               cudaStream_t s);
cudaError_t launch_norm2(int64_t n, const float2* v, double* out, double* part, int nparts, cudaStream_t s);
cudaError_t launch_grad_epilogue(int64_t nvox, float2* acc, const float2* v, double scale, double lam, float2* grad,
                                 const double* sq, double* loss, double* norm2, double* part, int nparts,
                                 cudaStream_t s);

}  // namespace fsld
