// fsld_kernels.cuh -- launch interface between the C ABI (fsld_capi.cu) and the kernels.
#pragma once

#include "fsld_common.cuh"

namespace fsld {

enum Op { OP_PROJECT = 0, OP_LOSS, OP_LOSS_GRAD, OP_BACKPROJECT, OP_HVP, OP_DIAG };

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
};

// ---------------------------------------------------------------------------
// Brick-binned path (fsld_brick.cu): the volume is cut into BT^3 bricks in
// frequency space; every (brick, batch image) pair whose slice plane crosses
// the brick is binned, and one CTA per work item (brick, <= BC images)
// gathers from / scatters into a shared-memory copy of the brick (+1 halo),
// so the adjoint costs one global reduction per brick voxel per item
// instead of 8 per pixel.
// ---------------------------------------------------------------------------
constexpr int BT = 8;                 // brick edge (voxels)
constexpr int BH = BT + 1;            // + halo for the floor+1 corners
constexpr int BH3 = BH * BH * BH;     // 729
constexpr int BC = 32;                // images per work item
constexpr int BW = 8;                 // warps per CTA
constexpr int BTHREADS = BW * 32;
constexpr int BMAXCAND = 448;         // per-warp candidate table (rows*row length bound)
constexpr uint32_t kGeomMagic = 0xF51DB200u;

struct GeomHeader {   // at the start of the scratch buffer (256-byte slot)
    uint32_t magic;
    int M, n_mask, pad0;
    const void* pix;
    unsigned rmax2;   // max kx^2+ky^2 over the mask
    int pad1[9];
};

struct ScratchLayout {
    size_t hdr, pix2p, rowmin, rowmax, cnt, off, fill, pairs, items, ctl, part, total;
    int nb, nbr, cap_pairs, cap_items, cap_part;
};

ScratchLayout scratch_layout(int M, int n_mask, int B);

struct BrickArgs {
    int M, c, nb, nbr, n_mask, B;
    float bnd;
    const int* pix2p;       // M*M -> compact pixel index or -1
    const int* rowmin;      // per py row (index py + c): min px (or large)
    const int* rowmax;
    const GeomHeader* hdr;
    const fsld_image_rec* recs;
    const int32_t* idx;
    const float2* v;
    const float2* x;
    float2* acc;
    int* cnt;
    int* off;
    int* fill;
    int* pairs;
    int4* items;
    int* ctl;
    double* part;
    int cap_pairs, cap_items;
};

cudaError_t launch_geom_prepare(int M, int n_mask, const short2* pix, const ScratchLayout& L, char* scratch,
                                cudaStream_t s);
cudaError_t launch_brick_loss_grad(const BrickArgs& a, double* sq_out, cudaStream_t s);

cudaError_t launch_slice(int op, int mode, bool det, const SliceArgs& a, int nblocks, cudaStream_t s);
cudaError_t launch_reduce(const double* part, int n, double* out, cudaStream_t s);
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
cudaError_t launch_norm2(int64_t n, const float2* v, double* out, double* part, int nparts, cudaStream_t s);

}  // namespace fsld
