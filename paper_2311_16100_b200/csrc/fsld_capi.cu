// fsld_capi.cu -- extern "C" entry points of libfsld_b200.so (include/fsld_b200.h).
//
// Validates arguments the way the reference raises ValueError (empty batch
// forward.py:562-563 / optim.py:179-180, bad mode forward.py:280-281), picks
// the launch geometry and enqueues the kernels on the caller's stream.
// Never throws, never synchronises.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>


#include "fsld_hostpool.h"
#include "fsld_kernels.cuh"

using namespace fsld;

namespace {

constexpr int kPixPerThreadTarget = 4;

// CUDA error -> status; FSLD_DEBUG=1 in the environment prints the CUDA error string to stderr.
int status_of(cudaError_t e) {
    if (e == cudaSuccess) return FSLD_OK;
    static const bool dbg = std::getenv("FSLD_DEBUG") != nullptr;
    if (dbg) std::fprintf(stderr, "fsld: CUDA error %d (%s)\n", (int)e, cudaGetErrorString(e));
    return FSLD_ECUDA;
}

bool geom_ok(int M, int mode, int n_mask, int B) {
    if (M < 2 || M > 1024) return false;
    if (mode != FSLD_MODE_NN && mode != FSLD_MODE_TRI) return false;
    if (n_mask < 1 || n_mask > M * M) return false;
    if (B < 1) return false;
    return true;
}

void tiling(int n_mask, int& tiles, int& ppt) {
    tiles = (n_mask + kThreads * kPixPerThreadTarget - 1) / (kThreads * kPixPerThreadTarget);
    if (tiles < 1) tiles = 1;
    ppt = (n_mask + kThreads * tiles - 1) / (kThreads * tiles);
}

SliceArgs make_args(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs, const int32_t* idx) {
    SliceArgs a{};
    a.M = M;
    a.c2 = (M + 1) / 2;
    a.bnd = (double)(M / 2 - 1);
    a.n_mask = n_mask;
    tiling(n_mask, a.tiles, a.ppt);
    a.pix = reinterpret_cast<const short2*>(pix);
    a.recs = recs;
    a.idx = idx;
    return a;
}

// Host-side record of the batch whose work items the last sorted call left in a scratch buffer
// (FSLD_REUSE_BINS check).  Not thread-safe across host threads sharing one scratch buffer.
struct BinKey {
    const void* scratch;
    const int32_t* idx;
    const fsld_image_rec* recs;
    int M, n_mask, B;
};
BinKey g_last_bins[8];
int g_last_bins_next = 0;
std::mutex g_registry_mu;  // guards the host-side bin / plan records (any host thread may call the ABI)

void note_bins(const void* scratch, const int32_t* idx, const fsld_image_rec* recs, int M, int n_mask, int B) {
    std::lock_guard<std::mutex> lk(g_registry_mu);
    for (BinKey& k : g_last_bins)
        if (k.scratch == scratch) {
            k = BinKey{scratch, idx, recs, M, n_mask, B};
            return;
        }
    g_last_bins[g_last_bins_next] = BinKey{scratch, idx, recs, M, n_mask, B};
    g_last_bins_next = (g_last_bins_next + 1) % 8;
}

void forget_bins(const void* scratch) {
    std::lock_guard<std::mutex> lk(g_registry_mu);
    for (BinKey& k : g_last_bins)
        if (k.scratch == scratch) k = BinKey{};
}

bool bins_match(const void* scratch, const int32_t* idx, const fsld_image_rec* recs, int M, int n_mask, int B) {
    std::lock_guard<std::mutex> lk(g_registry_mu);
    for (const BinKey& k : g_last_bins)
        if (k.scratch == scratch)
            return k.idx == idx && k.recs == recs && k.M == M && k.n_mask == n_mask && k.B == B;
    return false;
}

SortedArgs make_sorted(const ScratchLayout& L, int M, int n_mask, int B, const fsld_image_rec* recs,
                       const int32_t* idx, const void* v, const void* xs, const int8_t* pc, const int32_t* seg_off,
                       const int32_t* segs, void* grad_acc, void* scratch, const void* ptab = nullptr) {
    char* scr = reinterpret_cast<char*>(scratch);
    SortedArgs b{};
    b.ptab = ptab;
    b.M = M;
    b.c = (M + 1) / 2;
    b.nb = L.nb;
    b.nbr = L.nbr;
    b.n_mask = n_mask;
    b.B = B;
    b.bnd = (float)(M / 2 - 1);
    b.recs = recs;
    b.idx = idx;
    b.v = reinterpret_cast<const float2*>(v);
    b.xs = reinterpret_cast<const float2*>(xs);
    b.pc = reinterpret_cast<const char2*>(pc);
    b.seg_off = seg_off;
    b.segs = reinterpret_cast<const int2*>(segs);
    b.acc = reinterpret_cast<float2*>(grad_acc);
    b.cnt = reinterpret_cast<int*>(scr + L.cnt);
    b.off = reinterpret_cast<int*>(scr + L.off);
    b.fill = reinterpret_cast<int*>(scr + L.fill);
    b.pairs = reinterpret_cast<PairRec*>(scr + L.pairs);
    b.tmpl = reinterpret_cast<SegRec*>(scr + L.tmpl);
    b.items = reinterpret_cast<int4*>(scr + L.items);
    b.ctl = reinterpret_cast<int*>(scr + L.ctl);
    b.part = reinterpret_cast<double*>(scr + L.part);
    b.bidx = reinterpret_cast<int32_t*>(scr + L.bidx);
    b.gate = nullptr;
    b.cap_pairs = L.cap_pairs;
    b.cap_items = L.cap_items;
    b.out_scale = 1.0f;
    return b;
}

}  // namespace

namespace {
void drop_host_graphs_using(const void* p);  // (fsld_loss_grad_host's graph cache, below)
}  // namespace

extern "C" {

int fsld_abi_version(void) { return FSLD_ABI_VERSION; }

const char* fsld_status_string(int status) {
    switch (status) {
        case FSLD_OK: return "ok";
        case FSLD_EINVAL: return "invalid argument";
        case FSLD_ECUDA: return "CUDA error";
        case FSLD_ENODEV: return "no compute-capability-10.x device";
    }
    return "unknown status";
}

int fsld_device_count(int* count) {
    if (!count) return FSLD_EINVAL;
    int n = 0;
    *count = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return FSLD_ENODEV;
    }
    int good = 0;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++good;
    }
    *count = good;
    return good > 0 ? FSLD_OK : FSLD_ENODEV;
}

int fsld_host_alloc(size_t bytes, void** out) {
    if (!out || bytes == 0) return FSLD_EINVAL;
    *out = nullptr;
    return status_of(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
}

int fsld_host_free(void* p) {
    if (!p) return FSLD_OK;
    drop_host_graphs_using(p);  // a replay must never touch a freed (and maybe re-allocated) buffer
    return status_of(cudaFreeHost(p));
}

size_t fsld_scratch_bytes(int M, int n_mask, int B) {
    if (M < 2 || M > 1024) return 0;
    return scratch_layout(M, n_mask > 0 ? n_mask : 1, B > 0 ? B : 1).total;
}

int fsld_prepare(int M, int n_mask, const int16_t* pix, void* scratch, size_t scratch_bytes, void* stream) {
    if (M < 2 || M > 1024 || n_mask < 1 || n_mask > M * M || !pix || !scratch) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, 1);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // zero everything once (the brick binning relies on cnt[] == 0 on entry)
    cudaError_t e = cudaMemsetAsync(scratch, 0, scratch_bytes, s);
    if (e != cudaSuccess) return FSLD_ECUDA;
    GeomHeader h{};
    h.magic = kGeomMagic;
    h.M = M;
    h.n_mask = n_mask;
    h.pix = pix;
    return status_of(cudaMemcpyAsync(reinterpret_cast<char*>(scratch) + L.hdr, &h, sizeof(h), cudaMemcpyHostToDevice, s));
}

static int run_reducing(int op, int M, int mode, int n_mask, const int16_t* pix, const int8_t* pc,
                        const fsld_image_rec* recs, const int32_t* idx, int B, const void* v, const void* x,
                        void* grad_acc, double* sq_out, unsigned flags, const double* fx_scale, void* scratch,
                        size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B)) return FSLD_EINVAL;
    if ((!pix && !pc) || !recs || !v || !x || !sq_out || !scratch) return FSLD_EINVAL;
    if (op == OP_LOSS_GRAD && !grad_acc) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    char* scr = reinterpret_cast<char*>(scratch);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    SliceArgs a = make_args(M, n_mask, pix, recs, idx);
    const int nblocks = B * a.tiles;
    a.v = reinterpret_cast<const float2*>(v);
    a.x = reinterpret_cast<const float2*>(x);
    a.x_by_idx = 1;
    a.acc = grad_acc;
    a.partials = reinterpret_cast<double*>(scr + L.part);
    a.fx = fx_scale;
    a.pc = reinterpret_cast<const char2*>(pc);
    cudaError_t e = launch_slice(op, mode, det, a, nblocks, s);
    if (e != cudaSuccess) return FSLD_ECUDA;
    return status_of(launch_reduce(a.partials, nblocks, sq_out, s));
}

int fsld_loss_grad(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                   const int32_t* idx, int B, const void* v, const void* x, void* grad_acc, double* sq_out,
                   unsigned flags, const double* fx_scale, void* scratch, size_t scratch_bytes, void* stream) {
    return run_reducing(OP_LOSS_GRAD, M, mode, n_mask, pix, nullptr, recs, idx, B, v, x, grad_acc, sq_out, flags,
                        fx_scale, scratch, scratch_bytes, stream);
}

int fsld_loss(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, const int32_t* idx,
              int B, const void* v, const void* x, double* sq_out, void* scratch, size_t scratch_bytes,
              void* stream) {
    return run_reducing(OP_LOSS, M, mode, n_mask, pix, nullptr, recs, idx, B, v, x, nullptr, sq_out, 0u, nullptr,
                        scratch, scratch_bytes, stream);
}

int fsld_project(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                 const int32_t* idx, int B, const void* v, void* out, void* stream) {
    if (!geom_ok(M, mode, n_mask, B)) return FSLD_EINVAL;
    if (!pix || !recs || !v || !out) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, idx);
    a.v = reinterpret_cast<const float2*>(v);
    a.out = reinterpret_cast<float2*>(out);
    return status_of(launch_slice(OP_PROJECT, mode, false, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

static int run_scatter(int op, int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                       const int32_t* idx, int B, const void* src, void* acc, unsigned flags,
                       const double* fx_scale, void* stream) {
    if (!geom_ok(M, mode, n_mask, B)) return FSLD_EINVAL;
    if (!pix || !recs || !acc) return FSLD_EINVAL;
    if (op != OP_DIAG && !src) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, idx);
    if (op == OP_BACKPROJECT) {
        a.x = reinterpret_cast<const float2*>(src);
        a.x_by_idx = 0;
    } else {
        a.v = reinterpret_cast<const float2*>(src);
    }
    a.acc = acc;
    a.fx = fx_scale;
    return status_of(launch_slice(op, mode, det, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_backproject(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                     const int32_t* idx, int B, const void* img, void* acc, unsigned flags,
                     const double* fx_scale, void* stream) {
    return run_scatter(OP_BACKPROJECT, M, mode, n_mask, pix, recs, idx, B, img, acc, flags, fx_scale, stream);
}

int fsld_hvp(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, const int32_t* idx,
             int B, const void* z, void* acc, unsigned flags, const double* fx_scale, void* stream) {
    return run_scatter(OP_HVP, M, mode, n_mask, pix, recs, idx, B, z, acc, flags, fx_scale, stream);
}

int fsld_exact_diag(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                    const int32_t* idx, int B, void* acc, unsigned flags, const double* fx_scale, void* stream) {
    return run_scatter(OP_DIAG, M, mode, n_mask, pix, recs, idx, B, nullptr, acc, flags, fx_scale, stream);
}

int fsld_hutch_fold(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs,
                    const int32_t* idx, int B, const uint32_t* zbits, int k, void* acc, unsigned flags,
                    const double* fx_scale, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || k < 1) return FSLD_EINVAL;
    if (!pix || !recs || !zbits || !acc) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, idx);
    a.acc = acc;
    a.fx = fx_scale;
    return status_of(launch_hutch(mode, det, a, B * a.tiles, zbits, (k + 31) / 32, k,
                                  reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_pack_probes(int64_t n, int k, const double* z, uint32_t* zbits, int* bad, void* stream) {
    if (n < 1 || k < 1 || !z || !zbits) return FSLD_EINVAL;
    return status_of(launch_pack_probes(n, k, z, zbits, bad, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_gen_probes(int64_t n, int k, uint64_t seed, uint32_t* zbits, void* stream) {
    if (n < 1 || k < 1 || !zbits) return FSLD_EINVAL;
    return status_of(launch_gen_probes(n, k, seed, zbits, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_assign_nn(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs, const int32_t* idx, int B,
                   int32_t* out, void* stream) {
    if (!geom_ok(M, FSLD_MODE_NN, n_mask, B) || !pix || !recs || !out) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, idx);
    return status_of(launch_assign_nn(a, B * a.tiles, out, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_project_tab(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int B,
                     const void* v, const void* ftab, void* out, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || !pix || !recs || !v || !ftab || !out) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, nullptr);
    a.v = reinterpret_cast<const float2*>(v);
    a.ftab = reinterpret_cast<const float2*>(ftab);
    a.out = reinterpret_cast<float2*>(out);
    return status_of(launch_slice(OP_PROJECT, mode, false, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_backproject_tab(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int B,
                         const void* img, const void* ftab, void* acc, unsigned flags, const double* fx_scale,
                         void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || !pix || !recs || !img || !ftab || !acc) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, nullptr);
    a.x = reinterpret_cast<const float2*>(img);
    a.ftab = reinterpret_cast<const float2*>(ftab);
    a.acc = acc;
    a.fx = fx_scale;
    return status_of(launch_slice(OP_BACKPROJECT, mode, det, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_scatter_sq_tab(int M, int mode, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int B,
                        const void* wtab, void* acc, unsigned flags, const double* fx_scale, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || !pix || !recs || !wtab || !acc) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, pix, recs, nullptr);
    a.ftab = reinterpret_cast<const float2*>(wtab);
    a.acc = acc;
    a.fx = fx_scale;
    return status_of(launch_slice(OP_DIAG, mode, det, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- brick-sorted dataset layout

int fsld_sorted_count(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int N, int32_t* seg_off,
                      void* stream) {
    if (M < 2 || M > 256 || n_mask < 1 || n_mask > 65535 || N < 1 || !pix || !recs || !seg_off) return FSLD_EINVAL;
    return status_of(launch_sorted_count(M, n_mask, reinterpret_cast<const short2*>(pix), recs, N, seg_off,
                                         reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_sorted_fill(int M, int n_mask, const int16_t* pix, const fsld_image_rec* recs, int N, const void* x_in,
                     void* x_out, int8_t* pc_out, const int32_t* seg_off, int32_t* segs, void* stream) {
    if (M < 2 || M > 256 || n_mask < 1 || n_mask > 65535 || N < 1 || !pix || !recs || !pc_out || !seg_off || !segs)
        return FSLD_EINVAL;
    if (x_in && !x_out) return FSLD_EINVAL;
    return status_of(launch_sorted_fill(M, n_mask, reinterpret_cast<const short2*>(pix), recs, N,
                                        reinterpret_cast<const float2*>(x_in), reinterpret_cast<float2*>(x_out),
                                        reinterpret_cast<char2*>(pc_out), seg_off, reinterpret_cast<int2*>(segs),
                                        reinterpret_cast<cudaStream_t>(stream)));
}

size_t fsld_sorted_tables_bytes(int N, int n_mask) {
    if (N < 1 || n_mask < 1) return 0;
    return sorted_tables_bytes((long long)N * n_mask);
}

int fsld_sorted_tables(int M, int mode, int n_mask, const fsld_image_rec* recs, int N, const int8_t* pc,
                       const int32_t* seg_off, const int32_t* segs, void* ptab, void* stream) {
    if (M < 2 || M > 256 || n_mask < 1 || n_mask > 65535 || N < 1 || !recs || !pc || !seg_off || !segs || !ptab)
        return FSLD_EINVAL;
    if (mode != FSLD_MODE_NN && mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (reinterpret_cast<uintptr_t>(ptab) & 255) return FSLD_EINVAL;
    return status_of(launch_sorted_tables(M, n_mask, mode, recs, N, reinterpret_cast<const char2*>(pc), seg_off,
                                          reinterpret_cast<const int2*>(segs), ptab,
                                          reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_loss_grad_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                          const void* v, const void* xs, const int8_t* pc, const void* ptab, const int32_t* seg_off,
                          const int32_t* segs,
                          void* grad_acc, double* sq_out, unsigned flags, const double* fx_scale, void* scratch,
                          size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256) return FSLD_EINVAL;
    if (!recs || !v || !xs || !pc || !grad_acc || !sq_out || !scratch) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    // deterministic mode on the table-driven brick kernel (trilinear, tables built, B <= 1024)
    if (det && mode == FSLD_MODE_TRI && ptab && seg_off && segs && B <= kDetMaxBatch && !(flags & FSLD_TILE_PATH)) {
        const ScratchLayout L = scratch_layout(M, n_mask, B);
        if (scratch_bytes < L.total) return FSLD_EINVAL;
        SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, v, xs, pc, seg_off, segs, grad_acc, scratch, ptab);
        b.fxp = fx_scale;
        forget_bins(scratch);  // (these work items are in the deterministic order: not reused by FSLD_REUSE_BINS)
        return status_of(launch_sorted_loss_grad_det(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
    }
    // brick kernels: trilinear (tables or compute path); nearest-neighbour with tables on request
    const bool brick = (mode == FSLD_MODE_TRI || (ptab && (flags & FSLD_NN_BRICK))) && !det &&
                       !(flags & FSLD_TILE_PATH) && seg_off && segs;
    if (!brick)
        return run_reducing(OP_LOSS_GRAD, M, mode, n_mask, nullptr, pc, recs, idx, B, v, xs, grad_acc, sq_out, flags,
                            fx_scale, scratch, scratch_bytes, stream);
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, v, xs, pc, seg_off, segs, grad_acc, scratch, ptab);
    b.nn = mode == FSLD_MODE_NN;
    note_bins(scratch, idx, recs, M, n_mask, B);
    return status_of(launch_sorted_loss_grad(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_hvp_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B, const void* z,
                    const int8_t* pc, const void* ptab, const int32_t* seg_off, const int32_t* segs, void* acc, double* sq_out,
                    unsigned flags, void* scratch, size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || (mode != FSLD_MODE_TRI && !ptab)) return FSLD_EINVAL;
    if (flags & (FSLD_DETERMINISTIC | FSLD_TILE_PATH)) return FSLD_EINVAL;
    if (!recs || !idx || !z || !pc || !seg_off || !segs || !acc || !sq_out || !scratch) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    // xs = NULL: the kernel takes the images as zero (r = f P z)
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, z, nullptr, pc, seg_off, segs, acc, scratch, ptab);
    b.nn = mode == FSLD_MODE_NN;
    note_bins(scratch, idx, recs, M, n_mask, B);
    return status_of(launch_sorted_loss_grad(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_loss_grad_hutch_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                                const void* v, const void* xs, const int8_t* pc, const void* ptab,
                                const int32_t* seg_off,
                                const int32_t* segs, const uint32_t* zbits, void* grad_acc, float* fold,
                                double* sq_out, unsigned flags, void* scratch, size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (flags & (FSLD_DETERMINISTIC | FSLD_TILE_PATH)) return FSLD_EINVAL;
    if (!recs || !v || !xs || !pc || !seg_off || !segs || !zbits || !grad_acc || !fold || !sq_out || !scratch)
        return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, v, xs, pc, seg_off, segs, grad_acc, scratch, ptab);
    b.zbits = zbits;
    b.fold = fold;
    note_bins(scratch, idx, recs, M, n_mask, B);
    return status_of(launch_sorted_loss_grad(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_loss_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                     const void* v, const void* xs, const int8_t* pc, double* sq_out, void* scratch,
                     size_t scratch_bytes, void* stream) {
    if (!pc) return FSLD_EINVAL;
    return run_reducing(OP_LOSS, M, mode, n_mask, nullptr, pc, recs, idx, B, v, xs, nullptr, sq_out, 0u, nullptr,
                        scratch, scratch_bytes, stream);
}

int fsld_loss_sorted_tab(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                         const void* v, const void* xs, const int8_t* pc, const void* ptab, const int32_t* seg_off,
                         const int32_t* segs, double* sq_out, void* scratch, size_t scratch_bytes, void* stream) {
    if (!ptab || mode != FSLD_MODE_TRI || !seg_off || !segs)  // (no tables / nn: the tile kernel)
        return fsld_loss_sorted(M, mode, n_mask, recs, idx, B, v, xs, pc, sq_out, scratch, scratch_bytes, stream);
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || !recs || !v || !xs || !pc || !sq_out || !scratch)
        return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, v, xs, pc, seg_off, segs, nullptr, scratch, ptab);
    forget_bins(scratch);  // (these work items replace whatever the scratch held)
    return status_of(launch_sorted_loss_tab(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_exact_diag_sorted_tab(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                               const int8_t* pc, const void* ptab, const int32_t* seg_off, const int32_t* segs,
                               void* acc, unsigned flags, const double* fx_scale, void* scratch, size_t scratch_bytes,
                               void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (!recs || !pc || !ptab || !seg_off || !segs || !acc || !scratch) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && (!fx_scale || B > kDetMaxBatch)) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, nullptr, nullptr, pc, seg_off, segs, nullptr, scratch, ptab);
    b.fold = reinterpret_cast<float*>(acc);
    b.det = det ? 1 : 0;
    b.fxp = fx_scale;
    forget_bins(scratch);
    return status_of(launch_sorted_diag(b, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_project_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                        const void* v, const int8_t* pc, void* out, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || !recs || !v || !pc || !out) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, nullptr, recs, idx);
    a.v = reinterpret_cast<const float2*>(v);
    a.out = reinterpret_cast<float2*>(out);
    a.pc = reinterpret_cast<const char2*>(pc);
    a.x_by_idx = 1;
    return status_of(launch_slice(OP_PROJECT, mode, false, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_backproject_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int B,
                            const void* xs, const int8_t* pc, void* acc, unsigned flags, const double* fx_scale,
                            void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || !recs || !xs || !pc || !acc) return FSLD_EINVAL;
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (det && !fx_scale) return FSLD_EINVAL;
    SliceArgs a = make_args(M, n_mask, nullptr, recs, idx);
    a.x = reinterpret_cast<const float2*>(xs);
    a.x_by_idx = 1;
    a.pc = reinterpret_cast<const char2*>(pc);
    a.acc = acc;
    a.fx = fx_scale;
    return status_of(launch_slice(OP_BACKPROJECT, mode, det, a, B * a.tiles, reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_fixed_scale(const void* data, int64_t n, double mult, double add, double* fx_scale, void* stream) {
    if (!fx_scale || mult <= 0.0 || add < 0.0) return FSLD_EINVAL;
    return status_of(launch_fixed_scale(reinterpret_cast<const float2*>(data), n, mult, add, fx_scale,
                                        reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_grad_finalize(int64_t nvox, const void* acc, unsigned flags, const double* fx_scale, const void* v,
                       double scale, double lam, void* out, void* stream) {
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (nvox < 1 || !acc || !out || (det && !fx_scale)) return FSLD_EINVAL;
    return status_of(launch_grad_finalize(nvox, acc, det, fx_scale, reinterpret_cast<const float2*>(v), scale,
                                          lam, reinterpret_cast<float2*>(out),
                                          reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_real_finalize(int64_t nvox, const void* acc, unsigned flags, const double* fx_scale, double scale,
                       double add, float* out, void* stream) {
    const bool det = (flags & FSLD_DETERMINISTIC) != 0;
    if (nvox < 1 || !acc || !out || (det && !fx_scale)) return FSLD_EINVAL;
    return status_of(launch_real_finalize(nvox, acc, det, fx_scale, scale, add, out,
                                          reinterpret_cast<cudaStream_t>(stream)));
}

int fsld_norm2(int64_t n, const void* v, double* out, void* scratch, size_t scratch_bytes, void* stream) {
    const int nparts = 148 * 8;
    if (n < 1 || !v || !out || !scratch || scratch_bytes < nparts * sizeof(double)) return FSLD_EINVAL;
    // uses the first nparts doubles of the caller's scratch (a dedicated buffer, or any free region)
    return status_of(launch_norm2(n, reinterpret_cast<const float2*>(v), out, reinterpret_cast<double*>(scratch),
                                  nparts, reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"

extern "C" int fsld_grad_epilogue(int64_t nvox, void* acc, const void* v, double scale, double lam, void* grad,
                                  const double* sq, double* loss, double* norm2, void* scratch, size_t scratch_bytes,
                                  void* stream) {
    const int nparts = 148 * 8;
    if (nvox < 1 || !acc || !v || !grad || !sq || !scratch || scratch_bytes < nparts * sizeof(double))
        return FSLD_EINVAL;
    return status_of(launch_grad_epilogue(nvox, reinterpret_cast<float2*>(acc), reinterpret_cast<const float2*>(v),
                                          scale, lam, reinterpret_cast<float2*>(grad), sq, loss, norm2,
                                          reinterpret_cast<double*>(scratch), nparts,
                                          reinterpret_cast<cudaStream_t>(stream)));
}

// Debug: accumulate per-phase cycles of the brick kernel's item loop into buf[0..5]
// (5 phases + item count, summed over CTAs); NULL disables.  Not part of the stable ABI.
extern "C" int fsld_debug_phase_profile(unsigned long long* buf) {
    return status_of(set_phase_profile(buf));
}

// ---------------------------------------------------------------- Algorithm-1 step (fsld_step.cu)

extern "C" int fsld_precond_step(int64_t nvox, void* acc, const void* v, float* fold, float* d_avg, float* d,
                                 const float* dhat_fixed, const fsld_step_params* params, void* dir,
                                 void* grad_out, float* dhat_out, double* out4, void* scratch,
                                 size_t scratch_bytes, void* stream) {
    const int nparts = 148 * 4;  // one wave of precond_step_kernel (4 CTAs / SM)
    if (nvox < 1 || !acc || !v || !params || !dir || !out4 || !scratch ||
        scratch_bytes < 5 * nparts * sizeof(double))
        return FSLD_EINVAL;
    if (params->estimating && (!fold || !d_avg || !d)) return FSLD_EINVAL;
    for (const void* q : {(const void*)acc, v, (const void*)fold, (const void*)d_avg, (const void*)d,
                          (const void*)dhat_fixed, (const void*)dir, (const void*)grad_out, (const void*)dhat_out})
        if (reinterpret_cast<uintptr_t>(q) & 15) return FSLD_EINVAL;  // 16-byte vector accesses
    if (params->estimating && !(params->floor > 0.0)) return FSLD_EINVAL;
    return status_of(launch_precond_step(nvox, reinterpret_cast<float2*>(acc), reinterpret_cast<const float2*>(v),
                                         fold, d_avg, d, dhat_fixed, *params, reinterpret_cast<float2*>(dir),
                                         reinterpret_cast<float2*>(grad_out), dhat_out, out4,
                                         reinterpret_cast<double*>(scratch), nparts,
                                         reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_armijo_terms(int M, int mode, int n_mask, const int16_t* pix, const int8_t* pc,
                                 const fsld_image_rec* recs, const int32_t* idx, int B, const void* v,
                                 const void* d, const void* xs, double* out3, void* scratch, size_t scratch_bytes,
                                 void* stream) {
    if (!geom_ok(M, mode, n_mask, B)) return FSLD_EINVAL;
    if ((!pix && !pc) || !recs || !v || !d || !xs || !out3 || !scratch) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    char* scr = reinterpret_cast<char*>(scratch);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    SliceArgs a = make_args(M, n_mask, pix, recs, idx);
    const int nblocks = B * a.tiles;
    if (3 * nblocks > L.cap_part) return FSLD_EINVAL;
    a.v = reinterpret_cast<const float2*>(v);
    a.v2 = reinterpret_cast<const float2*>(d);
    a.x = reinterpret_cast<const float2*>(xs);
    a.x_by_idx = 1;
    a.partials = reinterpret_cast<double*>(scr + L.part);
    a.nparts = nblocks;
    a.pc = reinterpret_cast<const char2*>(pc);
    cudaError_t e = launch_slice(OP_ARMIJO, mode, false, a, nblocks, s);
    if (e != cudaSuccess) return FSLD_ECUDA;
    return status_of(launch_reduce_cols(a.partials, nblocks, 3, out3, s));
}

extern "C" int fsld_armijo_select(const double* sq, const double* rq, const double* qq, const double* vol,
                                  double scale, double lam, double c, int max_halvings, fsld_armijo_state* st,
                                  double* hist, int hist_cap, void* stream) {
    if (!sq || !rq || !qq || !vol || !st || !(scale > 0.0) || lam < 0.0 || !(c > 0.0 && c < 1.0) ||
        max_halvings < 0)
        return FSLD_EINVAL;
    return status_of(launch_armijo_select(sq, rq, qq, vol, scale, lam, c, max_halvings, st, hist, hist_cap,
                                          reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_hutch_fold_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx,
                                      int B, const int8_t* pc, const int32_t* seg_off, const int32_t* segs,
                                      const uint32_t* zbits, int k, float* fold, void* scratch, size_t scratch_bytes,
                                      void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI || k < 1 || k > 256) return FSLD_EINVAL;
    if (!recs || !pc || !seg_off || !segs || !zbits || !fold || !scratch) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, nullptr, nullptr, pc, seg_off, segs, nullptr, scratch);
    b.zbits = zbits;
    b.fold = fold;
    note_bins(scratch, idx, recs, M, n_mask, B);
    return status_of(launch_sorted_hutch(b, k, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_proj_energy_sorted(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx,
                                       int B, const void* d, const int8_t* pc, const int32_t* seg_off,
                                       const int32_t* segs, double* out, unsigned flags, void* scratch,
                                       size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (!recs || !d || !pc || !seg_off || !segs || !out || !scratch) return FSLD_EINVAL;
    if (flags & ~FSLD_REUSE_BINS) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    const bool reuse = (flags & FSLD_REUSE_BINS) != 0;
    if (reuse && !bins_match(scratch, idx, recs, M, n_mask, B)) return FSLD_EINVAL;
    SortedArgs b = make_sorted(L, M, n_mask, B, recs, idx, d, nullptr, pc, seg_off, segs, nullptr, scratch);
    if (reuse) b.gate = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) + L.gate);
    if (!reuse) note_bins(scratch, idx, recs, M, n_mask, B);
    return status_of(launch_sorted_energy(b, out, !reuse, reinterpret_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- metrics and ingest

extern "C" size_t fsld_fsc_scratch_bytes(int M, int max_radius) {
    if (M < 2 || max_radius < 0) return 0;
    return sizeof(double) * (size_t)fsc_grid() * 3 * (max_radius + 1);
}

extern "C" int fsld_fsc(int M, int max_radius, const void* u, const void* v, double* out, void* scratch,
                        size_t scratch_bytes, void* stream) {
    if (M < 2 || M > 1024 || max_radius < 0 || max_radius > M || !u || !v || !out || !scratch) return FSLD_EINVAL;
    if (scratch_bytes < fsld_fsc_scratch_bytes(M, max_radius)) return FSLD_EINVAL;
    return status_of(launch_fsc(M, max_radius, reinterpret_cast<const float2*>(u), reinterpret_cast<const float2*>(v),
                                reinterpret_cast<double*>(scratch), out, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_ctf_ring_power(const fsld_image_rec* recs, int N, const int16_t* ring, int n_ring, double* out,
                                   void* stream) {
    if (N < 0 || n_ring < 1 || (N > 0 && (!recs || !ring || !out))) return FSLD_EINVAL;
    return status_of(launch_ctf_ring_power(recs, N, reinterpret_cast<const short2*>(ring), n_ring, out,
                                           reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_mask_images(int M, int n_mask, const int32_t* mask, int N, const void* images, void* x,
                                void* stream) {
    if (M < 2 || n_mask < 1 || n_mask > M * M || N < 0 || !mask || (N > 0 && (!images || !x))) return FSLD_EINVAL;
    return status_of(launch_mask_images(M, n_mask, mask, N, images, x, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_apply_step(int64_t nvox, void* v, const void* dir, const fsld_armijo_state* st, void* stream) {
    if (nvox < 1 || !v || !dir || !st) return FSLD_EINVAL;
    if ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(dir)) & 15) return FSLD_EINVAL;
    return status_of(launch_apply_step(nvox, reinterpret_cast<float2*>(v), reinterpret_cast<const float2*>(dir), st,
                                       reinterpret_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- data-parallel all-reduce compaction

extern "C" int fsld_ball_gather(int64_t n, const int32_t* idx, const void* src, void* dst, int elem_bytes,
                                void* stream) {
    if (n < 1 || !idx || !src || !dst || (elem_bytes != 4 && elem_bytes != 8)) return FSLD_EINVAL;
    return status_of(launch_ball(true, n, idx, src, dst, elem_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_ball_scatter(int64_t n, const int32_t* idx, const void* src, void* dst, int elem_bytes,
                                 void* stream) {
    if (n < 1 || !idx || !src || !dst || (elem_bytes != 4 && elem_bytes != 8)) return FSLD_EINVAL;
    return status_of(launch_ball(false, n, idx, src, dst, elem_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- multi-batch binning plans

namespace {

struct PlanKey {
    const void* plan;
    int M, n_mask, K, B;
    long long total_pairs;
};
PlanKey g_plans[8];
int g_plans_next = 0;

void note_plan(const PlanKey& k) {
    std::lock_guard<std::mutex> lk(g_registry_mu);
    for (PlanKey& p : g_plans)
        if (p.plan == k.plan) {
            p = k;
            return;
        }
    g_plans[g_plans_next] = k;
    g_plans_next = (g_plans_next + 1) % 8;
}

bool find_plan(const void* plan, PlanKey& out) {
    std::lock_guard<std::mutex> lk(g_registry_mu);
    for (const PlanKey& p : g_plans)
        if (p.plan == plan) {
            out = p;
            return true;
        }
    return false;
}

// SortedArgs of batch k of a built plan (work items ready; scratch supplies the partial sums).
bool make_planned(SortedArgs& b, const void* plan, int M, int n_mask, int B, int k, const fsld_image_rec* recs,
                  const void* v, const void* xs, const int8_t* pc, void* grad_acc, void* scratch,
                  size_t scratch_bytes, const void* ptab = nullptr) {
    PlanKey pk;
    if (!find_plan(plan, pk)) return false;
    const PlanKey* p = &pk;
    if (p->M != M || p->n_mask != n_mask || p->B != B || k < 0 || k >= p->K) return false;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return false;
    const PlanLayout P = plan_layout(M, B, p->K, p->total_pairs);
    char* pl = reinterpret_cast<char*>(const_cast<void*>(plan));
    b = make_sorted(L, M, n_mask, B, recs, nullptr, v, xs, pc, nullptr, nullptr, grad_acc, scratch, ptab);
    b.ctl = reinterpret_cast<int*>(pl + P.ctl) + 16 * k;
    b.items = reinterpret_cast<int4*>(pl + P.items);
    b.pairs = reinterpret_cast<PairRec*>(pl + P.pairs);
    b.tmpl = reinterpret_cast<SegRec*>(pl + P.tmpl);
    b.cnt = b.off = b.fill = nullptr;  // binning already done
    return true;
}

}  // namespace

extern "C" size_t fsld_plan_bytes(int M, int n_mask, int B, int K, int64_t total_pairs) {
    if (M < 2 || M > 256 || n_mask < 1 || B < 1 || K < 1 || total_pairs < 0) return 0;
    return plan_layout(M, B, K, total_pairs).total;
}

extern "C" int fsld_plan_build(int M, int n_mask, const fsld_image_rec* recs, const int32_t* idx, int K, int B,
                               const int32_t* seg_off, const int32_t* segs, int64_t total_pairs, void* plan,
                               size_t plan_bytes, void* stream) {
    if (M < 2 || M > 256 || n_mask < 1 || n_mask > M * M || B < 1 || K < 1 || total_pairs < 0) return FSLD_EINVAL;
    if (!recs || !idx || !seg_off || !segs || !plan) return FSLD_EINVAL;
    const PlanLayout P = plan_layout(M, B, K, total_pairs);
    if (plan_bytes < P.total || P.cap_items > 0x7fffffffLL || total_pairs > 0x7fffffffLL) return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    SortedArgs a{};
    a.M = M;
    a.c = (M + 1) / 2;
    a.nb = L.nb;
    a.nbr = L.nbr;
    a.n_mask = n_mask;
    a.B = B;
    a.bnd = (float)(M / 2 - 1);
    a.recs = recs;
    a.idx = idx;
    a.seg_off = seg_off;
    a.segs = reinterpret_cast<const int2*>(segs);
    cudaError_t e = launch_plan_build(a, P, reinterpret_cast<char*>(plan), reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return FSLD_ECUDA;
    note_plan(PlanKey{plan, M, n_mask, K, B, (long long)total_pairs});
    return FSLD_OK;
}

extern "C" int fsld_loss_grad_planned(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan,
                                      int B, int k, const void* v, const void* xs, const int8_t* pc,
                                      const void* ptab, const uint32_t* zbits, void* grad_acc, float* fold, double* sq_out,
                                      void* scratch, size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (!recs || !plan || !v || !xs || !pc || !grad_acc || !sq_out || !scratch || (zbits && !fold)) return FSLD_EINVAL;
    SortedArgs b;
    if (!make_planned(b, plan, M, n_mask, B, k, recs, v, xs, pc, grad_acc, scratch, scratch_bytes, ptab))
        return FSLD_EINVAL;
    b.zbits = zbits;
    b.fold = fold;
    return status_of(launch_planned_loss_grad(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_loss_grad_planned_mc(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan,
                                         int B, int k, const void* v, const void* xs, const int8_t* pc,
                                         const void* ptab, void* grad_acc_mc, double* sq_out, void* scratch,
                                         size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (!recs || !plan || !v || !xs || !pc || !ptab || !grad_acc_mc || !sq_out || !scratch) return FSLD_EINVAL;
    SortedArgs b;
    if (!make_planned(b, plan, M, n_mask, B, k, recs, v, xs, pc, grad_acc_mc, scratch, scratch_bytes, ptab))
        return FSLD_EINVAL;
    b.mc = 1;
    return status_of(launch_planned_loss_grad(b, sq_out, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_loss_grad_step_planned(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan,
                                           int B, int k, const void* v, const void* xs, const int8_t* pc,
                                           const void* ptab, double scale, double lam, void* grad, double* sq_out, double* loss,
                                           void* scratch, size_t scratch_bytes, void* norm_scratch,
                                           size_t norm_scratch_bytes, void* stream) {
    const int n_norm = 148 * 8;
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (!recs || !plan || !v || !xs || !pc || !grad || !sq_out || !loss || !scratch || !norm_scratch ||
        norm_scratch_bytes < n_norm * sizeof(double) || v == grad)
        return FSLD_EINVAL;
    SortedArgs b;
    if (!make_planned(b, plan, M, n_mask, B, k, recs, v, xs, pc, grad, scratch, scratch_bytes, ptab))
        return FSLD_EINVAL;
    const int64_t nvox = (int64_t)M * M * M;
    return status_of(launch_planned_loss_grad_step(b, nvox, scale, lam, sq_out, loss,
                                                   reinterpret_cast<double*>(norm_scratch), n_norm,
                                                   reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int fsld_proj_energy_planned(int M, int mode, int n_mask, const fsld_image_rec* recs, const void* plan,
                                        int B, int k, const void* d, const int8_t* pc, double* out, void* scratch,
                                        size_t scratch_bytes, void* stream) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if (!recs || !plan || !d || !pc || !out || !scratch) return FSLD_EINVAL;
    SortedArgs b;
    if (!make_planned(b, plan, M, n_mask, B, k, recs, d, nullptr, pc, nullptr, scratch, scratch_bytes))
        return FSLD_EINVAL;
    return status_of(launch_sorted_energy(b, out, false, reinterpret_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- slab-pipelined host step
namespace {

// Per-device copy streams and events of fsld_loss_grad_host, created once.
struct HostPipe {
    cudaStream_t h2d = nullptr, d2h = nullptr, ks[2] = {nullptr, nullptr};
    cudaStream_t cap = nullptr;  // graphs are captured here (the caller's stream may be the legacy one)
    cudaEvent_t fork = nullptr, join = nullptr, eh[kMaxSlabs] = {}, ei[kMaxSlabs] = {}, ek[kMaxSlabs] = {},
                           ep[kMaxSlabs] = {};  // per slab: copied in, initialised, pass done, gradient packed
};
std::mutex g_pipe_mu;  // held while a call enqueues (the events are reused call after call)
HostPipe g_pipe[16];

cudaError_t pipe_for_device(HostPipe*& out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
    HostPipe& p = g_pipe[dev];
    if (!p.h2d) {
        const unsigned fl = cudaEventDisableTiming;
        if ((e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (int q = 0; q < 2; ++q)
            if ((e = cudaStreamCreateWithFlags(&p.ks[q], cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&p.cap, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&p.fork, fl)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&p.join, fl)) != cudaSuccess) return e;
        for (int g = 0; g < kMaxSlabs; ++g) {
            if ((e = cudaEventCreateWithFlags(&p.eh[g], fl)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&p.ek[g], fl)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&p.ei[g], fl)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&p.ep[g], fl)) != cudaSuccess) return e;
        }
    }
    out = &p;
    return cudaSuccess;
}

// Slabs of brick z-layers: first[g] .. first[g+1].  The copies in and out are the critical path, so
// the two slabs at each end are one layer thick (the first gradient slab is ready, and its copy
// out starts, early; little work is left after the last copy in) and the middle layers are split
// evenly into the remaining n_slabs - 4 (uniform slabs for n_slabs < 6 or few layers).
int slab_layers(int nb, int n_slabs, int* first) {
    int G = 0;
    first[0] = 0;
    if (n_slabs >= 6 && nb >= n_slabs) {
        const int mid = n_slabs - 4, mid_layers = nb - 4;
        int l = 0;
        for (int g = 0; g < 2; ++g) first[++G] = ++l;
        for (int g = 0; g < mid; ++g) first[++G] = (l += mid_layers / mid + (g < mid_layers % mid ? 1 : 0));
        for (int g = 0; g < 2; ++g) first[++G] = ++l;
        return G;
    }
    const int layers = (nb + n_slabs - 1) / n_slabs;
    for (int l = 0; l < nb;) first[++G] = (l = std::min(nb, l + layers));
    return G;
}

// Slab g = kz in [z0, z1) as at most two contiguous plane ranges of the FFT-ordered z axis.
int slab_pieces(int M, int z0, int z1, int zi0[2], int nz[2]) {
    int n = 0;
    if (z0 < 0) {
        zi0[n] = z0 + M;
        nz[n++] = (z1 < 0 ? z1 : 0) - z0;
    }
    if (z1 > 0) {
        const int a = z0 > 0 ? z0 : 0;
        zi0[n] = a;
        nz[n++] = z1 - a;
    }
    return n;
}

// The touched ball of the numpy-signature host step (fsld_loss_grad_host_np_ball), row by row: the voxels
// within the radius rt of the origin (the only ones a scatter can reach, grid.touched_ball) as one x range
// per storage row (z, y) -- one voxel of margin, rounded out to multiples of 4 voxels (whole 64-byte lines
// of complex128) -- and their packed order: slab by slab (as host_step_enqueue cuts them), plane by plane,
// row by row, so that every z-slab crosses PCIe as one contiguous range in each direction.
struct BallPack {
    int M = 0, n_slabs = 0, G = 0;
    double rt = 0.0;
    std::vector<int> xa, xb;        // per storage row z * M + y: the ball's voxels are x in [xa, xb)
    std::vector<int64_t> poff;      // per storage row: its offset in the packed order
    int row0[kMaxSlabs + 1] = {};   // slab g's rows in rows_dev
    int64_t off[kMaxSlabs + 1] = {};  // slab g's range of the packed order
    int sz[kMaxSlabs][2] = {}, sn[kMaxSlabs][2] = {}, snp[kMaxSlabs] = {};  // slab g's plane ranges (slab_pieces)
    int4* rows_dev = nullptr;       // (voxel offset, length, packed offset, -) of the non-empty rows, by slab
    float2 *vpack_dev = nullptr, *gpack_dev = nullptr;  // device staging of the packed volume / gradient
};

// The ball's x range [xa, xb) of the storage row (kz, ky), false if the row is off the ball.
bool ball_row(int M, int kz, int ky, double rt, int& xa, int& xb) {
    const int c = (M + 1) / 2;
    const double rem = rt * rt - (double)kz * kz - (double)ky * ky;
    if (rem < 0.0) return false;
    const int h = (int)std::sqrt(rem) + 1;
    xa = std::max(0, c - h) & ~3;
    xb = std::min(M, (c + h + 1 + 3) & ~3);
    return true;
}

void ball_pack_free(BallPack& bp) {
    cudaFree(bp.rows_dev);
    cudaFree(bp.vpack_dev);
    cudaFree(bp.gpack_dev);
    bp = BallPack{};
}

cudaError_t ball_pack_build(BallPack& bp, int M, int n_slabs, double rt) {
    ball_pack_free(bp);
    const int c = (M + 1) / 2, nb = (M + BT - 1) / BT;
    int first[kMaxSlabs + 1];
    bp.G = slab_layers(nb, n_slabs, first);
    bp.xa.assign((size_t)M * M, 0);
    bp.xb.assign((size_t)M * M, 0);
    bp.poff.assign((size_t)M * M, 0);
    std::vector<int4> rows;
    int64_t pos = 0;
    for (int g = 0; g < bp.G; ++g) {
        const int z0 = -c + BT * first[g], z1 = std::min(-c + BT * first[g + 1], M - c);
        bp.snp[g] = slab_pieces(M, z0, z1, bp.sz[g], bp.sn[g]);
        bp.row0[g] = (int)rows.size();
        bp.off[g] = pos;
        for (int q = 0; q < bp.snp[g]; ++q)
            for (int z = bp.sz[g][q]; z < bp.sz[g][q] + bp.sn[g][q]; ++z) {
                const int kz = z >= M - c ? z - M : z;
                for (int y = 0; y < M; ++y) {
                    int xa = 0, xb = 0;
                    if (!ball_row(M, kz, y - c, rt, xa, xb)) continue;
                    const size_t r = (size_t)z * M + y;
                    bp.xa[r] = xa;
                    bp.xb[r] = xb;
                    bp.poff[r] = pos;
                    rows.push_back(make_int4((int)(r * M + xa), xb - xa, (int)pos, 0));
                    pos += xb - xa;
                }
            }
    }
    bp.row0[bp.G] = (int)rows.size();
    bp.off[bp.G] = pos;
    cudaError_t e;
    if ((e = cudaMalloc(reinterpret_cast<void**>(&bp.rows_dev), sizeof(int4) * std::max<size_t>(1, rows.size()))) !=
            cudaSuccess ||
        (e = cudaMalloc(reinterpret_cast<void**>(&bp.vpack_dev), sizeof(float2) * (size_t)std::max<int64_t>(1, pos))) !=
            cudaSuccess ||
        (e = cudaMalloc(reinterpret_cast<void**>(&bp.gpack_dev), sizeof(float2) * (size_t)std::max<int64_t>(1, pos))) !=
            cudaSuccess ||
        (e = cudaMemcpy(bp.rows_dev, rows.data(), sizeof(int4) * rows.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
        ball_pack_free(bp);
        return e;
    }
    bp.M = M;
    bp.n_slabs = n_slabs;
    bp.rt = rt;
    return cudaSuccess;
}

}  // namespace

namespace {

// Everything a host step enqueues depends only on these (the batch rows are copied from a pinned
// staging buffer owned by the cached graph), so one captured graph per key is replayed.
struct HostStepKey {
    int M, n_mask, B, n_slabs;
    const void *recs, *v_host, *xs, *pc, *ptab, *seg_off, *segs, *grad_host, *out_host, *v_dev, *grad_dev,
        *idx_dev, *scratch, *grad_dev128;  // grad_dev128 != NULL: grad_host is complex128
    double scale, lam;
    const void* pack;  // != NULL (a BallPack): v_host / grad_host are packed balls, one contiguous copy per slab
    const void *slab_flags, *one_dev;  // != NULL: after slab g's gradient copy, *one_dev -> slab_flags[g] (pinned int)
    bool operator==(const HostStepKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};

// Enqueue one slab-pipelined host step on s (also used under stream capture).
cudaError_t host_step_enqueue(const HostStepKey& k, HostPipe* P, const int32_t* idx_host, cudaStream_t s) {
    const int M = k.M, n_mask = k.n_mask, B = k.B, n_slabs = k.n_slabs;
    const double scale = k.scale, lam = k.lam;
    const fsld_image_rec* recs = reinterpret_cast<const fsld_image_rec*>(k.recs);
    void* scratch = const_cast<void*>(k.scratch);
    void* v_dev = const_cast<void*>(k.v_dev);
    void* grad_dev = const_cast<void*>(k.grad_dev);
    int32_t* idx_dev = reinterpret_cast<int32_t*>(const_cast<void*>(k.idx_dev));
    const void* v_host = k.v_host;
    void* grad_host = const_cast<void*>(k.grad_host);
    double* out_host = reinterpret_cast<double*>(const_cast<void*>(k.out_host));
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    char* scr = reinterpret_cast<char*>(scratch);
    SortedArgs a = make_sorted(L, M, n_mask, B, recs, idx_dev, v_dev, k.xs, reinterpret_cast<const int8_t*>(k.pc),
                               reinterpret_cast<const int32_t*>(k.seg_off), reinterpret_cast<const int32_t*>(k.segs),
                               grad_dev, scratch, k.ptab);
    a.out_scale = (float)scale;
    const int c = (M + 1) / 2, nb = L.nb;
    int first[kMaxSlabs + 1];
    const int G = slab_layers(nb, n_slabs, first);
    SlabMap map{};
    for (int g = 0; g < G; ++g)
        for (int l = first[g]; l < first[g + 1]; ++l) map.of_layer[l] = (unsigned char)g;
    const size_t plane = (size_t)M * M * sizeof(float2);
    int4* gitems = reinterpret_cast<int4*>(scr + L.gitems);
    int* gctl = reinterpret_cast<int*>(scr + L.gctl);
    double* gpart = reinterpret_cast<double*>(scr + L.gpart);
    double* npart = reinterpret_cast<double*>(scr + L.npart);
    double* hout = reinterpret_cast<double*>(scr + L.hout);
    const char* vh = reinterpret_cast<const char*>(v_host);
    char* gh = reinterpret_cast<char*>(grad_host);
    char* vd = reinterpret_cast<char*>(v_dev);
    char* gd = reinterpret_cast<char*>(grad_dev);

    cudaError_t e = cudaSuccess;
    const BallPack* bp = reinterpret_cast<const BallPack*>(k.pack);
#define FSLD_TRY(x) do { if ((e = (x)) != cudaSuccess) return e; } while (0)
    // the slab passes' per-CTA partials live in kSlabCtas-sized slots: refuse an oversized grid
    // before anything is enqueued (nothing half-written)
    int grid_max = 0;
    FSLD_TRY(prepare_host_step(&grid_max));
    if (grid_max > kSlabCtas) return cudaErrorInvalidConfiguration;
    // batch rows first (2 KB: the binning must not queue behind a volume slab on the copy engine)
    FSLD_TRY(cudaMemcpyAsync(idx_dev, idx_host, sizeof(int32_t) * (size_t)B, cudaMemcpyHostToDevice, s));
    // (A/B) FSLD_HOST_BIN_FIRST=1: the binning ahead of the fork, so that the first pass never waits for
    // it -- measured slower (1.07 vs 0.95 ms per numpy call: the copies then start ~70 us later)
    static const bool bin_first = [] {
        const char* v = std::getenv("FSLD_HOST_BIN_FIRST");
        return v && v[0] == '1';
    }();
    auto binning = [&]() -> cudaError_t {  // per-step binning, regrouped by slab (independent of v)
        cudaError_t r = cudaMemsetAsync(gpart, 0, L.hout - L.gpart, s);
        if (r == cudaSuccess) r = launch_sorted_bin(a, s);
        if (r == cudaSuccess) r = launch_slab_items(a, map, G, gitems, gctl, s);
        return r;
    };
    if (bin_first) FSLD_TRY(binning());
    // fork: the copy streams start after whatever `stream` already holds (v_dev / grad_dev reuse)
    FSLD_TRY(cudaEventRecord(P->fork, s));
    FSLD_TRY(cudaStreamWaitEvent(P->h2d, P->fork, 0));
    FSLD_TRY(cudaStreamWaitEvent(P->d2h, P->fork, 0));
    int zi0[kMaxSlabs][2], nz[kMaxSlabs][2], np[kMaxSlabs];
    for (int g = 0; g < G; ++g) {
        const int z0 = -c + BT * first[g], z1 = std::min(-c + BT * first[g + 1], M - c);
        np[g] = slab_pieces(M, z0, z1, zi0[g], nz[g]);
        if (bp) {  // the slab's part of the packed ball in one copy (init() puts its rows into place)
            const size_t o = (size_t)bp->off[g] * sizeof(float2), nbytes = (size_t)(bp->off[g + 1] - bp->off[g]) * sizeof(float2);
            if (nbytes)
                FSLD_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(bp->vpack_dev) + o, vh + o, nbytes,
                                         cudaMemcpyHostToDevice, P->h2d));
        } else {
            for (int q = 0; q < np[g]; ++q)
                FSLD_TRY(cudaMemcpyAsync(vd + zi0[g][q] * plane, vh + zi0[g][q] * plane, nz[g][q] * plane,
                                         cudaMemcpyHostToDevice, P->h2d));
        }
        FSLD_TRY(cudaEventRecord(P->eh[g], P->h2d));
    }
    if (!bin_first) FSLD_TRY(binning());
    auto init = [&](int g) -> cudaError_t {  // grad = lam v on slab g (+ ||v||^2 partials), on `stream`
        cudaError_t r = cudaStreamWaitEvent(s, P->eh[g], 0);
        if (bp && r == cudaSuccess)  // (not on the copy stream: its copies run back to back)
            r = launch_ball_rows(false, bp->rows_dev + bp->row0[g], bp->row0[g + 1] - bp->row0[g], bp->vpack_dev, v_dev, s);
        for (int q = 0; q < np[g] && r == cudaSuccess; ++q) {
            const size_t o = (size_t)zi0[g][q] * M * M;
            r = launch_grad_init((int64_t)nz[g][q] * M * M, reinterpret_cast<const float2*>(v_dev) + o, lam,
                                 reinterpret_cast<float2*>(grad_dev) + o, npart + (2 * g + q) * kInitParts,
                                 kInitParts, s);
        }
        return r == cudaSuccess ? cudaEventRecord(P->ei[g], s) : r;
    };
    // Slab g's bricks read v up to the first plane of slab g + 1 and flush into it, so pass g
    // starts after slab g + 1 is copied and initialised.  Passes of neighbouring slabs only meet
    // in red.global adds, so they run concurrently (two kernel streams: one pass's tail overlaps
    // the next one's start).  Slab g's gradient is final once passes g - 1 and g are done.
    a.items = gitems;
    for (int g = 0; g < G; ++g) FSLD_TRY(init(g));
    for (int g = 0; g < G; ++g) {
        cudaStream_t ks = P->ks[g & 1];
        FSLD_TRY(cudaStreamWaitEvent(ks, P->ei[g + 1 < G ? g + 1 : g], 0));
        a.ctl = gctl + 16 * g;
        a.part = gpart + (size_t)g * kSlabCtas;
        int grid = 0;
        FSLD_TRY(launch_sorted_pass(a, ks, &grid));
        FSLD_TRY(cudaEventRecord(P->ek[g], ks));
        if (bp) {  // the slab's rows packed on the pass's stream, then one copy
            const size_t o = (size_t)bp->off[g] * sizeof(float2), nbytes = (size_t)(bp->off[g + 1] - bp->off[g]) * sizeof(float2);
            if (g > 0) FSLD_TRY(cudaStreamWaitEvent(ks, P->ek[g - 1], 0));
            FSLD_TRY(launch_ball_rows(true, bp->rows_dev + bp->row0[g], bp->row0[g + 1] - bp->row0[g], grad_dev,
                                      bp->gpack_dev, ks));
            FSLD_TRY(cudaEventRecord(P->ep[g], ks));
            FSLD_TRY(cudaStreamWaitEvent(P->d2h, P->ep[g], 0));
            if (nbytes)
                FSLD_TRY(cudaMemcpyAsync(gh + o, reinterpret_cast<char*>(bp->gpack_dev) + o, nbytes,
                                         cudaMemcpyDeviceToHost, P->d2h));
        }
        if (!bp) {
            FSLD_TRY(cudaStreamWaitEvent(P->d2h, P->ek[g], 0));
            if (g > 0) FSLD_TRY(cudaStreamWaitEvent(P->d2h, P->ek[g - 1], 0));
        }
        for (int q = 0; q < (bp ? 0 : np[g]); ++q) {
            if (k.grad_dev128) {  // complex128 out: cast the finished slab on the device, copy 16 B / voxel
                char* g128 = reinterpret_cast<char*>(const_cast<void*>(k.grad_dev128));
                FSLD_TRY(launch_cast_c64_c128((int64_t)nz[g][q] * M * M, gd + zi0[g][q] * plane,
                                              g128 + 2 * zi0[g][q] * plane, P->d2h));
                FSLD_TRY(cudaMemcpyAsync(gh + 2 * zi0[g][q] * plane, g128 + 2 * zi0[g][q] * plane,
                                         2 * nz[g][q] * plane, cudaMemcpyDeviceToHost, P->d2h));
            } else {
                FSLD_TRY(cudaMemcpyAsync(gh + zi0[g][q] * plane, gd + zi0[g][q] * plane, nz[g][q] * plane,
                                         cudaMemcpyDeviceToHost, P->d2h));
            }
        }
        if (k.slab_flags)  // (posted writes keep their order: the flag lands after the slab's data)
            FSLD_TRY(cudaMemcpyAsync(reinterpret_cast<int*>(const_cast<void*>(k.slab_flags)) + g, k.one_dev, sizeof(int),
                                     cudaMemcpyDeviceToHost, P->d2h));
    }
    for (int q = 0; q < 2 && q < G; ++q) FSLD_TRY(cudaStreamWaitEvent(s, P->ek[G - 1 - q], 0));
    FSLD_TRY(cudaEventRecord(P->join, P->d2h));
    FSLD_TRY(launch_loss_finalize(gpart, G * kSlabCtas, npart, G * 2 * kInitParts, scale, lam, hout, hout + 1, s));
    FSLD_TRY(cudaMemcpyAsync(out_host, hout, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FSLD_TRY(cudaStreamWaitEvent(s, P->join, 0));
#undef FSLD_TRY
    return cudaSuccess;
}

struct HostGraph {
    HostStepKey key{};
    int dev = -1;
    cudaGraphExec_t exec = nullptr;
    int32_t* idx_pinned = nullptr;  // the graph's source of the batch rows
    cudaEvent_t done = nullptr;     // after the last replay: idx_pinned may be rewritten
    unsigned long long used = 0;
};
HostGraph g_graphs[8];
unsigned long long g_graph_clock = 0;

void drop_graph(HostGraph& h) {
    if (h.done) cudaEventSynchronize(h.done), cudaEventDestroy(h.done);
    if (h.exec) cudaGraphExecDestroy(h.exec);
    if (h.idx_pinned) cudaFreeHost(h.idx_pinned);
    h = HostGraph{};
}

// The cached graph for (device, key), captured on first use (LRU over 8 entries).
cudaError_t host_graph(const HostStepKey& k, HostPipe* P, HostGraph*& out) {
    cudaStream_t s = P->cap;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    HostGraph* lru = &g_graphs[0];
    for (HostGraph& h : g_graphs) {
        if (h.exec && h.dev == dev && h.key == k) {
            h.used = ++g_graph_clock;
            out = &h;
            return cudaSuccess;
        }
        if (h.used < lru->used) lru = &h;
    }
    drop_graph(*lru);
    HostGraph& h = *lru;
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&h.idx_pinned), sizeof(int32_t) * (size_t)k.B,
                           cudaHostAllocDefault)) != cudaSuccess) {
        h = HostGraph{};
        return e;
    }
    if ((e = cudaEventCreateWithFlags(&h.done, cudaEventDisableTiming)) != cudaSuccess) {
        drop_graph(h);
        return e;
    }
    cudaGraph_t g = nullptr;
    e = prepare_host_step(nullptr);  // lazily initialised launch state (attributes, grid sizes): not under capture
    if (e == cudaSuccess) e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        const cudaError_t e1 = host_step_enqueue(k, P, h.idx_pinned, s);
        e = cudaStreamEndCapture(s, &g);
        if (e1 != cudaSuccess) e = e1;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&h.exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        cudaGetLastError();
        drop_graph(h);
        return e;
    }
    h.key = k;
    h.dev = dev;
    h.used = ++g_graph_clock;
    out = &h;
    return cudaSuccess;
}

// Every cached graph whose copies read or write host buffer p (its memcpy nodes hold the address
// as it was when captured): dropped before p is freed, and on fsld_host_step_reset().
void drop_host_graphs_using(const void* p) {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    for (HostGraph& h : g_graphs)
        if (h.exec && (!p || h.key.v_host == p || h.key.grad_host == p || h.key.out_host == p || h.key.slab_flags == p || h.key.pack == p)) drop_graph(h);
}

}  // namespace

extern "C" int fsld_host_step_reset(void) {
    drop_host_graphs_using(nullptr);
    return FSLD_OK;
}

static int loss_grad_host_impl(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host,
                               int B, const void* v_host, const void* xs, const int8_t* pc, const void* ptab,
                               const int32_t* seg_off, const int32_t* segs, double scale, double lam,
                               void* grad_host, double* out_host, void* v_dev, void* grad_dev, int32_t* idx_dev,
                               int n_slabs, void* scratch, size_t scratch_bytes, void* stream, void* grad_dev128,
                               const BallPack* pack = nullptr, int* slab_flags = nullptr,
                               const int* one_dev = nullptr) {
    if (!geom_ok(M, mode, n_mask, B) || M > 256 || mode != FSLD_MODE_TRI) return FSLD_EINVAL;
    if ((slab_flags != nullptr) != (one_dev != nullptr) || (pack && (grad_dev128 || pack->M != M || pack->n_slabs != n_slabs)))
        return FSLD_EINVAL;
    if (!recs || !idx_host || !v_host || !xs || !pc || !seg_off || !segs || !grad_host || !out_host || !v_dev ||
        !grad_dev || !idx_dev || !scratch || v_dev == grad_dev || n_slabs < 1 || n_slabs > kMaxSlabs)
        return FSLD_EINVAL;
    const ScratchLayout L = scratch_layout(M, n_mask, B);
    if (scratch_bytes < L.total) return FSLD_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    HostStepKey k;
    std::memset(&k, 0, sizeof(k));  // padding bytes take part in the key comparison
    k.M = M;
    k.n_mask = n_mask;
    k.B = B;
    k.n_slabs = n_slabs;
    k.recs = recs;
    k.v_host = v_host;
    k.xs = xs;
    k.pc = pc;
    k.ptab = ptab;
    k.seg_off = seg_off;
    k.segs = segs;
    k.grad_host = grad_host;
    k.out_host = out_host;
    k.v_dev = v_dev;
    k.grad_dev = grad_dev;
    k.grad_dev128 = grad_dev128;
    k.idx_dev = idx_dev;
    k.scratch = scratch;
    k.scale = scale;
    k.lam = lam;
    k.pack = pack;
    k.slab_flags = slab_flags;
    k.one_dev = one_dev;
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    HostPipe* P = nullptr;
    cudaError_t e = pipe_for_device(P);
    if (e != cudaSuccess) return status_of(e);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(s, &cs)) != cudaSuccess) return status_of(e);
    static const bool no_graph = [] {  // FSLD_HOST_GRAPH=0: enqueue every call (A/B of the graph replay)
        const char* v = std::getenv("FSLD_HOST_GRAPH");
        return v && v[0] == '0';
    }();
    if (cs != cudaStreamCaptureStatusNone || no_graph)  // the caller's own capture, or no replay
        return status_of(host_step_enqueue(k, P, idx_host, s));
    HostGraph* h = nullptr;
    if ((e = host_graph(k, P, h)) != cudaSuccess) return status_of(e);
    if ((e = cudaEventSynchronize(h->done)) != cudaSuccess) return status_of(e);  // previous replay read its rows
    std::memcpy(h->idx_pinned, idx_host, sizeof(int32_t) * (size_t)B);
    if ((e = cudaGraphLaunch(h->exec, s)) != cudaSuccess) return status_of(e);
    note_bins(scratch, idx_dev, recs, M, n_mask, B);
    return status_of(cudaEventRecord(h->done, s));
}

extern "C" int fsld_loss_grad_host(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host,
                                   int B, const void* v_host, const void* xs, const int8_t* pc, const void* ptab,
                                   const int32_t* seg_off, const int32_t* segs, double scale, double lam,
                                   void* grad_host, double* out_host, void* v_dev, void* grad_dev, int32_t* idx_dev,
                                   int n_slabs, void* scratch, size_t scratch_bytes, void* stream) {
    return loss_grad_host_impl(M, mode, n_mask, recs, idx_host, B, v_host, xs, pc, ptab, seg_off, segs, scale, lam,
                               grad_host, out_host, v_dev, grad_dev, idx_dev, n_slabs, scratch, scratch_bytes, stream,
                               nullptr);
}

extern "C" int fsld_loss_grad_host_c128(int M, int mode, int n_mask, const fsld_image_rec* recs,
                                        const int32_t* idx_host, int B, const void* v_host, const void* xs,
                                        const int8_t* pc, const void* ptab, const int32_t* seg_off,
                                        const int32_t* segs, double scale, double lam, void* grad_host_c128,
                                        double* out_host, void* v_dev, void* grad_dev, void* grad_dev128,
                                        int32_t* idx_dev, int n_slabs, void* scratch, size_t scratch_bytes,
                                        void* stream) {
    if (!grad_dev128 || grad_dev128 == v_dev || grad_dev128 == grad_dev) return FSLD_EINVAL;
    return loss_grad_host_impl(M, mode, n_mask, recs, idx_host, B, v_host, xs, pc, ptab, seg_off, segs, scale, lam,
                               grad_host_c128, out_host, v_dev, grad_dev, idx_dev, n_slabs, scratch, scratch_bytes,
                               stream, grad_dev128);
}

// ---------------------------------------------------------------- numpy-signature host step
namespace {
struct NpStage {  // per device: page-locked complex64 staging of v and of the gradient, device complex128 staging
    int64_t n = 0;
    float2 *v64 = nullptr, *g64 = nullptr;
    double2* g128_dev = nullptr;
    int* flags = nullptr;    // page-locked: slab g's gradient has landed in g64 (touched-ball step)
    int* one_dev = nullptr;  // device constant 1, the source of the flag copies
    BallPack bp;             // the touched ball's rows and packed order (rebuilt when M / slabs / radius change)
};
NpStage g_np[16];
std::mutex g_np_mu;  // one numpy-signature call at a time (the staging is per device)

cudaError_t np_stage(int64_t n, NpStage*& out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
    NpStage& st = g_np[dev];
    if (st.n != n) {
        if (st.v64) {
            drop_host_graphs_using(st.v64);
            drop_host_graphs_using(st.g64);
            drop_host_graphs_using(st.flags);
            drop_host_graphs_using(&st.bp);
            ball_pack_free(st.bp);
            cudaFreeHost(st.v64);
            cudaFreeHost(st.g64);
            cudaFreeHost(st.flags);
            cudaFree(st.g128_dev);
            cudaFree(st.one_dev);
        }
        st = NpStage{};
        if ((e = cudaHostAlloc(reinterpret_cast<void**>(&st.v64), sizeof(float2) * (size_t)n, cudaHostAllocDefault)) !=
                cudaSuccess ||
            (e = cudaHostAlloc(reinterpret_cast<void**>(&st.g64), sizeof(float2) * (size_t)n, cudaHostAllocDefault)) !=
                cudaSuccess ||
            (e = cudaMalloc(reinterpret_cast<void**>(&st.g128_dev), sizeof(double2) * (size_t)n)) != cudaSuccess ||
            (e = cudaHostAlloc(reinterpret_cast<void**>(&st.flags), sizeof(int) * kMaxSlabs, cudaHostAllocDefault)) !=
                cudaSuccess ||
            (e = cudaMalloc(reinterpret_cast<void**>(&st.one_dev), sizeof(int))) != cudaSuccess)
            return e;
        const int one = 1;
        if ((e = cudaMemcpy(st.one_dev, &one, sizeof(int), cudaMemcpyHostToDevice)) != cudaSuccess) return e;
        st.n = n;
    }
    out = &st;
    return cudaSuccess;
}

// complex128 <-> complex64 over n complex elements on the library's host thread pool (streaming stores)
void np_cast(const double* src, float* dst, int64_t n) {
    fsld_host::parallel_for(n, 1 << 15, [&](int64_t i0, int64_t i1) {
        fsld_host_cast_f64_to_f32(src + 2 * i0, dst + 2 * i0, 2 * (i1 - i0));
    });
}
void np_cast_back(const float* src, double* dst, int64_t n) {
    fsld_host::parallel_for(n, 1 << 15, [&](int64_t i0, int64_t i1) {
        fsld_host_cast_f32_to_f64(src + 2 * i0, dst + 2 * i0, 2 * (i1 - i0));
    });
}
}  // namespace

// Measured on the B200 box (cfg3, tools/e2e_split.py): the call is bound by host memory traffic (the
// complex128 volume read and the complex128 gradient written are ~67 MB, the complex64 staging another
// ~34 MB); overlapping the slab casts with the copies (device waits on host-written flags) made every
// phase slower through that contention (1.31 vs 1.22 ms), so the cast runs first, on all host cores.
//
// touch_radius > 0: the data term only reaches voxels within that radius of the origin
// (grid.touched_ball: max |k| of the mask + sqrt(3)); off that ball the gradient is lam v and the loss
// only sees ||v||^2 -- both computed here on the host threads in fp64 while the device works.  Only
// the ball crosses PCIe, packed row by row (BallPack: ~58 % of the cube at M=128), one contiguous
// complex64 range per z-slab in each direction: the cast in writes the packed staging, a row kernel puts
// each slab's rows into the device volume; each finished gradient slab is packed on the device, copied,
// flagged, and cast to complex128 into the result by the host threads while later slabs are in flight
// (measured on the B200 box: the copy engine reads host memory at ~30 GB/s, so the call is bound by the
// bytes of the volume going up; whole planes 1.30 ms, (y, x) boxes per slab 1.02 ms, the packed ball see
// DESIGN section 6).
extern "C" int fsld_loss_grad_host_np_ball(int M, int mode, int n_mask, const fsld_image_rec* recs,
                                           const int32_t* idx_host, int B, const double* v128_host, const void* xs,
                                           const int8_t* pc, const void* ptab, const int32_t* seg_off,
                                           const int32_t* segs, double scale, double lam, double* grad128_host,
                                           double* out_host, void* v_dev, void* grad_dev, int32_t* idx_dev,
                                           int n_slabs, void* scratch, size_t scratch_bytes, void* stream,
                                           double touch_radius) {
    if (!v128_host || !grad128_host || !out_host || M < 2 || M > 256 || n_slabs < 1 || n_slabs > kMaxSlabs)
        return FSLD_EINVAL;
    if ((reinterpret_cast<uintptr_t>(v128_host) | reinterpret_cast<uintptr_t>(grad128_host)) & 15) return FSLD_EINVAL;
    const int64_t n = (int64_t)M * M * M;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_np_mu);
    NpStage* st = nullptr;
    cudaError_t e = np_stage(n, st);
    if (e != cudaSuccess) return status_of(e);
    // a page-locked output array is written by the copy engine (the device casts each finished slab to
    // complex128); any other memory gets the complex64 gradient cast back by the host threads
    cudaPointerAttributes pa{};
    const bool out_pinned = cudaPointerGetAttributes(&pa, grad128_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const bool ball = touch_radius > 0.0 && std::isfinite(touch_radius);
    if (!ball) {
        np_cast(v128_host, reinterpret_cast<float*>(st->v64), n);
        const int rc = loss_grad_host_impl(M, mode, n_mask, recs, idx_host, B, st->v64, xs, pc, ptab, seg_off, segs,
                                           scale, lam, out_pinned ? static_cast<void*>(grad128_host) : st->g64,
                                           out_host, v_dev, grad_dev, idx_dev, n_slabs, scratch, scratch_bytes,
                                           stream, out_pinned ? static_cast<void*>(st->g128_dev) : nullptr);
        if (rc != FSLD_OK) return rc;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return status_of(e);
        if (!out_pinned) np_cast_back(reinterpret_cast<const float*>(st->g64), grad128_host, n);
        return FSLD_OK;
    }
    BallPack& bp = st->bp;
    if (bp.M != M || bp.n_slabs != n_slabs || bp.rt != touch_radius) {
        drop_host_graphs_using(&bp);
        if ((e = ball_pack_build(bp, M, n_slabs, touch_radius)) != cudaSuccess) return status_of(e);
    }
    static const bool trace = std::getenv("FSLD_NP_TRACE") != nullptr;  // (per-phase host times on stderr)
    auto now = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t0 = trace ? now() : 0.0;
    double in_sq[256], out_sq[256];  // per-plane sums of |v|^2 on / off the ball (fixed order)
    float* v64 = reinterpret_cast<float*>(st->v64);
    fsld_host::parallel_for(M, 1, [&](int64_t za, int64_t zb) {
        for (int64_t z = za; z < zb; ++z) {
            double t = 0.0;
            for (int64_t r = z * M; r < (z + 1) * M; ++r)
                if (bp.xb[r] > bp.xa[r])
                    t += fsld_host::cast_f64_to_f32_sumsq(v128_host + 2 * (r * M + bp.xa[r]), v64 + 2 * bp.poff[r],
                                                          2 * (int64_t)(bp.xb[r] - bp.xa[r]));
            in_sq[z] = t;
        }
        fsld_host::store_fence();
    });
    const double t1 = trace ? now() : 0.0;
    volatile int* flags = st->flags;
    for (int g = 0; g < kMaxSlabs; ++g) flags[g] = 0;
    // the packed complex64 gradient into the page-locked staging slab by slab, one flag per finished slab
    const int rc = loss_grad_host_impl(M, mode, n_mask, recs, idx_host, B, st->v64, xs, pc, ptab, seg_off, segs, scale,
                                       lam, st->g64, out_host, v_dev, grad_dev, idx_dev, n_slabs, scratch,
                                       scratch_bytes, stream, nullptr, &bp, st->flags, st->one_dev);
    if (rc != FSLD_OK) return rc;
    const double t2 = trace ? now() : 0.0;
    // while the device works: grad = lam v off the ball (running it after the last slab instead measured
    // 0.98-1.03 vs 0.92 ms per call)
    auto fill_outside = [&] {
    fsld_host::parallel_for(M, 1, [&](int64_t za, int64_t zb) {
        for (int64_t z = za; z < zb; ++z) {
            double t = 0.0;
            for (int64_t r = z * M; r < (z + 1) * M; ++r) {  // (a row off the ball: xa = xb = 0)
                const int64_t o = 2 * r * M, xa = bp.xa[r], xb = bp.xb[r];
                t += fsld_host::scale_f64_sumsq(v128_host + o, grad128_host + o, 2 * xa, lam);
                t += fsld_host::scale_f64_sumsq(v128_host + o + 2 * xb, grad128_host + o + 2 * xb, 2 * (M - xb), lam);
            }
            out_sq[z] = t;
        }
        fsld_host::store_fence();
    });
    };
    fill_outside();
    const double t3 = trace ? now() : 0.0;
    // each finished slab: its rows cast to complex128 into the result while the later slabs are in flight
    const float* g64 = reinterpret_cast<const float*>(st->g64);
    for (int g = 0; g < bp.G; ++g) {
        for (unsigned spin = 0; flags[g] == 0; ++spin) {
            fsld_host::cpu_pause();
            if ((spin & 0xfff) == 0xfff) {  // a failed or finished stream never sets the flag: do not spin on it
                const cudaError_t q = cudaStreamQuery(s);
                if (q != cudaErrorNotReady) {
                    if (q != cudaSuccess) return status_of(q);
                    if (flags[g] == 0) return FSLD_ECUDA;
                }
            }
        }
        for (int q = 0; q < bp.snp[g]; ++q) {
            const int za = bp.sz[g][q];
            fsld_host::parallel_for(bp.sn[g][q], 1, [&](int64_t ia, int64_t ib) {
                for (int64_t r = (za + ia) * M; r < (za + ib) * M; ++r)
                    if (bp.xb[r] > bp.xa[r])
                        fsld_host_cast_f32_to_f64(g64 + 2 * bp.poff[r], grad128_host + 2 * (r * M + bp.xa[r]),
                                                  2 * (int64_t)(bp.xb[r] - bp.xa[r]));
            });
        }
    }
    const double t4 = trace ? now() : 0.0;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return status_of(e);
    if (trace)
        std::fprintf(stderr, "np_ball: cast %.3f launch %.3f fill %.3f slabs %.3f wait %.3f ms\n", t1 - t0, t2 - t1,
                     t3 - t2, t4 - t3, now() - t4);
    // the device's loss used the norm of its own (partly stale) copy of v: ||v||^2 from the host sums
    double norm = 0.0;
    for (int z = 0; z < M; ++z) norm += in_sq[z] + out_sq[z];
    out_host[1] = 0.5 * scale * out_host[0] + 0.5 * lam * norm;
    return FSLD_OK;
}

extern "C" int64_t fsld_ball_voxels(int M, double touch_radius) {
    if (M < 2 || M > 256 || !(touch_radius > 0.0) || !std::isfinite(touch_radius)) return (int64_t)M * M * M;
    const int c = (M + 1) / 2;
    int64_t n = 0;
    for (int kz = -c; kz < M - c; ++kz)
        for (int ky = -c; ky < M - c; ++ky) {
            int xa = 0, xb = 0;
            if (ball_row(M, kz, ky, touch_radius, xa, xb)) n += xb - xa;
        }
    return n;
}

extern "C" int fsld_loss_grad_host_np(int M, int mode, int n_mask, const fsld_image_rec* recs, const int32_t* idx_host,
                                      int B, const double* v128_host, const void* xs, const int8_t* pc,
                                      const void* ptab, const int32_t* seg_off, const int32_t* segs, double scale,
                                      double lam, double* grad128_host, double* out_host, void* v_dev,
                                      void* grad_dev, int32_t* idx_dev, int n_slabs, void* scratch,
                                      size_t scratch_bytes, void* stream) {
    return fsld_loss_grad_host_np_ball(M, mode, n_mask, recs, idx_host, B, v128_host, xs, pc, ptab, seg_off, segs,
                                       scale, lam, grad128_host, out_host, v_dev, grad_dev, idx_dev, n_slabs, scratch,
                                       scratch_bytes, stream, 0.0);
}
