// plan.cu — HBM-resident plans, the CUDA-graph time loop and the C ABI
// (include/sf_b200.h) that replaces the reference's JIT'd Operator() entry.
//
// Reference call path being replaced:
//   Operator::apply (op.cpp:126-161) -> CompiledKernel::invoke (jit.cpp:104-148)
//   -> generated Operator(u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w):
//        for t: aliases (K6) -> stencil (K2/K3) -> inject (K4) -> sample (K5)
// Here: plan create = build time (constants folded, buffers allocated in HBM),
// apply = H2D, nt steps replayed from a cached CUDA graph, D2H.
//
// Layout of this file:
//   plan state (sf_plan, PointSet)          host <-> HBM transfers, point CSR
//   kernel tables + launchers               per-thread-load / scalar TMA /
//                                           vector ring / queue-vector / 2D /
//                                           diffusion; tensor maps; PDL
//   launch_stencil / sparse launches        incl. the fused sparse epilogue
//   NCCL (dlopen'd) halo exchange           slab steps, in-process chain
//   step enqueue: acoustic, diffusion (temporal blocking), FWI forward/adjoint
//   tile-sorted injection CSR, graphs       build_fused, ensure_fused, run_steps
//   geometry                                chunk_grid, set_grid, enable_tma
//   plan construction, upload / download    setup_acoustic, upload_any, ...
//   autotune, SFG1 + text I/O, self-test    then the extern "C" entry points
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sf_b200.h"
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler injects NVTX

#include "kernels.cuh"
#include "tma_stencil.cuh"
#include "vec_stencil.cuh"
#include "diffusion_tb.cuh"
#include "sf_internal.h"
#include "medium.h"

namespace sfb {

// NVTX range over a phase of a C-ABI call (upload / time loop / download /
// FWI sweeps / autotune / slab chain); shows up in Nsight Systems timelines.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {
thread_local std::string g_error;

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SF_CUDA(expr)                                                                    \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw Status(e_ == cudaErrorMemoryAllocation ? SF_ERR_OOM : SF_ERR_CUDA,     \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));            \
    } while (0)

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    SF_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}

void dfree(void* p) {
    if (p) cudaFree(p);
}

} // namespace

void set_error(const std::string& msg) { g_error = msg; }

// One sparse point set ("src" or "rec") on the device, plus the injection CSR
// when the set injects.
struct PointSet {
    int64_t np = 0;
    int64_t nt = 0;
    float* series = nullptr;  // [nt][np]
    int* ci = nullptr;        // [np][ndim]
    float* w = nullptr;       // [np][2^ndim]
    // injection CSR over distinct target cells
    int ncells = 0;
    int nband0 = 0;  // slabs: the first nband0 cells lie in the boundary bands
    int64_t* cell_off = nullptr;
    int* start = nullptr;
    int* cp = nullptr;
    float* cw = nullptr;
    std::vector<int32_t> host_ci;  // last uploaded indices (validated)
    // host copy of the device CSR (change detection: a re-upload of the same
    // points leaves the device buffers, and the graphs that use them, alone)
    std::vector<int64_t> h_cells;
    std::vector<int> h_start, h_cp;
    std::vector<float> h_cw;
    size_t cap_cells = 0, cap_contrib = 0;
    uint64_t version = 0;  // bumped whenever the device CSR changes
};

} // namespace sfb

// rows-per-lane selector of the 16-warp radius-4 ring kernel with the a0
// register queue (one row per lane)
constexpr int kRplAq = 17;
constexpr int kRplAq2 = 18;  // the same, two planes per pass (SF_VEC_AQ2=1; A/B)

struct sf_plan {
    enum Kind { ACOUSTIC, DIFFUSION, FWI } kind;
    int device = 0;
    cudaStream_t stream = nullptr;
    int ndim = 3;
    int64_t n[3] = {1, 1, 1};
    int64_t pitch = 0, plane = 0, slot_elems = 0;
    int64_t nt = 0;
    int nslots = 3;
    sfb::AcousticConstants ac{};       // constants the launchers use
    sfb::AcousticConstants ac_fwd{}, ac_adj{};  // FWI: both directions
    sfb::DiffusionConstants dc{};
    // device mirrors
    float* slot[3] = {nullptr, nullptr, nullptr};
    float* staging = nullptr;  // dense copy of one field for host transfers
    float* dscratch[2] = {nullptr, nullptr};  // diffusion: second buffer pair (temporal blocking)
    bool diffusion_tb = true;
    int tb_tile = 64;  // temporal-blocking core tile (radius 1 only: 48 .. 96)
    int tb_rv = 2;     // rows per thread visit (radius 1, 64-wide tiles: 2 measured +2 %)
    CUtensorMap tm_dx[2], tm_dy[2];  // diffusion: 2D maps over slots / scratch (box SW x SW)
    float* m = nullptr;
    float* eta = nullptr;
    sfb::PointSet src, rec;
    // FWI
    float* hist = nullptr;  // (nt+2) levels
    float* grad = nullptr;
    float* v[3] = {nullptr, nullptr, nullptr};
    // launch geometry
    dim3 grid3;
    int zchunk = 0;
    int z0 = 0, z1 = 0;  // axis-0 planes the stencil updates (local coordinates)
    int tile_nx = 1, tile_ty = 8;  // 3D stencil tile: (32*tile_nx) x tile_ty
    int resident = 0;              // CTAs per SM of the chosen stencil kernel
    // TMA pipeline path (3D forward/adjoint without the FWI gradient)
    bool use_tma = false;
    bool use_vec = false;  // 4 points/thread, LDS.128 variant of the TMA pipeline
    bool use_vecq = false; // ... with the a0 neighbours in a register queue (radius >= 5)
    int vecq_ring = 0;  // ... form: 0 by radius, 1 future a0 planes from a shared-memory core ring
                        // (vecq2), 2 compiler-scheduled addressing, 3 pinned loop state
    int vec_warps = 8;
    int vec_rpl = 1;  // vector kernel: rows of four points per lane (1 or 2)
    bool vec_aq = true;  // 16-warp radius-4 ring kernel with the a0 register queue (SF_VEC_AQ=0: ring loads)
    // kernel selector: kRplAq picks the a0-queue instance (geometry as rpl = 1)
    int vec_kernel_rpl() const {
        const bool shape_ok = vec_rpl == 1 && tile_nx == 2 && ac.radius == 4;
        if (shape_ok && vec_aq && vec_aq2 && vec_warps == 16) return kRplAq2;
        return shape_ok && ((vec_aq && vec_warps == 16) || (vec_aq8 && vec_warps == 8)) ? kRplAq : vec_rpl;
    }
    bool vec_aq2 = false;
    bool vec_aq8 = false;  // the same for the 8-warp 64 x 16 tiles (SF_VEC_AQ8=1; A/B)
    int tma_stages = 4;
    int stages_override = 0;  // autotune: > 0 forces the pipeline depth
    size_t tma_smem = 0;
    CUtensorMap tm_cur[3], tm_pme[3], tm_m, tm_eta;
    // FWI: history (nt+2 levels), adjoint slots v, gradient
    CUtensorMap tm_hist_cur, tm_hist_pme, tm_v_cur[3], tm_v_pme[3], tm_grad;
    // the gradient kernel's own 64 x 8 boxes when the forward runs 8-warp tiles
    CUtensorMap tm_m_g, tm_eta_g, tm_hist_pme_g, tm_v_cur_g[3], tm_v_pme_g[3];
    dim3 grid_grad;          // GRAD launches use 4-warp CTAs (6 boxes per stage)
    int zchunk_grad = 0;
    size_t smem_grad = 0;
    int tma_stages_grad = 4;
    std::map<std::pair<int64_t, int64_t>, cudaGraphExec_t> graphs;
    std::vector<std::string> arg_names;
    std::vector<int64_t> arg_bytes;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // sf_plan_invoke with the upload overlapped by the first time steps
    // (invoke_overlapped): the copy stream and one event per plane chunk
    cudaStream_t io = nullptr;
    std::vector<cudaEvent_t> ev_up;
    int64_t launches_per_step = 0;
    // depth-slab decomposition; a whole grid is one slab
    bool slab = false;
    int64_t global_n0 = 0, plane0 = 0, own_begin = 0, own_end = 0;
    int own_lo = 0, own_hi = 0;  // owned planes in local coordinates
    bool has_lower = false, has_upper = false;
    // NCCL transport (one process per GPU)
    void* nccl_comm = nullptr;
    int nccl_rank = -1, nccl_nranks = 0;
    cudaEvent_t ev_copy = nullptr;  // in-process chain: halo copies issued
    // overlap of the halo exchange with the inner planes (slabs, owned >= 2r)
    struct ZRange {
        int z0 = 0, z1 = 0;
        dim3 grid;
        int zchunk = 0;
    };
    bool overlap = false;
    bool overlap_disabled = false;
    ZRange zr_lo, zr_hi, zr_in;
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_band = nullptr, ev_comm = nullptr;
    // fused sparse epilogue of the vector kernel: tile-sorted injection CSR
    struct FusedSparse {
        bool ok = false;          // built and every cell inside the tile grid
        uint64_t key[8] = {};     // (csr version, grid, zchunk, tile, z-range)
        int* tile_start = nullptr;
        int64_t* cell = nullptr;
        int* start = nullptr;
        int* cp = nullptr;
        float* cw = nullptr;
        size_t cap_tiles = 0, cap_cells = 0, cap_contrib = 0;
    } fused, fused_adj;  // fused_adj: FWI adjoint + gradient kernel (its own tiles)
    bool fused_disabled = false;  // SF_NO_FUSED_SPARSE=1
    // all-zero eta boxes per (tile, plane) for the vector kernels
    // (TmaStencilArgs::eta0); recomputed when eta is rewritten (eta_gen)
    struct EtaFlags {
        uint32_t* bits = nullptr;
        size_t cap = 0;
        int tx = 0, ty = 0, ntx = 0, nty = 0, words = 0;
        uint64_t gen = 0;  // eta_gen the bits describe (0 = none)
    } eta0, eta0_grad;
    uint64_t eta_gen = 1;
    bool eta_skip_disabled = false;  // SF_NO_ETA_SKIP=1

    ~sf_plan();
};

namespace sfb {
namespace {

using Plan = sf_plan;

int64_t field_numel(const Plan& p) {
    int64_t v = 1;
    for (int i = 0; i < p.ndim; ++i) v *= p.n[i];
    return v;
}

// rows of the dense reference layout (product of all but the last axis)
int64_t dense_rows(const Plan& p) { return field_numel(p) / p.n[p.ndim - 1]; }

// Dense host rows <-> padded device rows through a dense device staging
// buffer: one contiguous copy (full PCIe rate) plus a repack kernel, instead
// of a strided 2D copy of 1124-byte rows.
unsigned repack_grid(int64_t rows) {
    return static_cast<unsigned>(std::min<int64_t>(rows, 148 * 16));
}

void h2d_field(const Plan& p, float* dst, const float* src) {
    const int64_t last = p.n[p.ndim - 1];
    const int64_t rows = dense_rows(p);
    SF_CUDA(cudaMemcpyAsync(p.staging, src, sizeof(float) * rows * last, cudaMemcpyHostToDevice,
                            p.stream));
    repack_rows_kernel<<<repack_grid(rows), 256, 0, p.stream>>>(dst, p.pitch, p.staging, last, rows,
                                                               static_cast<int>(last));
}

void d2h_field(const Plan& p, float* dst, const float* src) {
    const int64_t last = p.n[p.ndim - 1];
    const int64_t rows = dense_rows(p);
    repack_rows_kernel<<<repack_grid(rows), 256, 0, p.stream>>>(p.staging, last, src, p.pitch, rows,
                                                               static_cast<int>(last));
    SF_CUDA(cudaMemcpyAsync(dst, p.staging, sizeof(float) * rows * last, cudaMemcpyDeviceToHost,
                            p.stream));
}

int64_t device_offset(const Plan& p, const int32_t* c) {
    if (p.ndim == 3) return c[0] * p.plane + static_cast<int64_t>(c[1]) * p.pitch + c[2];
    return c[0] * p.pitch + c[1];
}

void alloc_points(Plan& p, PointSet& s, int64_t np, int64_t nt) {
    s.np = np;
    s.nt = nt;
    const int corners = 1 << p.ndim;
    s.series = dalloc<float>(static_cast<size_t>(std::max<int64_t>(nt, 1) * np));
    s.ci = dalloc<int>(static_cast<size_t>(np * p.ndim));
    s.w = dalloc<float>(static_cast<size_t>(np * corners));
    SF_CUDA(cudaMemsetAsync(s.series, 0, sizeof(float) * std::max<int64_t>(nt, 1) * np, p.stream));
    SF_CUDA(cudaMemsetAsync(s.ci, 0, sizeof(int) * np * p.ndim, p.stream));
    SF_CUDA(cudaMemsetAsync(s.w, 0, sizeof(float) * np * corners, p.stream));
    s.host_ci.assign(static_cast<size_t>(np * p.ndim), 0);
}

void free_points(PointSet& s) {
    dfree(s.series);
    dfree(s.ci);
    dfree(s.w);
    dfree(s.cell_off);
    dfree(s.start);
    dfree(s.cp);
    dfree(s.cw);
    s = PointSet{};
}

// Validate indices (the reference would index out of bounds silently) and
// build the deterministic injection CSR: distinct target cells, each with its
// (p, w[p][k]) contributions in ascending p.
void clear_graphs(Plan& p) {
    for (auto& kv : p.graphs) cudaGraphExecDestroy(kv.second);
    p.graphs.clear();
}

void upload_points(Plan& p, PointSet& s, const float* series, const int* ci, const float* w,
                   bool injects) {
    const int corners = 1 << p.ndim;
    if (series)
        SF_CUDA(cudaMemcpyAsync(s.series, series, sizeof(float) * s.nt * s.np,
                                cudaMemcpyHostToDevice, p.stream));
    if (ci) {
        for (int64_t q = 0; q < s.np; ++q)
            for (int d = 0; d < p.ndim; ++d) {
                const int v = ci[q * p.ndim + d];
                if (v < 0 || v > p.n[d] - 2)
                    throw Status(SF_ERR_INVALID, "sparse cell index out of range at point " +
                                                     std::to_string(q));
            }
        s.host_ci.assign(ci, ci + s.np * p.ndim);
        SF_CUDA(cudaMemcpyAsync(s.ci, ci, sizeof(int) * s.np * p.ndim, cudaMemcpyHostToDevice,
                                p.stream));
    }
    if (w)
        SF_CUDA(cudaMemcpyAsync(s.w, w, sizeof(float) * s.np * corners, cudaMemcpyHostToDevice,
                                p.stream));
    if (!injects || !(ci || w)) return;
    if (!w || !ci)
        throw Status(SF_ERR_INVALID, "injection needs cell indices and weights together");
    struct Contrib {
        int64_t off;
        int p;
        float w;
        int band;  // 0: a slab's boundary band (sent to a neighbour), 1: inner
    };
    const int r = p.ac.radius;
    auto band_of = [&](int c0) {
        if (p.slab && ((p.has_lower && c0 < p.own_lo + r) || (p.has_upper && c0 >= p.own_hi - r)))
            return 0;
        return p.slab ? 1 : 0;
    };
    std::vector<Contrib> cs;
    cs.reserve(static_cast<size_t>(s.np * corners));
    for (int64_t q = 0; q < s.np; ++q)
        for (int k = 0; k < corners; ++k) {
            int32_t c[3];
            for (int d = 0; d < p.ndim; ++d) c[d] = s.host_ci[q * p.ndim + d] + ((k >> d) & 1);
            // a slab applies only the corners it owns; neighbours apply theirs
            if (c[0] < p.own_lo || c[0] >= p.own_hi) continue;
            cs.push_back({device_offset(p, c), static_cast<int>(q), w[q * corners + k], band_of(c[0])});
        }
    // stable sort by (band, cell) keeps ascending p within a cell
    std::stable_sort(cs.begin(), cs.end(), [](const Contrib& a, const Contrib& b) {
        return a.band != b.band ? a.band < b.band : a.off < b.off;
    });
    std::vector<int64_t> cells;
    std::vector<int> start, cp;
    std::vector<float> cw;
    int nband0 = 0;
    for (size_t i = 0; i < cs.size(); ++i) {
        if (i == 0 || cs[i].off != cs[i - 1].off) {
            cells.push_back(cs[i].off);
            start.push_back(static_cast<int>(i));
            if (cs[i].band == 0) ++nband0;
        }
        cp.push_back(cs[i].p);
        cw.push_back(cs[i].w);
    }
    start.push_back(static_cast<int>(cs.size()));
    if (cells.empty()) {  // nothing owned: keep a valid empty CSR
        cells.push_back(0);
        start.assign(2, 0);
        cp.push_back(0);
        cw.push_back(0.0f);
    }
    const int ncells = cs.empty() ? 0 : static_cast<int>(cells.size());
    const int nb0 = cs.empty() ? 0 : nband0;
    if (s.cell_off && ncells == s.ncells && nb0 == s.nband0 && cells == s.h_cells &&
        start == s.h_start && cp == s.h_cp && cw == s.h_cw)
        return;  // same points: device CSR and captured graphs stay valid
    // the CSR changed: captured graphs bake its sizes (and maybe pointers)
    clear_graphs(p);
    if (!s.cell_off || cells.size() > s.cap_cells || cp.size() > s.cap_contrib) {
        dfree(s.cell_off);
        dfree(s.start);
        dfree(s.cp);
        dfree(s.cw);
        s.cap_cells = cells.size();
        s.cap_contrib = cp.size();
        s.cell_off = dalloc<int64_t>(s.cap_cells);
        s.start = dalloc<int>(s.cap_cells + 1);
        s.cp = dalloc<int>(s.cap_contrib);
        s.cw = dalloc<float>(s.cap_contrib);
    }
    s.ncells = ncells;
    s.nband0 = nb0;
    // synchronous copies (earlier work on the stream may still read the CSR)
    SF_CUDA(cudaStreamSynchronize(p.stream));
    SF_CUDA(cudaMemcpy(s.cell_off, cells.data(), cells.size() * sizeof(int64_t),
                       cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(s.start, start.data(), start.size() * sizeof(int), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(s.cp, cp.data(), cp.size() * sizeof(int), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(s.cw, cw.data(), cw.size() * sizeof(float), cudaMemcpyHostToDevice));
    s.h_cells = std::move(cells);
    s.h_start = std::move(start);
    s.h_cp = std::move(cp);
    s.h_cw = std::move(cw);
    ++s.version;
}

// ---------------------------------------------------------------------------
// launch helpers

// Tile shapes compiled for the 3D stencil: TY in {8, 16}; NX (points per
// thread along a2) up to 4 for R <= 4 and up to 2 above (register queue of
// NX*(2R+1) floats).
template <int R, bool FWD, bool GRAD>
void launch_acoustic3d_t(int nx, int ty, dim3 g, cudaStream_t st, const StencilArgs& A) {
#define SF_T(NXV, TYV)                                                              \
    if (nx == NXV && ty == TYV) {                                                   \
        acoustic3d_kernel<R, FWD, TYV, NXV, GRAD><<<g, dim3(32, TYV), 0, st>>>(A);  \
        return;                                                                     \
    }
    SF_T(1, 8) SF_T(1, 16) SF_T(2, 8) SF_T(2, 16)
    if constexpr (R <= 4) { SF_T(3, 8) SF_T(3, 16) SF_T(4, 8) SF_T(4, 16) }
#undef SF_T
    throw Status(SF_ERR_INVALID, "tile shape not compiled for this order");
}

template <int R, bool FWD, bool GRAD>
const void* acoustic3d_ptr_t(int nx, int ty) {
#define SF_T(NXV, TYV) \
    if (nx == NXV && ty == TYV) return reinterpret_cast<const void*>(&acoustic3d_kernel<R, FWD, TYV, NXV, GRAD>);
    SF_T(1, 8) SF_T(1, 16) SF_T(2, 8) SF_T(2, 16)
    if constexpr (R <= 4) { SF_T(3, 8) SF_T(3, 16) SF_T(4, 8) SF_T(4, 16) }
#undef SF_T
    return nullptr;
}

template <bool FWD, bool GRAD>
const void* acoustic3d_ptr(int r, int nx, int ty) {
    switch (r) {
        case 1: return acoustic3d_ptr_t<1, FWD, GRAD>(nx, ty);
        case 2: return acoustic3d_ptr_t<2, FWD, GRAD>(nx, ty);
        case 3: return acoustic3d_ptr_t<3, FWD, GRAD>(nx, ty);
        case 4: return acoustic3d_ptr_t<4, FWD, GRAD>(nx, ty);
        case 5: return acoustic3d_ptr_t<5, FWD, GRAD>(nx, ty);
        case 6: return acoustic3d_ptr_t<6, FWD, GRAD>(nx, ty);
        case 7: return acoustic3d_ptr_t<7, FWD, GRAD>(nx, ty);
        case 8: return acoustic3d_ptr_t<8, FWD, GRAD>(nx, ty);
        default: return nullptr;
    }
}

template <bool FWD, bool GRAD>
void launch_acoustic3d_r(int r, int nx, int ty, dim3 g, cudaStream_t st, const StencilArgs& A) {
    switch (r) {
#define SF_CASE(RR)                                                                 \
    case RR:                                                                        \
        launch_acoustic3d_t<RR, FWD, GRAD>(nx, ty, g, st, A);                        \
        break;
        SF_CASE(1) SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8)
#undef SF_CASE
        default:
            throw Status(SF_ERR_INVALID, "radius out of range");
    }
}

// ---- TMA path ------------------------------------------------------------
int tma_max_nx(int r) { return r <= 4 ? 4 : 2; }

template <int R, bool FWD>
const void* tma_ptr_t(int nx) {
    switch (nx) {
        case 1: return reinterpret_cast<const void*>(&acoustic3d_tma_kernel<R, FWD, 8, 1>);
        case 2: return reinterpret_cast<const void*>(&acoustic3d_tma_kernel<R, FWD, 8, 2>);
        case 3:
            if constexpr (R <= 4) return reinterpret_cast<const void*>(&acoustic3d_tma_kernel<R, FWD, 8, 3>);
            return nullptr;
        case 4:
            if constexpr (R <= 4) return reinterpret_cast<const void*>(&acoustic3d_tma_kernel<R, FWD, 8, 4>);
            return nullptr;
        default: return nullptr;
    }
}

template <bool FWD>
const void* tma_ptr(int r, int nx) {
    switch (r) {
        case 1: return tma_ptr_t<1, FWD>(nx);
        case 2: return tma_ptr_t<2, FWD>(nx);
        case 3: return tma_ptr_t<3, FWD>(nx);
        case 4: return tma_ptr_t<4, FWD>(nx);
        case 5: return tma_ptr_t<5, FWD>(nx);
        case 6: return tma_ptr_t<6, FWD>(nx);
        case 7: return tma_ptr_t<7, FWD>(nx);
        case 8: return tma_ptr_t<8, FWD>(nx);
        default: return nullptr;
    }
}

int tma_box_width(int r, int nx) { return 32 * nx + 2 * ((r + 3) / 4 * 4); }

size_t tma_smem_bytes(int r, int nx, int stages) {
    const int wb = tma_box_width(r, nx);
    const int cur = (wb * (8 + 2 * r) * 4 + 127) / 128 * 128;
    const int pme = (32 * nx * 8 * 4 + 127) / 128 * 128;
    return 256 + static_cast<size_t>(2 * r + stages) * cur + static_cast<size_t>(stages) * 3 * pme;
}

// ---- vectorised TMA path (4 consecutive a2 points per thread) -------------
// tile_nx selects the tile width for the vector kernel: 2 -> 64-wide tiles
// (16 lanes per row), 1 -> 32-wide (8 lanes per row); rpl = rows per lane.
// Compiled shapes (warps, nx, rpl): (4,2,1) (8,2,1) (4,1,1) (8,1,1) (2,1,2) (4,2,2), and
// (16,2,1) at radius 4.
template <bool FWD, int RR>
const void* vec_ptr_r(int warps, int nx, int rpl) {
    if (rpl == 2) {
        if (nx == 1 && warps == 2)
            return reinterpret_cast<const void*>(&acoustic3d_vec_kernel<RR, FWD, 2, false, 8, 2>);
        if (nx == 2 && warps == 4)
            return reinterpret_cast<const void*>(&acoustic3d_vec_kernel<RR, FWD, 4, false, 16, 2>);
        return nullptr;
    }
    if (nx == 1)
        return warps == 4   ? reinterpret_cast<const void*>(&acoustic3d_vec_kernel<RR, FWD, 4, false, 8>)
               : warps == 8 ? reinterpret_cast<const void*>(&acoustic3d_vec_kernel<RR, FWD, 8, false, 8>)
                            : nullptr;
    if (rpl == kRplAq2)
        return RR == 4 && warps == 16 ? reinterpret_cast<const void*>(
                                            &acoustic3d_vec_kernel<4, FWD, 16, false, 16, 1, true, 2>)
                                      : nullptr;
    if (rpl == kRplAq) {  // radius 4, 64-wide tiles, a0 register queue
        if (RR != 4) return nullptr;
        return warps == 16 ? reinterpret_cast<const void*>(
                                 &acoustic3d_vec_kernel<4, FWD, 16, false, 16, 1, true>)
               : warps == 8 ? reinterpret_cast<const void*>(
                                  &acoustic3d_vec_kernel<4, FWD, 8, false, 16, 1, true>)
                            : nullptr;
    }
    if (warps == 16)  // 64 x 32 tiles, one CTA per SM (radius 4 only)
        return RR == 4 ? reinterpret_cast<const void*>(&acoustic3d_vec_kernel<4, FWD, 16>) : nullptr;
    return warps == 4 ? reinterpret_cast<const void*>(&acoustic3d_vec_kernel<RR, FWD, 4>)
                      : reinterpret_cast<const void*>(&acoustic3d_vec_kernel<RR, FWD, 8>);
}

template <bool FWD>
const void* vec_ptr(int r, int warps, int nx = 2, int rpl = 1) {
    switch (r) {
        case 1: return vec_ptr_r<FWD, 1>(warps, nx, rpl);
        case 2: return vec_ptr_r<FWD, 2>(warps, nx, rpl);
        case 3: return vec_ptr_r<FWD, 3>(warps, nx, rpl);
        case 4: return vec_ptr_r<FWD, 4>(warps, nx, rpl);
        default: return nullptr;
    }
}

size_t vec_smem_bytes(int r, int warps, int stages, int npme = 3, int nx = 2, int rpl = 1) {
    const int ra = (r + 3) / 4 * 4;
    const int tx = 32 * nx, ty = 4 * warps * rpl / nx;
    const int wb = tx + 2 * ra, h = ty + 2 * r;
    const int cur = (wb * h * 4 + 127) / 128 * 128;
    const int pme = (tx * ty * 4 + 127) / 128 * 128;
    return 256 + static_cast<size_t>(2 * r + stages) * cur +
           static_cast<size_t>(stages) * npme * pme;
}

template <bool FWD>
const void* vecq_ptr(int r, int warps, int ring = 0) {
#define SF_V(RR)                                                                               \
    case RR:                                                                                   \
        if (ring == 1 && warps == 4) return reinterpret_cast<const void*>(&acoustic3d_vecq2_kernel<RR, FWD, 4>); \
        if (ring == 4) return reinterpret_cast<const void*>(&acoustic3d_vecqt_kernel<RR, FWD>);                \
        if ((ring == 5 || (ring == 0 && RR == 6)) && warps == 4) return reinterpret_cast<const void*>(&acoustic3d_vecq_kernel<RR, FWD, 4, true>); \
        if (ring == 5 && warps == 8) return reinterpret_cast<const void*>(&acoustic3d_vecq_kernel<RR, FWD, 8, true>); \
        if (warps == 12) return RR >= 7 ? (ring == 5 ? reinterpret_cast<const void*>(&acoustic3d_vecq_kernel<(RR >= 7 ? RR : 7), FWD, 12, true>) \
                                                     : reinterpret_cast<const void*>(&acoustic3d_vecq_kernel<(RR >= 7 ? RR : 7), FWD, 12>)) : nullptr; \
        if (ring == 2 && warps == 4) return reinterpret_cast<const void*>(&acoustic3d_vecq_free_kernel<RR, FWD, 4>); \
        return warps == 4 ? reinterpret_cast<const void*>(&acoustic3d_vecq_kernel<RR, FWD, 4>) \
                          : reinterpret_cast<const void*>(&acoustic3d_vecq_kernel<RR, FWD, 8>);
    switch (r) {
        SF_V(5) SF_V(6) SF_V(7) SF_V(8)
        default: return nullptr;
    }
#undef SF_V
}

size_t vecq_smem_bytes(int r, int warps, int stages, bool ring = false) {
    const int ra = (r + 3) / 4 * 4;
    const int cur = ((64 + 2 * ra) * (2 * warps + 2 * r) * 4 + 127) / 128 * 128;
    const int pme = (64 * 2 * warps * 4 + 127) / 128 * 128;
    if (ring)  // + the core box of plane z+R per stage and the ring of R + S core planes
        return 256 + static_cast<size_t>(stages) * (cur + 4 * pme) + static_cast<size_t>(r + stages) * pme;
    return 256 + static_cast<size_t>(stages) * (cur + 3 * pme);
}

template <bool FWD>
void launch_vecq(int r, int warps, dim3 g, size_t smem, cudaStream_t st, const TmaStencilArgs& A,
                 int ring = 0) {
    const dim3 b(32 * warps);
#define SF_V(RR)                                                                   \
    case RR:                                                                       \
        if (ring == 1 && warps == 4)                                               \
            acoustic3d_vecq2_kernel<RR, FWD, 4><<<g, b, smem, st>>>(A);            \
        else if (ring == 4)                                                        \
            acoustic3d_vecqt_kernel<RR, FWD><<<g, dim3(128), smem, st>>>(A);       \
        else if ((ring == 5 || (ring == 0 && RR == 6)) && warps == 4)              \
            acoustic3d_vecq_kernel<RR, FWD, 4, true><<<g, b, smem, st>>>(A);       \
        else if (ring == 5 && warps == 8)                                          \
            acoustic3d_vecq_kernel<RR, FWD, 8, true><<<g, b, smem, st>>>(A);       \
        else if (warps == 12 && RR >= 7 && ring == 5)                              \
            acoustic3d_vecq_kernel<(RR >= 7 ? RR : 7), FWD, 12, true><<<g, b, smem, st>>>(A); \
        else if (warps == 12 && RR >= 7)                                           \
            acoustic3d_vecq_kernel<(RR >= 7 ? RR : 7), FWD, 12><<<g, b, smem, st>>>(A); \
        else if (ring == 2 && warps == 4)                                          \
            acoustic3d_vecq_free_kernel<RR, FWD, 4><<<g, b, smem, st>>>(A);        \
        else if (warps == 4)                                                       \
            acoustic3d_vecq_kernel<RR, FWD, 4><<<g, b, smem, st>>>(A);             \
        else                                                                       \
            acoustic3d_vecq_kernel<RR, FWD, 8><<<g, b, smem, st>>>(A);             \
        return;
    switch (r) {
        SF_V(5) SF_V(6) SF_V(7) SF_V(8)
        default: throw Status(SF_ERR_INVALID, "queue vector stencil compiled for radius 5..8");
    }
#undef SF_V
}

// FWI adjoint + gradient, vectorised: 4-warp CTAs (6 boxes per stage)
const void* vec_grad_ptr(int r) {
    switch (r) {
        case 1: return reinterpret_cast<const void*>(&acoustic3d_vec_kernel<1, false, 4, true>);
        case 2: return reinterpret_cast<const void*>(&acoustic3d_vec_kernel<2, false, 4, true>);
        case 3: return reinterpret_cast<const void*>(&acoustic3d_vec_kernel<3, false, 4, true>);
        case 4: return reinterpret_cast<const void*>(&acoustic3d_vec_kernel<4, false, 4, true>);
        default: return nullptr;
    }
}

void launch_vec_grad(int r, dim3 g, size_t smem, cudaStream_t st, const TmaStencilArgs& A) {
    const dim3 b(160);  // 4 consumer warps + the TMA producer warp
    switch (r) {
        case 1: acoustic3d_vec_kernel<1, false, 4, true><<<g, b, smem, st>>>(A); return;
        case 2: acoustic3d_vec_kernel<2, false, 4, true><<<g, b, smem, st>>>(A); return;
        case 3: acoustic3d_vec_kernel<3, false, 4, true><<<g, b, smem, st>>>(A); return;
        case 4: acoustic3d_vec_kernel<4, false, 4, true><<<g, b, smem, st>>>(A); return;
        default: throw Status(SF_ERR_INVALID, "vector gradient stencil compiled for radius <= 4");
    }
}

// Programmatic dependent launch: a vector-kernel launch may begin while the
// previous kernel on the stream drains (its CTAs prefetch the static m/eta
// boxes, then griddepcontrol.wait for the previous grid before touching
// anything it wrote). SF_NO_PDL=1 launches plainly.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SF_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

// Set for the launch that follows a chunk's eta-flag kernel in
// invoke_overlapped: the flags are what a producer warp reads before
// griddepcontrol.wait, so that launch is plainly stream-ordered.
thread_local bool g_plain_launches = false;

template <typename Kern>
void launch_pdl(Kern kernel, dim3 g, dim3 b, size_t smem, cudaStream_t st, const TmaStencilArgs& A) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() && !g_plain_launches ? 1 : 0;
    SF_CUDA(cudaLaunchKernelEx(&cfg, kernel, A));
}

template <bool FWD>
void launch_vec(int r, int warps, int nx, int rpl, dim3 g, size_t smem, cudaStream_t st,
                const TmaStencilArgs& A) {
    const dim3 b(32 * (warps + 1));  // + the TMA producer warp
#define SF_V(RR)                                                                             \
    case RR:                                                                                 \
        if (rpl == kRplAq2)                                                                  \
            launch_pdl(acoustic3d_vec_kernel<4, FWD, 16, false, 16, 1, true, 2>, g, b, smem, st, A); \
        else if (rpl == kRplAq && warps == 16)                                               \
            launch_pdl(acoustic3d_vec_kernel<4, FWD, 16, false, 16, 1, true>, g, b, smem, st, A); \
        else if (rpl == kRplAq)                                                              \
            launch_pdl(acoustic3d_vec_kernel<4, FWD, 8, false, 16, 1, true>, g, b, smem, st, A); \
        else if (rpl == 2 && nx == 1)                                                        \
            launch_pdl(acoustic3d_vec_kernel<RR, FWD, 2, false, 8, 2>, g, b, smem, st, A);   \
        else if (rpl == 2)                                                                   \
            launch_pdl(acoustic3d_vec_kernel<RR, FWD, 4, false, 16, 2>, g, b, smem, st, A);  \
        else if (nx == 1 && warps == 8)                                                      \
            launch_pdl(acoustic3d_vec_kernel<RR, FWD, 8, false, 8>, g, b, smem, st, A);      \
        else if (nx == 1)                                                                    \
            launch_pdl(acoustic3d_vec_kernel<RR, FWD, 4, false, 8>, g, b, smem, st, A);      \
        else if (warps == 4)                                                                 \
            launch_pdl(acoustic3d_vec_kernel<RR, FWD, 4>, g, b, smem, st, A);                \
        else if (warps == 16)                                                                \
            launch_pdl(acoustic3d_vec_kernel<4, FWD, 16>, g, b, smem, st, A);                \
        else                                                                                 \
            launch_pdl(acoustic3d_vec_kernel<RR, FWD, 8>, g, b, smem, st, A);                \
        return;
    switch (r) {
        SF_V(1) SF_V(2) SF_V(3) SF_V(4)
        default: throw Status(SF_ERR_INVALID, "vector stencil compiled for radius <= 4");
    }
#undef SF_V
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    // resolved once (thread-safe static initialisation); a failed lookup is
    // retried on the next call rather than cached
    static const PFN_cuTensorMapEncodeTiled_v12000 cached = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            ptr = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }();
    if (cached) return cached;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    SF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !ptr)
        throw Status(SF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
}

// 3D map over one padded field: dims (n2, n1, n0), row/plane strides in
// bytes (multiples of 16 by the 32-float pitch), box (bx, by, 1).
// 4D map over `levels` consecutive padded fields (a time slot: 1 level; the
// FWI history: nt+2): dims (n2, n1, n0, levels), strides in bytes (16-byte
// multiples by the 32-float pitch), box (bx, by, 1, 1).
void make_tensor_map(CUtensorMap* map, const Plan& p, const float* base, uint32_t bx, uint32_t by,
                     int64_t levels = 1) {
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(p.n[2]), static_cast<cuuint64_t>(p.n[1]),
                          static_cast<cuuint64_t>(p.n[0]), static_cast<cuuint64_t>(levels)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(p.pitch) * 4,
                             static_cast<cuuint64_t>(p.plane) * 4,
                             static_cast<cuuint64_t>(p.slot_elems) * 4};
    cuuint32_t box[4] = {bx, by, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                      const_cast<float*>(base), dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Status(SF_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

void setup_tma(Plan& p) {
    const int r = p.ac.radius;
    const int nx = p.tile_nx;
    // vector kernels: ring/queue (64 x 2*warps tiles) or ring with 32-wide tiles
    const int vnx = p.use_vecq ? 2 : nx;
    const uint32_t wb = static_cast<uint32_t>(p.use_vec ? 32 * vnx + 2 * ((r + 3) / 4 * 4)
                                                        : tma_box_width(r, nx));
    const uint32_t ty = static_cast<uint32_t>(
        p.use_vec ? 4 * p.vec_warps * (p.use_vecq ? 1 : p.vec_rpl) / vnx : 8);
    const uint32_t tx = static_cast<uint32_t>(p.use_vec ? 32 * vnx : 32 * nx);
    const uint32_t cy = ty + static_cast<uint32_t>(2 * r);
    for (int s = 0; s < 3; ++s) {
        if (p.slot[s]) {
            make_tensor_map(&p.tm_cur[s], p, p.slot[s], wb, cy);
            make_tensor_map(&p.tm_pme[s], p, p.slot[s], tx, ty);
        }
    }
    make_tensor_map(&p.tm_m, p, p.m, tx, ty);
    make_tensor_map(&p.tm_eta, p, p.eta, tx, ty);
    if (p.kind == Plan::FWI) {
        // forward (history levels): the stencil's tile; adjoint slots v and the
        // gradient kernel's m / eta / u-history boxes: its fixed 64 x 8 tile
        const uint32_t gty = 8, gcy = gty + static_cast<uint32_t>(2 * r);
        make_tensor_map(&p.tm_hist_cur, p, p.hist, wb, cy, p.nt + 2);
        make_tensor_map(&p.tm_hist_pme, p, p.hist, tx, ty, p.nt + 2);
        make_tensor_map(&p.tm_hist_pme_g, p, p.hist, 64, gty, p.nt + 2);
        make_tensor_map(&p.tm_m_g, p, p.m, 64, gty);
        make_tensor_map(&p.tm_eta_g, p, p.eta, 64, gty);
        const uint32_t gwb = 64 + 2 * static_cast<uint32_t>((r + 3) / 4 * 4);
        for (int s = 0; s < 3; ++s) {
            make_tensor_map(&p.tm_v_cur[s], p, p.v[s], wb, cy);
            make_tensor_map(&p.tm_v_pme[s], p, p.v[s], tx, ty);
            make_tensor_map(&p.tm_v_cur_g[s], p, p.v[s], gwb, gcy);
            make_tensor_map(&p.tm_v_pme_g[s], p, p.v[s], 64, gty);
        }
    }
    if (p.use_vecq) {
        const bool ring = p.vecq_ring == 1 && p.vec_warps == 4;
        int stages = ring ? 2 : 3;  // ring: 2 stages keep 4 CTAs per SM within shared memory
        if (const char* env = std::getenv("SF_TMA_STAGES")) {
            const int v = std::atoi(env);
            if (v >= 2 && v <= 12) stages = v;
        }
        if (p.stages_override >= 2) stages = std::min(p.stages_override, 12);
        p.tma_stages = stages;  // <= 12: barriers + eta flags share 256 bytes
        p.tma_smem = vecq_smem_bytes(r, p.vec_warps, stages, ring);
        if (p.vecq_ring == 4) {
            // TMEM queue: 128 columns per CTA, so at most 4 CTAs per SM may be
            // resident (a fifth would wait in tcgen05.alloc): shared memory
            // sized to allow no more than 4
            p.vec_warps = 4;
            p.tma_smem = std::max<size_t>(p.tma_smem, 228 * 1024 / 5 + 1024);
        }
        for (int fwd = 0; fwd < 2; ++fwd) {
            const void* fn = fwd ? vecq_ptr<true>(r, p.vec_warps, p.vecq_ring)
                                 : vecq_ptr<false>(r, p.vec_warps, p.vecq_ring);
            if (!fn) throw Status(SF_ERR_INVALID, "queue vector stencil not compiled");
            SF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(p.tma_smem)));
        }
        return;
    }
    if (p.use_vec) {
        int stages = 3;
        const int rpl = p.vec_rpl;
        const size_t ctas = p.vec_warps == 16 ? 1 : 2;  // CTAs per SM the depth must leave room for
        while (stages > 2 && vec_smem_bytes(r, p.vec_warps, stages, 3, nx, rpl) * ctas > 226 * 1024)
            --stages;
        if (const char* env = std::getenv("SF_TMA_STAGES")) {
            const int v = std::atoi(env);
            if (v >= 2 && v <= 12) stages = v;
        }
        if (p.stages_override >= 2) stages = std::min(p.stages_override, 12);
        p.tma_stages = stages;  // <= 12: barriers + eta flags share 256 bytes
        p.tma_smem = vec_smem_bytes(r, p.vec_warps, stages, 3, nx, rpl);
        for (int fwd = 0; fwd < 2; ++fwd) {
            const void* fn = fwd ? vec_ptr<true>(r, p.vec_warps, nx, p.vec_kernel_rpl())
                                 : vec_ptr<false>(r, p.vec_warps, nx, p.vec_kernel_rpl());
            if (!fn) throw Status(SF_ERR_INVALID, "vector stencil not compiled");
            SF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(p.tma_smem)));
        }
        if (p.kind == Plan::FWI) {
            // the gradient kernel streams 6 boxes per stage and prefers a deeper
            // pipeline than the forward (C5 adjoint: 4 stages 166 ms, 3 stages
            // 174 ms per sweep); SF_TMA_STAGES_GRAD overrides
            int gst = 4;
            if (const char* env = std::getenv("SF_TMA_STAGES_GRAD")) {
                const int v = std::atoi(env);
                if (v >= 2 && v <= 12) gst = v;
            }
            p.tma_stages_grad = gst;
            make_tensor_map(&p.tm_grad, p, p.grad, 64, 8);
            p.smem_grad = vec_smem_bytes(r, 4, gst, 6);
            SF_CUDA(cudaFuncSetAttribute(vec_grad_ptr(r), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(p.smem_grad)));
        }
        return;
    }
    // 3 planes in flight measured best on B200 (c2: S=3 86.6 us, S=4 101 us,
    // S=8 161 us per launch: occupancy beats depth); at least 2 CTAs per SM
    int stages = 3;
    while (stages > 2 && tma_smem_bytes(r, nx, stages) * 2 > 220 * 1024) --stages;
    if (const char* env = std::getenv("SF_TMA_STAGES")) {
        const int v = std::atoi(env);
        if (v >= 2 && v <= 16) stages = v;
    }
    if (p.stages_override >= 2) stages = p.stages_override;
    p.tma_stages = stages;
    p.tma_smem = tma_smem_bytes(r, nx, stages);
    for (int fwd = 0; fwd < 2; ++fwd) {
        const void* fn = fwd ? tma_ptr<true>(r, nx) : tma_ptr<false>(r, nx);
        if (!fn) throw Status(SF_ERR_INVALID, "TMA tile not compiled");
        SF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(p.tma_smem)));
    }
}

template <int R, bool FWD>
void launch_tma_t(int nx, dim3 g, size_t smem, cudaStream_t st, const TmaStencilArgs& A) {
    dim3 b(32, 8);
    switch (nx) {
        case 1: acoustic3d_tma_kernel<R, FWD, 8, 1><<<g, b, smem, st>>>(A); return;
        case 2: acoustic3d_tma_kernel<R, FWD, 8, 2><<<g, b, smem, st>>>(A); return;
        case 3:
            if constexpr (R <= 4) { acoustic3d_tma_kernel<R, FWD, 8, 3><<<g, b, smem, st>>>(A); return; }
            break;
        case 4:
            if constexpr (R <= 4) { acoustic3d_tma_kernel<R, FWD, 8, 4><<<g, b, smem, st>>>(A); return; }
            break;
    }
    throw Status(SF_ERR_INVALID, "TMA tile not compiled");
}

template <bool FWD>
void launch_tma(int r, int nx, dim3 g, size_t smem, cudaStream_t st, const TmaStencilArgs& A) {
    switch (r) {
        case 1: return launch_tma_t<1, FWD>(nx, g, smem, st, A);
        case 2: return launch_tma_t<2, FWD>(nx, g, smem, st, A);
        case 3: return launch_tma_t<3, FWD>(nx, g, smem, st, A);
        case 4: return launch_tma_t<4, FWD>(nx, g, smem, st, A);
        case 5: return launch_tma_t<5, FWD>(nx, g, smem, st, A);
        case 6: return launch_tma_t<6, FWD>(nx, g, smem, st, A);
        case 7: return launch_tma_t<7, FWD>(nx, g, smem, st, A);
        case 8: return launch_tma_t<8, FWD>(nx, g, smem, st, A);
        default: throw Status(SF_ERR_INVALID, "radius out of range");
    }
}

template <bool FWD>
void launch_acoustic2d_r(int r, dim3 g, dim3 b, cudaStream_t st, const StencilArgs& A) {
    switch (r) {
#define SF_CASE(RR)                                              \
    case RR:                                                     \
        acoustic2d_kernel<RR, FWD><<<g, b, 0, st>>>(A);          \
        break;
        SF_CASE(1) SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8)
#undef SF_CASE
        default:
            throw Status(SF_ERR_INVALID, "radius out of range");
    }
}

void launch_diffusion_r(int r, dim3 g, dim3 b, cudaStream_t st, const DiffusionArgs& A) {
    switch (r) {
#define SF_CASE(RR)                                              \
    case RR:                                                     \
        diffusion_kernel<RR><<<g, b, 0, st>>>(A);                \
        break;
        SF_CASE(1) SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8)
#undef SF_CASE
        default:
            throw Status(SF_ERR_INVALID, "radius out of range");
    }
}

StencilArgs stencil_args(const Plan& p, float* out, const float* cur, const float* prev) {
    StencilArgs A{};
    A.out = out;
    A.cur = cur;
    A.prev = prev;
    A.m = p.m;
    A.eta = p.eta;
    A.pitch = p.pitch;
    A.plane = p.plane;
    A.n0 = static_cast<int>(p.n[0]);
    A.n1 = static_cast<int>(p.n[1]);
    A.n2 = static_cast<int>(p.ndim == 3 ? p.n[2] : 1);
    A.zchunk = p.zchunk;
    A.z0 = p.z0;
    A.z1 = p.z1;
    A.ce = p.ac.ce;
    A.cm = p.ac.cm;
    for (int k = 0; k < 3; ++k) A.tc[k] = p.ac.tc[k];
    A.c0 = p.ac.c0;
    for (int j = 0; j < 8; ++j) A.cj[j] = p.ac.cj[j];
    return A;
}

// Tensor maps (halo'd box + plain box) and level addressing `f`.
struct MapSel {
    const CUtensorMap* cur = nullptr;
    const CUtensorMap* pme = nullptr;
    int level = 0;
    // the FWI gradient kernel's 64 x 8 boxes of the same buffer (v slots, history)
    const CUtensorMap* cur_g = nullptr;
    const CUtensorMap* pme_g = nullptr;
};

bool map_for(const Plan& p, const float* f, MapSel* m) {
    for (int s = 0; s < 3; ++s) {
        if (p.slot[s] && f == p.slot[s]) {
            *m = {&p.tm_cur[s], &p.tm_pme[s], 0};
            return true;
        }
        if (p.v[s] && f == p.v[s]) {
            *m = {&p.tm_v_cur[s], &p.tm_v_pme[s], 0, &p.tm_v_cur_g[s], &p.tm_v_pme_g[s]};
            return true;
        }
    }
    if (p.hist && f >= p.hist) {
        const int64_t d = f - p.hist;
        if (d % p.slot_elems == 0 && d / p.slot_elems < p.nt + 2) {
            *m = {&p.tm_hist_cur, &p.tm_hist_pme, static_cast<int>(d / p.slot_elems), nullptr,
                  &p.tm_hist_pme_g};
            return true;
        }
    }
    return false;
}

// Sparse work folded into the vector kernel's epilogue (TmaStencilArgs).
struct Epilogue {
    const PointSet* inj = nullptr;  // inject this step's row (tile-sorted CSR)
    int64_t inj_row = 0;
    const PointSet* smp = nullptr;  // sample the previous step from `cur`
    int64_t smp_row = 0;
};

void launch_stencil(const Plan& p, float* out, const float* cur, const float* prev,
                    float* grad = nullptr, const float* uhist = nullptr,
                    const sf_plan::ZRange* zr = nullptr, const Epilogue* epi = nullptr) {
    if (zr && zr->z0 >= zr->z1) return;
    const dim3 grid3 = zr ? zr->grid : p.grid3;
    MapSel mc, mp, mo, mu;
    const bool maps = p.use_tma && p.ndim == 3 && map_for(p, cur, &mc) && map_for(p, prev, &mp);
    const bool grad_ok =
        !grad || (p.use_vec && !p.use_vecq && map_for(p, out, &mo) && map_for(p, uhist, &mu) &&
                  mc.cur_g && mp.pme_g && mo.pme_g && mu.pme_g);
    if (maps && grad_ok) {
        TmaStencilArgs T;
        std::memset(&T, 0, sizeof T);
        T.cur = *mc.cur;
        T.prev = *mp.pme;
        T.lv_cur = mc.level;
        T.lv_prev = mp.level;
        T.cur_ptr = cur;  // the level's own base: queue-head loads add no level offset
        T.level_elems = 0;
        T.m = p.tm_m;
        T.eta = p.tm_eta;
        T.out = out;
        T.pitch = static_cast<int>(p.pitch);
        T.plane = static_cast<int>(p.plane);
        T.n0 = static_cast<int>(p.n[0]);
        T.n1 = static_cast<int>(p.n[1]);
        T.n2 = static_cast<int>(p.n[2]);
        T.zchunk = zr ? zr->zchunk : p.zchunk;
        T.z0 = zr ? zr->z0 : p.z0;
        T.z1 = zr ? zr->z1 : p.z1;
        T.stages = p.tma_stages;
        T.ce = p.ac.ce;
        T.cm = p.ac.cm;
        for (int k = 0; k < 3; ++k) T.tc[k] = p.ac.tc[k];
        T.c0 = p.ac.c0;
        for (int j = 0; j < 8; ++j) T.cj[j] = p.ac.cj[j];
        {
            const sf_plan::EtaFlags& ef = grad ? p.eta0_grad : p.eta0;
            if (ef.bits && ef.gen == p.eta_gen && (p.use_vec || p.use_vecq)) {
                T.eta0 = ef.bits;
                T.eta0_ntx = ef.ntx;
                T.eta0_words = ef.words;
            }
        }
        T.pk_one = f2_splat_host(1.0f);
        T.pk_ce = f2_splat_host(T.ce);
        T.pk_cm = f2_splat_host(T.cm);
        for (int k = 0; k < 3; ++k) T.pk_tc[k] = f2_splat_host(T.tc[k]);
        T.pk_c0 = f2_splat_host(T.c0);
        for (int j = 0; j < 8; ++j) T.pk_cj[j] = f2_splat_host(T.cj[j]);
        if (grad) {  // the gradient kernel's own 64 x 8 boxes of every buffer
            T.stages = p.tma_stages_grad;
            T.cur = *mc.cur_g;
            T.prev = *mp.pme_g;
            T.old = *mo.pme_g;
            T.uh = *mu.pme_g;
            T.m = p.tm_m_g;
            T.eta = p.tm_eta_g;
            T.lv_uh = mu.level;
            T.grad = p.tm_grad;
            T.gradp = grad;
            T.zchunk = p.zchunk_grad;
            if (epi && epi->inj && p.fused_adj.ok && epi->inj->np > 0 && epi->inj->ncells > 0) {
                T.inj_tile_start = p.fused_adj.tile_start;
                T.inj_cell = p.fused_adj.cell;
                T.inj_start = p.fused_adj.start;
                T.inj_cp = p.fused_adj.cp;
                T.inj_cw = p.fused_adj.cw;
                T.inj_row = epi->inj->series + epi->inj_row * epi->inj->np;
                T.mfield = p.m;
                T.inj_scale = p.ac.src_scale;
            }
            if (epi && epi->smp && epi->smp->np > 0) {
                T.smp_field = cur;
                T.smp_ci = epi->smp->ci;
                T.smp_w = epi->smp->w;
                T.smp_out = epi->smp->series + epi->smp_row * epi->smp->np;
                T.smp_np = static_cast<int>(epi->smp->np);
            }
            launch_vec_grad(p.ac.radius, p.grid_grad, p.smem_grad, p.stream, T);
            return;
        }
        if (p.use_vecq) {
            T.cur_core = *mc.pme;
            if (p.ac.forward)
                launch_vecq<true>(p.ac.radius, p.vec_warps, grid3, p.tma_smem, p.stream, T, p.vecq_ring);
            else
                launch_vecq<false>(p.ac.radius, p.vec_warps, grid3, p.tma_smem, p.stream, T, p.vecq_ring);
            return;
        }
        if (p.use_vec) {
            if (epi && epi->inj && p.fused.ok && epi->inj->np > 0 && epi->inj->ncells > 0) {
                T.inj_tile_start = p.fused.tile_start;
                T.inj_cell = p.fused.cell;
                T.inj_start = p.fused.start;
                T.inj_cp = p.fused.cp;
                T.inj_cw = p.fused.cw;
                T.inj_row = epi->inj->series + epi->inj_row * epi->inj->np;
                T.mfield = p.m;
                T.inj_scale = p.ac.src_scale;
            }
            if (epi && epi->smp && epi->smp->np > 0) {
                T.smp_field = cur;
                T.smp_ci = epi->smp->ci;
                T.smp_w = epi->smp->w;
                T.smp_out = epi->smp->series + epi->smp_row * epi->smp->np;
                T.smp_np = static_cast<int>(epi->smp->np);
            }
            if (p.ac.forward)
                launch_vec<true>(p.ac.radius, p.vec_warps, p.tile_nx, p.vec_kernel_rpl(), grid3,
                                 p.tma_smem, p.stream, T);
            else
                launch_vec<false>(p.ac.radius, p.vec_warps, p.tile_nx, p.vec_kernel_rpl(), grid3,
                                  p.tma_smem, p.stream, T);
            return;
        }
        if (p.ac.forward)
            launch_tma<true>(p.ac.radius, p.tile_nx, grid3, p.tma_smem, p.stream, T);
        else
            launch_tma<false>(p.ac.radius, p.tile_nx, grid3, p.tma_smem, p.stream, T);
        return;
    }
    StencilArgs A = stencil_args(p, out, cur, prev);
    A.grad = grad;
    A.uhist = uhist;
    if (zr) {
        A.z0 = zr->z0;
        A.z1 = zr->z1;
        A.zchunk = zr->zchunk;
    }
    const int r = p.ac.radius;
    if (p.ndim == 3) {
        if (grad) {
            launch_acoustic3d_r<false, true>(r, p.tile_nx, p.tile_ty, grid3, p.stream, A);
        } else if (p.ac.forward) {
            launch_acoustic3d_r<true, false>(r, p.tile_nx, p.tile_ty, grid3, p.stream, A);
        } else {
            launch_acoustic3d_r<false, false>(r, p.tile_nx, p.tile_ty, grid3, p.stream, A);
        }
    } else {
        dim3 b(64, 4);
        dim3 g(static_cast<unsigned>((p.n[1] + 63) / 64), static_cast<unsigned>((p.n[0] + 3) / 4));
        if (p.ac.forward)
            launch_acoustic2d_r<true>(r, g, b, p.stream, A);
        else
            launch_acoustic2d_r<false>(r, g, b, p.stream, A);
    }
}

void launch_inject(const Plan& p, const PointSet& s, float* field, int64_t row, int first = 0,
                   int count = -1, int zf0 = 0, int zf1 = 0) {
    if (count < 0) count = s.ncells - first;
    if (count <= 0 || s.np == 0) return;
    InjectArgs A{};
    A.field = field;
    A.m = p.m;
    A.row = s.series + row * s.np;
    A.cell_off = s.cell_off;
    A.start = s.start;
    A.cp = s.cp;
    A.cw = s.cw;
    A.scale = p.ac.src_scale;
    A.cell_off = s.cell_off + first;
    A.start = s.start + first;
    A.ncells = count;
    A.plane = p.plane;
    A.zf0 = zf0;
    A.zf1 = zf1;
    inject_kernel<<<(count + 255) / 256, 256, 0, p.stream>>>(A);
}

void launch_sample(const Plan& p, const PointSet& s, const float* field, int64_t row, int zf0 = 0,
                   int zf1 = 0) {
    if (s.np == 0) return;
    SampleArgs A{};
    A.zf0 = zf0;
    A.zf1 = zf1;
    A.field = field;
    A.ci = s.ci;
    A.w = s.w;
    A.out = s.series + row * s.np;
    A.pitch = p.pitch;
    A.plane = p.plane;
    A.np = static_cast<int>(s.np);
    const unsigned g = static_cast<unsigned>((s.np + 255) / 256);
    if (p.ndim == 3)
        sample_kernel<3><<<g, 256, 0, p.stream>>>(A);
    else
        sample_kernel<2><<<g, 256, 0, p.stream>>>(A);
}


// ---------------------------------------------------------------------------
// NCCL, loaded at run time (dlopen) so the library never pins an NCCL build
// into processes that also load PyTorch's: the copy already mapped in the
// process (RTLD_NOLOAD) is preferred, else the system libnccl.so.2.
struct NcclId {
    char internal[128];  // ncclUniqueId
};
struct NcclApi {
    int (*GetUniqueId)(NcclId*) = nullptr;
    int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
constexpr int kNcclFloat32 = 7;  // ncclFloat32 in nccl.h

const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (loaded) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) throw Status(SF_ERR_CUDA, "libnccl.so.2 not found");
    auto sym = [&](const char* n) {
        void* f = dlsym(h, n);
        if (!f) throw Status(SF_ERR_CUDA, std::string("NCCL symbol missing: ") + n);
        return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    loaded = true;
    return api;
}

void nccl_check(int rc, const char* what) {
    if (rc != 0)
        throw Status(SF_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(rc));
}

// Halo exchange of the level just written (after injection, so halos carry
// injected values): my first r owned planes go down, my last r owned planes
// go up; the neighbours' planes land in my r-deep halos. Planes are
// contiguous (axis 0 is the slowest), one message per face.
void launch_exchange_nccl(const Plan& p, float* f) {
    const NcclApi& N = nccl();
    const int r = p.ac.radius;
    const size_t count = static_cast<size_t>(r) * static_cast<size_t>(p.plane);
    nccl_check(N.GroupStart(), "ncclGroupStart");
    if (p.has_lower) {
        nccl_check(N.Send(f + static_cast<int64_t>(p.own_lo) * p.plane, count, kNcclFloat32,
                          p.nccl_rank - 1, p.nccl_comm, p.stream), "ncclSend");
        nccl_check(N.Recv(f + static_cast<int64_t>(p.own_lo - r) * p.plane, count, kNcclFloat32,
                          p.nccl_rank - 1, p.nccl_comm, p.stream), "ncclRecv");
    }
    if (p.has_upper) {
        nccl_check(N.Send(f + static_cast<int64_t>(p.own_hi - r) * p.plane, count, kNcclFloat32,
                          p.nccl_rank + 1, p.nccl_comm, p.stream), "ncclSend");
        nccl_check(N.Recv(f + static_cast<int64_t>(p.own_hi) * p.plane, count, kNcclFloat32,
                          p.nccl_rank + 1, p.nccl_comm, p.stream), "ncclRecv");
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
}

// Injection then sampling on `field`: one fused single-CTA launch when both
// point sets are small, else the two grid-wide kernels.
constexpr int kFusedSparseMax = 4096;

void launch_inject_sample(const Plan& p, const PointSet& inj, const PointSet& smp, float* field,
                          int64_t row) {
    if (inj.ncells <= kFusedSparseMax && smp.np <= kFusedSparseMax) {
        InjectArgs I{};
        I.field = field;
        I.m = p.m;
        I.row = inj.series + row * inj.np;
        I.cell_off = inj.cell_off;
        I.start = inj.start;
        I.cp = inj.cp;
        I.cw = inj.cw;
        I.scale = p.ac.src_scale;
        I.ncells = inj.np ? inj.ncells : 0;
        SampleArgs S{};
        S.field = field;
        S.ci = smp.ci;
        S.w = smp.w;
        S.out = smp.series + row * smp.np;
        S.pitch = p.pitch;
        S.plane = p.plane;
        S.np = static_cast<int>(smp.np);
        const int threads = static_cast<int>(
            std::min<int64_t>(1024, std::max<int64_t>(32, (std::max<int64_t>(I.ncells, smp.np) + 31) / 32 * 32)));
        if (p.ndim == 3)
            inject_sample_kernel<3><<<1, threads, 0, p.stream>>>(I, S);
        else
            inject_sample_kernel<2><<<1, threads, 0, p.stream>>>(I, S);
        return;
    }
    launch_inject(p, inj, field, row);
    launch_sample(p, smp, field, row);
}

bool fused_sparse_active(const Plan& p);

int64_t launches_per_step_of(const Plan& p) {
    if (p.kind == Plan::DIFFUSION) return 1;  // per step without temporal blocking
    if (p.nccl_comm && p.overlap) return 6;  // 3 stencil ranges, 2 injections, sampling
    if (p.nccl_comm && (p.has_lower || p.has_upper)) return 3;
    if (fused_sparse_active(p)) return 1;  // + one sampling launch per step range
    const PointSet& inj = p.ac.forward ? p.src : p.rec;
    const PointSet& smp = p.ac.forward ? p.rec : p.src;
    return (inj.ncells <= kFusedSparseMax && smp.np <= kFusedSparseMax) ? 2 : 3;
}

// One step of the reference time loop. Step k maps to t = k (forward) or
// t = nt - k (adjoint); slot aliases as in codegen.cpp:336-354.
struct StepSlots {
    float* out;
    float* cur;
    float* prev;
    int64_t row;  // sparse series row of this step
};

StepSlots step_slots(const Plan& p, int64_t k, float* const* u) {
    if (p.ac.forward) {
        const int64_t t = k;
        return {u[(t + 1) % 3], u[t % 3], u[(t + 2) % 3], t};
    }
    const int64_t t = p.nt - k;
    return {u[(t + 2) % 3], u[t % 3], u[(t + 1) % 3], t - 1};
}

// The vector ring kernel carries the sparse work of single-domain 3D plans
// when every injection cell lies in its tile grid (ensure_fused).
bool fused_sparse_active(const Plan& p) {
    return p.fused.ok && !p.fused_disabled && (p.kind == Plan::ACOUSTIC || p.kind == Plan::FWI) &&
           p.ndim == 3 && p.use_vec && !p.use_vecq && !p.slab && !p.nccl_comm;
}

// [first, last): the step range being enqueued (fused sampling lags one step)
void enqueue_acoustic_step(Plan& p, int64_t k, float* const* u, bool stencil_only = false,
                           int64_t first = 0, int64_t last = -1) {
    const StepSlots st = step_slots(p, k, u);
    const PointSet& inj = p.ac.forward ? p.src : p.rec;
    const PointSet& smp = p.ac.forward ? p.rec : p.src;
    if (p.nccl_comm && p.overlap && !stencil_only) {
        // boundary bands + their injection -> exchange on the comm stream
        // while the inner planes are updated and injected
        launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &p.zr_lo);
        launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &p.zr_hi);
        launch_inject(p, inj, st.out, st.row, 0, inj.nband0);
        SF_CUDA(cudaEventRecord(p.ev_band, p.stream));
        SF_CUDA(cudaStreamWaitEvent(p.comm, p.ev_band, 0));
        {
            Plan& q = p;
            std::swap(q.stream, q.comm);  // exchange enqueued on the comm stream
            try {
                launch_exchange_nccl(q, st.out);
            } catch (...) {
                std::swap(q.stream, q.comm);
                throw;
            }
            std::swap(q.stream, q.comm);
        }
        SF_CUDA(cudaEventRecord(p.ev_comm, p.comm));
        launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &p.zr_in);
        launch_inject(p, inj, st.out, st.row, inj.nband0, inj.ncells - inj.nband0);
        SF_CUDA(cudaStreamWaitEvent(p.stream, p.ev_comm, 0));
        launch_sample(p, smp, st.out, st.row);
        return;
    }
    if (!stencil_only && fused_sparse_active(p)) {
        // one launch per step: injection of this step in the CTAs' epilogue,
        // sampling of the previous step (k > first) from this step's cur
        Epilogue epi;
        epi.inj = &inj;
        epi.inj_row = st.row;
        if (k > first) {
            epi.smp = &smp;
            epi.smp_row = p.ac.forward ? st.row - 1 : st.row + 1;
        }
        launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, nullptr, &epi);
        if (k + 1 == last) launch_sample(p, smp, st.out, st.row);
        return;
    }
    launch_stencil(p, st.out, st.cur, st.prev);
    if (stencil_only) return;
    if (p.nccl_comm && (p.has_lower || p.has_upper)) {
        launch_inject(p, inj, st.out, st.row);
        launch_exchange_nccl(p, st.out);
        launch_sample(p, smp, st.out, st.row);
        return;
    }
    launch_inject_sample(p, inj, smp, st.out, st.row);
}

// In-process chain of slab plans (one host thread; plans on one or several
// devices): per step every slab runs stencil + injection, copies its
// boundary planes into its neighbours' halos on its own stream, and samples
// once the neighbours' copies into its halos are done. Ordering across
// streams uses one event per plan (recorded after its copies).
void chain_step(sf_plan* const* P, int n, int64_t k) {
    const int r = P[0]->ac.radius;
    for (int i = 0; i < n; ++i) {
        Plan& p = *P[i];
        SF_CUDA(cudaSetDevice(p.device));
        if (k > 0) {  // neighbours' halo copies of the previous step landed
            if (i > 0) SF_CUDA(cudaStreamWaitEvent(p.stream, P[i - 1]->ev_copy, 0));
            if (i + 1 < n) SF_CUDA(cudaStreamWaitEvent(p.stream, P[i + 1]->ev_copy, 0));
        }
        const StepSlots st = step_slots(p, k, p.slot);
        const PointSet& inj = p.ac.forward ? p.src : p.rec;
        if (p.overlap) {  // same split as the NCCL path: bands, copies, then inner planes
            launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &p.zr_lo);
            launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &p.zr_hi);
            launch_inject(p, inj, st.out, st.row, 0, inj.nband0);
        } else {
            launch_stencil(p, st.out, st.cur, st.prev);
            launch_inject(p, inj, st.out, st.row);
        }
        const size_t bytes = static_cast<size_t>(r) * p.plane * sizeof(float);
        if (i > 0) {
            Plan& q = *P[i - 1];
            const StepSlots sq = step_slots(q, k, q.slot);
            SF_CUDA(cudaMemcpyPeerAsync(sq.out + static_cast<int64_t>(q.own_hi) * q.plane, q.device,
                                        st.out + static_cast<int64_t>(p.own_lo) * p.plane,
                                        p.device, bytes, p.stream));
        }
        if (i + 1 < n) {
            Plan& q = *P[i + 1];
            const StepSlots sq = step_slots(q, k, q.slot);
            SF_CUDA(cudaMemcpyPeerAsync(sq.out + static_cast<int64_t>(q.own_lo - r) * q.plane,
                                        q.device,
                                        st.out + static_cast<int64_t>(p.own_hi - r) * p.plane,
                                        p.device, bytes, p.stream));
        }
        SF_CUDA(cudaEventRecord(p.ev_copy, p.stream));
        if (p.overlap) {
            launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &p.zr_in);
            launch_inject(p, inj, st.out, st.row, inj.nband0, inj.ncells - inj.nband0);
        }
    }
    for (int i = 0; i < n; ++i) {
        Plan& p = *P[i];
        SF_CUDA(cudaSetDevice(p.device));
        if (i > 0) SF_CUDA(cudaStreamWaitEvent(p.stream, P[i - 1]->ev_copy, 0));
        if (i + 1 < n) SF_CUDA(cudaStreamWaitEvent(p.stream, P[i + 1]->ev_copy, 0));
        const StepSlots st = step_slots(p, k, p.slot);
        launch_sample(p, p.ac.forward ? p.rec : p.src, st.out, st.row);
    }
}

void enqueue_diffusion_step(Plan& p, int64_t t) {
    DiffusionArgs A{};
    A.cur = p.slot[t % 2];
    A.out = p.slot[(t + 1) % 2];
    A.pitch = p.pitch;
    A.n0 = static_cast<int>(p.n[0]);
    A.n1 = static_cast<int>(p.n[1]);
    A.c0 = p.dc.c0;
    A.has_c0 = p.dc.has_c0;
    for (int j = 0; j < 8; ++j) A.cj[j] = p.dc.cj[j];
    dim3 b(64, 4);
    dim3 g(static_cast<unsigned>((p.n[1] + 63) / 64), static_cast<unsigned>((p.n[0] + 3) / 4));
    launch_diffusion_r(p.dc.radius, g, b, p.stream, A);
}

// Temporally blocked diffusion (diffusion_tb_kernel): TMAX = 8/R steps per
// launch on 64x64 tiles, (64 + 16)^2-float ping-pong buffers.
constexpr int kTbTile = 64;

template <int R, int TILE, int RV = 1>
void launch_diffusion_tb_t(dim3 g, cudaStream_t st, const DiffusionTBArgs& A) {
    constexpr int TMAX = 8 / R > 0 ? 8 / R : 1;
    using L = TbLayout<R, TILE, TMAX>;
    // function attributes are per device: remember which devices have it
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    SF_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(done.load() & bit)) {
        SF_CUDA(cudaFuncSetAttribute(&diffusion_tb_kernel<R, TILE, TMAX, RV>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(L::smem)));
        done.fetch_or(bit);
    }
    diffusion_tb_kernel<R, TILE, TMAX, RV><<<g, 256, L::smem, st>>>(A);
}

int diffusion_box(int r, int tile = kTbTile) {
    const int tmax = 8 / r > 0 ? 8 / r : 1;
    return tile + 2 * ((tmax * r + 3) / 4 * 4);
}

void make_map_2d(CUtensorMap* map, const Plan& p, const float* base, uint32_t box) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.n[1]), static_cast<cuuint64_t>(p.n[0])};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.pitch) * 4};
    cuuint32_t bx[2] = {box, box};
    cuuint32_t es[2] = {1, 1};
    CUresult r = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                      const_cast<float*>(base), dims, strides, bx, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Status(SF_ERR_CUDA, "cuTensorMapEncodeTiled (2D) failed: " + std::to_string(r));
}

int diffusion_tmax(int r) { return 8 / r > 0 ? 8 / r : 1; }

void launch_diffusion_tb(int r, int tile, int rv, dim3 g, cudaStream_t st,
                         const DiffusionTBArgs& A) {
    if (r == 1) {
        if (rv == 2 && tile == kTbTile) return launch_diffusion_tb_t<1, kTbTile, 2>(g, st, A);
        switch (tile) {
            case 48: return launch_diffusion_tb_t<1, 48>(g, st, A);
            case 56: return launch_diffusion_tb_t<1, 56>(g, st, A);
            case 72: return launch_diffusion_tb_t<1, 72>(g, st, A);
            case 80: return launch_diffusion_tb_t<1, 80>(g, st, A);
            case 96: return launch_diffusion_tb_t<1, 96>(g, st, A);
            default: return launch_diffusion_tb_t<1, kTbTile>(g, st, A);
        }
    }
    switch (r) {
        case 2: return launch_diffusion_tb_t<2, kTbTile>(g, st, A);
        case 3: return launch_diffusion_tb_t<3, kTbTile>(g, st, A);
        case 4: return launch_diffusion_tb_t<4, kTbTile>(g, st, A);
        case 5: return launch_diffusion_tb_t<5, kTbTile>(g, st, A);
        case 6: return launch_diffusion_tb_t<6, kTbTile>(g, st, A);
        case 7: return launch_diffusion_tb_t<7, kTbTile>(g, st, A);
        case 8: return launch_diffusion_tb_t<8, kTbTile>(g, st, A);
        default: throw Status(SF_ERR_INVALID, "radius out of range");
    }
}

// Steps [b, e): copy both slots into the scratch pair (boundary values),
// then alternate read/write pairs launch by launch; the final pair is copied
// back into the slots if it is the scratch one.
void enqueue_diffusion_tb(Plan& p, int64_t b, int64_t e) {
    const size_t bytes = sizeof(float) * p.slot_elems;
    for (int s = 0; s < 2; ++s)
        SF_CUDA(cudaMemcpyAsync(p.dscratch[s], p.slot[s], bytes, cudaMemcpyDeviceToDevice, p.stream));
    float* X[2] = {p.slot[0], p.slot[1]};
    float* Y[2] = {p.dscratch[0], p.dscratch[1]};
    const int tmax = diffusion_tmax(p.dc.radius);
    dim3 g(static_cast<unsigned>((p.n[1] + p.tb_tile - 1) / p.tb_tile),
           static_cast<unsigned>((p.n[0] + p.tb_tile - 1) / p.tb_tile));
    bool in_x = true;
    for (int64_t t = b; t < e;) {
        const int T = static_cast<int>(std::min<int64_t>(tmax, e - t));
        DiffusionTBArgs A;
        std::memset(&A, 0, sizeof A);
        float* const* wr = in_x ? Y : X;
        A.src0 = in_x ? p.tm_dx[0] : p.tm_dy[0];
        A.src1 = in_x ? p.tm_dx[1] : p.tm_dy[1];
        A.dst[0] = wr[0];
        A.dst[1] = wr[1];
        A.pitch = p.pitch;
        A.n0 = static_cast<int>(p.n[0]);
        A.n1 = static_cast<int>(p.n[1]);
        A.t0 = static_cast<int>(t);
        A.T = T;
        A.c0 = p.dc.c0;
        A.has_c0 = p.dc.has_c0;
        for (int j = 0; j < 8; ++j) A.cj[j] = p.dc.cj[j];
        launch_diffusion_tb(p.dc.radius, p.tb_tile, p.tb_rv, g, p.stream, A);
        in_x = !in_x;
        t += T;
    }
    if (!in_x)
        for (int s = 0; s < 2; ++s)
            SF_CUDA(cudaMemcpyAsync(p.slot[s], p.dscratch[s], bytes, cudaMemcpyDeviceToDevice,
                                    p.stream));
}

int64_t diffusion_launches(const Plan& p, int64_t steps) {
    if (!p.diffusion_tb) return steps;
    const int64_t tmax = diffusion_tmax(p.dc.radius);
    return (steps + tmax - 1) / tmax;
}

// FWI phases (config 5): forward into the HBM history, then the adjoint
// sweep with the delayed gradient term fused into the stencil.
void enqueue_fwi_forward(Plan& p) {
    p.ac = p.ac_fwd;
    const int64_t L = p.slot_elems;
    SF_CUDA(cudaMemsetAsync(p.hist, 0, sizeof(float) * 2 * L, p.stream));
    const bool fused = fused_sparse_active(p);
    for (int64_t t = 0; t < p.nt; ++t) {
        float* out = p.hist + (t + 2) * L;
        if (fused) {  // injection of step t, sampling of step t-1 in the epilogue
            Epilogue epi;
            epi.inj = &p.src;
            epi.inj_row = t;
            if (t > 0) {
                epi.smp = &p.rec;
                epi.smp_row = t - 1;
            }
            launch_stencil(p, out, p.hist + (t + 1) * L, p.hist + t * L, nullptr, nullptr, nullptr,
                           &epi);
            if (t + 1 == p.nt) launch_sample(p, p.rec, out, t);
            continue;
        }
        launch_stencil(p, out, p.hist + (t + 1) * L, p.hist + t * L);
        launch_inject_sample(p, p.src, p.rec, out, t);
    }
}

void enqueue_fwi_adjoint(Plan& p) {
    p.ac = p.ac_adj;  // adjoint term order and direction (acoustic.cpp:187-198)
    const int64_t L = p.slot_elems;
    for (int s = 0; s < 3; ++s) SF_CUDA(cudaMemsetAsync(p.v[s], 0, sizeof(float) * L, p.stream));
    SF_CUDA(cudaMemsetAsync(p.grad, 0, sizeof(float) * L, p.stream));
    // the gradient kernel (t < nt) carries the residual injection of its step
    // and the source sampling of the step before in its epilogue when the
    // tile-sorted CSR exists; the first step (no gradient term) does not
    const bool fused = p.fused_adj.ok && !p.fused_disabled;
    for (int64_t t = p.nt; t >= 1; --t) {
        float* out = p.v[(t + 2) % 3];
        const float* cur = p.v[t % 3];
        const float* prev = p.v[(t + 1) % 3];
        if (t <= p.nt - 1) {  // term for time t+1: v(t+2) is still in `out`
            if (fused) {
                Epilogue epi;
                epi.inj = &p.rec;
                epi.inj_row = t - 1;
                if (t <= p.nt - 2) {  // step t+1 sampled row t; step nt sampled itself
                    epi.smp = &p.src;
                    epi.smp_row = t;
                }
                launch_stencil(p, out, cur, prev, p.grad, p.hist + (t + 2) * L, nullptr, &epi);
                if (t == 1) launch_sample(p, p.src, out, 0);
                continue;
            }
            launch_stencil(p, out, cur, prev, p.grad, p.hist + (t + 2) * L);
        } else {
            launch_stencil(p, out, cur, prev);
        }
        launch_inject_sample(p, p.rec, p.src, out, t - 1);
    }
    if (p.nt >= 1) {  // term for time 1
        dim3 b(128);
        dim3 g(static_cast<unsigned>((p.n[2] + 127) / 128), static_cast<unsigned>(p.n[1]),
               static_cast<unsigned>(p.n[0]));
        grad_final_kernel<<<g, b, 0, p.stream>>>(p.grad, p.hist + 2 * L, p.v[2 % 3], p.v[1 % 3],
                                                 p.v[0], p.ac.cm, p.pitch, p.plane,
                                                 static_cast<int>(p.n[0]),
                                                 static_cast<int>(p.n[1]),
                                                 static_cast<int>(p.n[2]), p.ac.radius);
    }
    p.ac = p.ac_fwd;
}

// graph keys: [b, e) step ranges; negative keys for special sequences
constexpr int64_t kStencilOnly = -1, kFwiForward = -2, kFwiAdjoint = -3;

void enqueue_steps(Plan& p, int64_t b, int64_t e) {
    if (b == kStencilOnly) {
        if (p.kind == Plan::DIFFUSION && p.diffusion_tb) return enqueue_diffusion_tb(p, 0, p.nt);
        for (int64_t k = 0; k < p.nt; ++k) {
            if (p.kind == Plan::DIFFUSION)
                enqueue_diffusion_step(p, k);
            else
                enqueue_acoustic_step(p, k, p.slot, true);
        }
        return;
    }
    if (b == kFwiForward) return enqueue_fwi_forward(p);
    if (b == kFwiAdjoint) return enqueue_fwi_adjoint(p);
    if (p.kind == Plan::DIFFUSION && p.diffusion_tb) return enqueue_diffusion_tb(p, b, e);
    for (int64_t k = b; k < e; ++k) {
        if (p.kind == Plan::DIFFUSION)
            enqueue_diffusion_step(p, k);
        else
            enqueue_acoustic_step(p, k, p.slot, false, b, e);
    }
}

// Tile-sorted copy of the injection CSR for the fused epilogue: cells of
// CTA b (launch order) in [tile_start[b], tile_start[b+1]), each cell's
// contributions still in ascending point order. Rebuilt when the points or
// the tile geometry change; not built (fused path off) when a cell lies
// outside the planes / tiles the stencil kernel covers.
// Build (or keep) one tile-sorted CSR: `inj`'s cells grouped by the CTA of
// the launch geometry (grid, zchunk, tx x ty tiles over planes [z0, z1)).
void build_fused(Plan& p, sf_plan::FusedSparse& f, const PointSet& inj, dim3 grid, int zchunk,
                 int64_t tx, int64_t ty) {
    const uint64_t key[8] = {inj.version + 1, grid.x, grid.y, grid.z,
                             static_cast<uint64_t>(zchunk), static_cast<uint64_t>(tx),
                             static_cast<uint64_t>(ty),
                             (static_cast<uint64_t>(p.z0) << 32) | static_cast<uint32_t>(p.z1)};
    if (std::memcmp(key, f.key, sizeof key) == 0) return;
    std::memcpy(f.key, key, sizeof key);
    clear_graphs(p);
    f.ok = false;
    const int64_t gx = grid.x, gy = grid.y, gz = grid.z;
    const int64_t ntiles = gx * gy * gz;
    const int nc = inj.ncells;
    std::vector<int64_t> tile(static_cast<size_t>(nc));
    for (int i = 0; i < nc; ++i) {
        const int64_t off = inj.h_cells[i];
        const int64_t a0 = off / p.plane, a1 = (off % p.plane) / p.pitch, a2 = off % p.pitch;
        if (a0 < p.z0 || a0 >= p.z1 || a2 >= gx * tx || a1 >= gy * ty) return;
        tile[i] = a2 / tx + gx * (a1 / ty + gy * ((a0 - p.z0) / zchunk));
        if (tile[i] >= ntiles) return;
    }
    std::vector<int> order(static_cast<size_t>(nc));
    for (int i = 0; i < nc; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tile[a] < tile[b]; });
    std::vector<int> tstart(static_cast<size_t>(ntiles + 1), 0);
    std::vector<int64_t> cell;
    std::vector<int> start, cp;
    std::vector<float> cw;
    for (int i = 0; i < nc; ++i) ++tstart[tile[i] + 1];
    // dense point sets (e.g. a full receiver grid injecting residuals) would
    // pile thousands of cells onto the few CTAs of one z-chunk, serialised in
    // their epilogue: a grid-wide injection kernel is faster there (measured,
    // C5 adjoint +5 %). Fuse only while every CTA has at most one cell per
    // consumer thread.
    for (int64_t t = 0; t < ntiles; ++t)
        if (tstart[t + 1] > 128) return;
    for (int64_t t = 0; t < ntiles; ++t) tstart[t + 1] += tstart[t];
    for (int oi : order) {
        cell.push_back(inj.h_cells[oi]);
        start.push_back(static_cast<int>(cp.size()));
        for (int j = inj.h_start[oi]; j < inj.h_start[oi + 1]; ++j) {
            cp.push_back(inj.h_cp[j]);
            cw.push_back(inj.h_cw[j]);
        }
    }
    start.push_back(static_cast<int>(cp.size()));
    if (cell.empty()) cell.push_back(0);
    if (cp.empty()) {
        cp.push_back(0);
        cw.push_back(0.0f);
    }
    if (static_cast<size_t>(ntiles + 1) > f.cap_tiles) {
        dfree(f.tile_start);
        f.cap_tiles = static_cast<size_t>(ntiles + 1);
        f.tile_start = dalloc<int>(f.cap_tiles);
    }
    if (cell.size() > f.cap_cells) {
        dfree(f.cell);
        dfree(f.start);
        f.cap_cells = cell.size();
        f.cell = dalloc<int64_t>(f.cap_cells);
        f.start = dalloc<int>(f.cap_cells + 1);
    }
    if (cp.size() > f.cap_contrib) {
        dfree(f.cp);
        dfree(f.cw);
        f.cap_contrib = cp.size();
        f.cp = dalloc<int>(f.cap_contrib);
        f.cw = dalloc<float>(f.cap_contrib);
    }
    SF_CUDA(cudaStreamSynchronize(p.stream));
    SF_CUDA(cudaMemcpy(f.tile_start, tstart.data(), tstart.size() * sizeof(int), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(f.cell, cell.data(), cell.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(f.start, start.data(), start.size() * sizeof(int), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(f.cp, cp.data(), cp.size() * sizeof(int), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMemcpy(f.cw, cw.data(), cw.size() * sizeof(float), cudaMemcpyHostToDevice));
    f.ok = true;
}

// Tile-sorted copies of the injection CSR for the fused epilogue: cells of
// CTA b (launch order) in [tile_start[b], tile_start[b+1]), each cell's
// contributions still in ascending point order. Rebuilt when the points or
// the tile geometry change; not built (fused path off) when a cell lies
// outside the planes / tiles the stencil kernel covers.
void ensure_fused(Plan& p) {
    // FWI: the forward sweep (p.ac is the forward set outside the adjoint)
    if (p.fused_disabled || (p.kind != Plan::ACOUSTIC && p.kind != Plan::FWI) || p.ndim != 3 ||
        !p.use_vec || p.use_vecq || p.slab || p.nccl_comm) {
        p.fused.ok = false;
        p.fused_adj.ok = false;
        return;
    }
    const PointSet& inj = p.ac.forward ? p.src : p.rec;
    build_fused(p, p.fused, inj, p.grid3, p.zchunk, 32 * p.tile_nx,
                4 * p.vec_warps * p.vec_rpl / p.tile_nx);
    if (p.kind == Plan::FWI)  // adjoint + gradient kernel: 64 x 8 tiles, rec injects
        build_fused(p, p.fused_adj, p.rec, p.grid_grad, p.zchunk_grad, 64, 8);
}

// eta0 bits for one tile shape (see TmaStencilArgs::eta0): recomputed on the
// plan stream when eta was rewritten or the tile shape changed; a new buffer
// drops the cached graphs (they hold the pointer).
// Sizes the flag words for the tile geometry; returns the number of 32-plane
// groups. launch_eta_flags then fills groups [word0, word0 + nwords).
int prepare_eta_flags(Plan& p, sf_plan::EtaFlags& f, int tx, int ty) {
    const int n0 = static_cast<int>(p.n[0]), n1 = static_cast<int>(p.n[1]),
              n2 = static_cast<int>(p.n[2]);
    const int ntx = (n2 + tx - 1) / tx, nty = (n1 + ty - 1) / ty, words = (n0 + 31) / 32;
    const size_t need = static_cast<size_t>(ntx) * nty * words;
    if (need > f.cap) {
        clear_graphs(p);
        SF_CUDA(cudaStreamSynchronize(p.stream));
        dfree(f.bits);
        f.bits = dalloc<uint32_t>(need);
        f.cap = need;
    }
    if (f.tx != tx || f.ty != ty) clear_graphs(p);
    f.tx = tx;
    f.ty = ty;
    f.ntx = ntx;
    f.nty = nty;
    f.words = words;
    return words;
}

void launch_eta_flags(Plan& p, sf_plan::EtaFlags& f, int word0, int nwords) {
    if (nwords <= 0) return;
    eta_zero_flags_kernel<<<dim3(static_cast<unsigned>(f.ntx * f.nty), static_cast<unsigned>(nwords)),
                            256, 0, p.stream>>>(p.eta, p.pitch, p.plane, static_cast<int>(p.n[0]),
                                                static_cast<int>(p.n[1]), static_cast<int>(p.n[2]),
                                                f.tx, f.ty, f.ntx, f.words, f.bits, word0);
    SF_CUDA(cudaGetLastError());
}

void compute_eta_flags(Plan& p, sf_plan::EtaFlags& f, int tx, int ty) {
    if (f.gen == p.eta_gen && f.tx == tx && f.ty == ty) return;
    const int words = prepare_eta_flags(p, f, tx, ty);
    launch_eta_flags(p, f, 0, words);
    f.gen = p.eta_gen;
}

bool eta_flags_wanted(const Plan& p) {
    return !(p.eta_skip_disabled || p.ndim != 3 || !p.eta || !(p.use_vec || p.use_vecq)) &&
           (p.kind == Plan::ACOUSTIC || p.kind == Plan::FWI);
}

void eta_flag_tile(const Plan& p, int* tx, int* ty) {
    *tx = p.use_vecq ? 64 : 32 * p.tile_nx;
    *ty = p.use_vecq ? 2 * p.vec_warps : 4 * p.vec_warps * p.vec_rpl / p.tile_nx;
}

void ensure_eta_flags(Plan& p) {
    if (!eta_flags_wanted(p)) return;
    int tx, ty;
    eta_flag_tile(p, &tx, &ty);
    compute_eta_flags(p, p.eta0, tx, ty);
    if (p.kind == Plan::FWI) compute_eta_flags(p, p.eta0_grad, 64, 8);
}

// Steps [b, e) as one cached CUDA graph (the OpenMP team + barriers of the
// generated loop become graph edges; launches cost ~graph-node latency).
void run_steps(Plan& p, int64_t b, int64_t e) {
    if (b >= e && b >= 0) return;
    if (b >= 0 || b == kFwiForward || b == kFwiAdjoint) ensure_fused(p);
    ensure_eta_flags(p);
    auto key = std::make_pair(b, e);
    auto it = p.graphs.find(key);
    if (it == p.graphs.end()) {
        NvtxRange cap("capture time loop into a CUDA graph");
        cudaGraph_t g = nullptr;
        SF_CUDA(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_steps(p, b, e);
        } catch (...) {
            cudaStreamEndCapture(p.stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        SF_CUDA(cudaStreamEndCapture(p.stream, &g));
        cudaGraphExec_t ge = nullptr;
        SF_CUDA(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        it = p.graphs.emplace(key, ge).first;
    }
    SF_CUDA(cudaGraphLaunch(it->second, p.stream));
}

int max_tile_nx(int r) { return r <= 4 ? 4 : 2; }

// Grid for the chosen tile: tiles over (a2, a1) and chunks over a0. The
// chunk count is picked with a small cost model: CTAs run in waves of
// (#SM x resident CTAs/SM), each CTA costs its chunk length plus the 2R-plane
// queue warm-up, so minimise waves(gz) * (chunk(gz) + 2R) over the chunkings
// that put at least one full wave on the machine.
// Chunking cost model for one kernel shape (tile wx x wy, resident CTAs/SM).
void chunk_grid(const Plan& p, int64_t wx, int64_t wy, int per_sm, dim3* grid, int* zchunk,
                int64_t nz = -1) {
    const int r = p.ac.radius;
    const int64_t gx = (p.n[2] + wx - 1) / wx, gy = (p.n[1] + wy - 1) / wy;
    if (nz < 0) nz = p.z1 - p.z0;
    if (nz < 1) nz = 1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
    if (per_sm < 1) per_sm = 1;
    const int64_t slots = static_cast<int64_t>(sms) * per_sm;
    double best_cost = 1e30;
    int64_t best_gz = 1;
    for (int64_t gz = 1; gz <= nz; ++gz) {
        const int64_t zc = (nz + gz - 1) / gz;
        if (gz > 1 && zc < std::min<int64_t>(nz, 2 * r + 6)) break;
        if (gx * gy * gz < slots && (nz + gz) / (gz + 1) >= 2 * r + 6) continue;  // fill every SM
        const int64_t waves = (gx * gy * gz + slots - 1) / slots;
        const double cost = static_cast<double>(waves) * static_cast<double>(zc + 2 * r);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best_gz = gz;
        }
    }
    if (const char* env = std::getenv("SF_ZCHUNKS")) {  // experiments: force the chunk count
        const int64_t v = std::atoll(env);
        if (v >= 1 && v <= nz) best_gz = v;
    }
    const int64_t zc = (nz + best_gz - 1) / best_gz;
    *zchunk = static_cast<int>(zc);
    *grid = dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy),
                 static_cast<unsigned>((nz + zc - 1) / zc));
}

void set_grid(Plan& p) {
    const int r = p.ac.radius;
    const int64_t wx = p.use_vecq ? 64 : 32 * p.tile_nx;
    const int64_t wy = p.use_vecq ? 2 * p.vec_warps
                       : p.use_vec ? 4 * p.vec_warps * p.vec_rpl / p.tile_nx
                                   : p.tile_ty;
    int per_sm = 0;
    if (p.use_vecq) {
        const void* fn = p.ac.forward ? vecq_ptr<true>(r, p.vec_warps, p.vecq_ring)
                                      : vecq_ptr<false>(r, p.vec_warps, p.vecq_ring);
        if (fn)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * p.vec_warps, p.tma_smem);
    } else if (p.use_vec) {
        const void* fn = p.ac.forward ? vec_ptr<true>(r, p.vec_warps, p.tile_nx, p.vec_kernel_rpl())
                                      : vec_ptr<false>(r, p.vec_warps, p.tile_nx, p.vec_kernel_rpl());
        if (fn)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * (p.vec_warps + 1),
                                                          p.tma_smem);
    } else if (p.use_tma) {
        const void* fn = p.ac.forward ? tma_ptr<true>(r, p.tile_nx) : tma_ptr<false>(r, p.tile_nx);
        if (fn) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, p.tma_smem);
    } else {
        const void* fn = p.ac.forward ? acoustic3d_ptr<true, false>(r, p.tile_nx, p.tile_ty)
                                      : acoustic3d_ptr<false, false>(r, p.tile_nx, p.tile_ty);
        if (fn) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * p.tile_ty, 0);
    }
    p.resident = per_sm;
    chunk_grid(p, wx, wy, per_sm, &p.grid3, &p.zchunk);
    if (p.slab) {
        // exchange overlap: boundary bands first, inner planes while the
        // halos are in flight (needs at least 2r owned interior planes)
        const int own0 = std::max(p.own_lo, p.z0), own1 = std::min(p.own_hi, p.z1);
        p.overlap = !p.overlap_disabled && (p.has_lower || p.has_upper) && own1 - own0 >= 2 * r + 1;
        if (p.overlap) {
            auto setr = [&](sf_plan::ZRange& z, int a, int b) {
                z.z0 = a;
                z.z1 = b;
                if (b > a) chunk_grid(p, wx, wy, per_sm, &z.grid, &z.zchunk, b - a);
            };
            const int lo_end = p.has_lower ? own0 + r : own0;
            const int hi_beg = p.has_upper ? own1 - r : own1;
            setr(p.zr_lo, own0, lo_end);
            setr(p.zr_hi, hi_beg, own1);
            setr(p.zr_in, lo_end, hi_beg);
        }
    }
    if (p.kind == Plan::FWI && p.use_vec && !p.use_vecq) {
        int g = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g, vec_grad_ptr(r), 160, p.smem_grad);
        chunk_grid(p, 64, 8, g, &p.grid_grad, &p.zchunk_grad);
    }
}

// Default tile: the NX <= max that wastes the fewest lanes on the a2 extent
// (281 -> NX 3: three 96-wide tiles cover 288), TY 8. SF_TILE="nx,ty"
// overrides (autotuning experiments).
void choose_geometry(Plan& p) {
    if (p.kind == Plan::DIFFUSION || p.ndim == 2) return;
    const int r = p.ac.radius;
    int best = 1;
    int64_t best_cover = INT64_MAX;
    for (int k = 1; k <= max_tile_nx(r); ++k) {
        const int64_t w = 32 * k;
        const int64_t cover = (p.n[2] + w - 1) / w * w;
        if (cover <= best_cover) {
            best_cover = cover;
            best = k;
        }
    }
    p.tile_nx = best;
    p.tile_ty = 8;
    if (const char* env = std::getenv("SF_TILE")) {
        int nx = 0, ty = 0;
        if (std::sscanf(env, "%d,%d", &nx, &ty) == 2 && nx >= 1 && nx <= max_tile_nx(r) &&
            (ty == 8 || ty == 16)) {
            p.tile_nx = nx;
            p.tile_ty = ty;
        }
    }
    set_grid(p);
}

// Switch a 3D plan to a TMA pipeline once its slots exist.
//
// Radius <= 4 (space order <= 8): the vectorised TMA kernel (4 points per
// thread, LDS.128 neighbours). Measured per launch on B200 against the
// scalar TMA kernel / per-thread-load kernel: c2 order 4 81.0 vs 86.6 vs
// 111 us; c3 order 4 412 vs 505 vs 555 us; order 6 484 vs 584 vs 605 us;
// order 8 533 (8 warps) vs 851 vs 708 us. 4-warp CTAs for radius <= 3,
// 8-warp CTAs at radius 4. Above radius 4 the ring no longer fits next to a
// useful occupancy: the queue-vector kernel keeps the a0 neighbours in
// registers (c3 order 12: 677 vs 891 us; order 16: 837 vs 1027 us for the
// per-thread-load kernel; 4-warp CTAs, 3 stages). Overrides: SF_VEC=0 /
// SF_VECQ=0 (scalar paths), SF_VEC_WARPS, SF_TMA=1 (scalar TMA at any order),
// SF_NO_TMA=1 (per-thread loads only).
void enable_tma(Plan& p) {
    if (p.ndim != 3) return;
    if (const char* env = std::getenv("SF_NO_FUSED_SPARSE")) p.fused_disabled = env[0] == '1';
    if (const char* env = std::getenv("SF_NO_ETA_SKIP")) p.eta_skip_disabled = env[0] == '1';
    {  // queue-vector stencil with the shared-memory core ring (vecq2), opt-in with
       // SF_VECQ2=1: 122 instead of 160 registers at radius 8 (4 CTAs per SM), but
       // the extra LDS.128 of the future planes make the LSU a second bottleneck:
       // sustained order 12 747 vs 692 us, order 16 798 vs 768 us per step
        const char* e = std::getenv("SF_VECQ2");
        p.vecq_ring = e && e[0] == '1' ? 1 : 0;
        if (const char* f = std::getenv("SF_VECQ_FORM")) {  // queue kernel form (A/B)
            if (std::strcmp(f, "free") == 0) p.vecq_ring = 2;
            if (std::strcmp(f, "pinned") == 0) p.vecq_ring = 3;
            if (std::strcmp(f, "tmem") == 0) p.vecq_ring = 4;
            if (std::strcmp(f, "last") == 0) p.vecq_ring = 5;  // decoupled, last warp out refills
        }
    }
    if (const char* env = std::getenv("SF_NO_TMA"))
        if (env[0] == '1') return;
    const char* vec = std::getenv("SF_VEC");
    const bool vec_on = !(vec && vec[0] == '0');
    const char* vq = std::getenv("SF_VECQ");
    if (vec_on && p.ac.radius <= 4) {
        p.use_vec = true;
        // FWI: the forward runs the same tile choice as a plain forward plan;
        // the 4-warp gradient kernel has its own maps (setup_tma)
        p.vec_warps = p.ac.radius <= 3 ? 4 : 8;
        if (p.ac.radius == 4 && p.kind != Plan::FWI) {
            // 64 x 32 tiles (16 consumer warps, one CTA per SM): the cur box
            // carries 1.41x instead of 1.69x its points, so less L2 and
            // shared-memory traffic per point -- C4 3878 vs 3966 us, C3
            // order 8 502 vs 508 us per step (interleaved A/B) -- where the
            // taller tiles do not pad the a1 extent by more than ~3 %
            const int64_t n1 = p.n[1] - 4;
            const int64_t pad16 = (n1 + 15) / 16 * 16, pad32 = (n1 + 31) / 32 * 32;
            if (pad32 * 100 <= pad16 * 103) p.vec_warps = 16;
        }
        if (const char* w = std::getenv("SF_VEC_WARPS")) {
            const int v = std::atoi(w);
            p.vec_warps = v == 4 ? 4 : v == 16 && p.ac.radius == 4 ? 16 : 8;
        }
        // tile width: 64 (16 lanes per row) unless 32-wide 4-warp tiles
        // cover the interior with fewer padded points (FWI: 64 wide, one set
        // of maps serves the forward and gradient kernels)
        p.tile_nx = 2;
        if (const char* e = std::getenv("SF_VEC_AQ8")) p.vec_aq8 = std::atoi(e) != 0;
        if (p.kind != Plan::FWI) {
            const int r = p.ac.radius;
            auto cover = [&](int nx, int warps) {
                const int64_t tx = 32 * nx, ty = 4 * warps / nx;
                return ((p.n[2] - r + tx - 1) / tx * tx) * ((p.n[1] - r + ty - 1) / ty * ty);
            };
            if (cover(1, 4) < cover(2, p.vec_warps)) {
                p.tile_nx = 1;
                p.vec_warps = 4;
            }
            if (const char* e = std::getenv("SF_VEC_NX")) {
                p.tile_nx = std::atoi(e) == 1 ? 1 : 2;
                if (p.tile_nx == 1) {  // 32-wide tiles: 32 x 16 (4 warps) or 32 x 32 (8 warps)
                    const char* w = std::getenv("SF_VEC_WARPS");
                    p.vec_warps = w && std::atoi(w) == 8 ? 8 : 4;
                }
            }
            if (const char* e = std::getenv("SF_VEC_AQ")) p.vec_aq = std::atoi(e) != 0;
            if (const char* e = std::getenv("SF_VEC_AQ2")) p.vec_aq2 = std::atoi(e) != 0;
            // two rows per lane: same tile, half the consumer warps
            p.vec_rpl = 1;
            if (const char* e = std::getenv("SF_VEC_RPL"))
                if (std::atoi(e) == 2 && (p.tile_nx == 1 || p.vec_warps == 8)) {
                    p.vec_rpl = 2;
                    p.vec_warps = p.tile_nx == 1 ? 2 : 4;
                }
        }
        setup_tma(p);
        p.use_tma = true;
        set_grid(p);
        return;
    }
    if (vec_on && p.ac.radius >= 5 && !(vq && vq[0] == '0')) {
        p.use_vec = true;
        p.use_vecq = true;
        p.vec_warps = 4;
        if (const char* w = std::getenv("SF_VEC_WARPS")) {
            const int v = std::atoi(w);
            p.vec_warps = v == 8 ? 8 : (v == 12 && p.ac.radius >= 7) ? 12 : 4;  // 64 x 8 / 16 / 24 tiles
        }
        setup_tma(p);
        p.use_tma = true;
        set_grid(p);
        return;
    }
    const char* force = std::getenv("SF_TMA");
    if (p.ac.radius > 3 && !(force && force[0] == '1')) return;
    if (p.ac.radius > 4 && !std::getenv("SF_TILE")) p.tile_nx = 1;
    setup_tma(p);
    p.use_tma = true;
    set_grid(p);
}



void init_device(Plan& p, int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw Status(SF_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= count) throw Status(SF_ERR_INVALID, "device index out of range");
    p.device = device;
    SF_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    SF_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        throw Status(SF_ERR_CUDA, std::string("device ") + prop.name +
                                      " is not sm_100-class; this library is built for sm_100a");
    SF_CUDA(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
    SF_CUDA(cudaEventCreate(&p.ev0));
    SF_CUDA(cudaEventCreate(&p.ev1));
}

int64_t field_slack(const Plan& p);

void layout(Plan& p, int ndim, const int64_t* shape) {
    p.ndim = ndim;
    for (int i = 0; i < 3; ++i) p.n[i] = i < ndim ? shape[i] : 1;
    const int64_t last = shape[ndim - 1];
    p.pitch = round_up(last, 32);
    if (ndim == 3) {
        p.plane = p.n[1] * p.pitch;
        p.slot_elems = p.n[0] * p.plane;
    } else {
        p.plane = 0;
        p.slot_elems = p.n[0] * p.pitch;
    }
    for (int i = 0; i < ndim; ++i)
        if (shape[i] > (int64_t{1} << 30)) throw Status(SF_ERR_INVALID, "extent too large");
    if (p.slot_elems + field_slack(p) >= (int64_t{1} << 31))
        throw Status(SF_ERR_INVALID, "field exceeds 2^31 elements (32-bit offsets)");
    p.staging = dalloc<float>(static_cast<size_t>(field_numel(p)));
}

// Guard slack after every field: the 3D stencil's tile loads are
// unpredicated, and tiles overhanging the a1/a2 extents read up to one plane
// past the last plane (never stored). Nothing before the base is touched:
// every halo read starts at plane >= r.
int64_t field_slack(const Plan& p) { return (p.ndim == 3 ? p.plane : 0) + 64 * p.pitch + 1024; }

float* alloc_field(Plan& p) {
    float* f = dalloc<float>(static_cast<size_t>(p.slot_elems + field_slack(p)));
    SF_CUDA(cudaMemsetAsync(f, 0, sizeof(float) * p.slot_elems, p.stream));
    return f;
}

void check_acoustic_desc(const sf_acoustic_desc* d) {
    if (!d) throw Status(SF_ERR_INVALID, "null descriptor");
    if (d->ndim < 2 || d->ndim > 3) throw Status(SF_ERR_INVALID, "acoustic needs 2 or 3 dims");
    if (d->space_order < 2 || d->space_order > 16 || d->space_order % 2)
        throw Status(SF_ERR_INVALID, "space_order must be even and >= 2, got " +
                                         std::to_string(d->space_order));
    for (int i = 0; i < d->ndim; ++i)
        if (d->shape[i] < d->space_order + 1)
            throw Status(SF_ERR_INVALID, "extent " + std::to_string(d->shape[i]) +
                                             " too small for order " +
                                             std::to_string(d->space_order));
    if (d->nt < 0 || d->n_src < 1 || d->n_rec < 1)
        throw Status(SF_ERR_INVALID, "nt must be >= 0 and point sets non-empty");
    if (!(d->dt > 0) || !(d->spacing > 0)) throw Status(SF_ERR_INVALID, "dt/spacing must be > 0");
}

void setup_acoustic(Plan& p, const sf_acoustic_desc* d, int device, bool fwi) {
    check_acoustic_desc(d);
    init_device(p, device);
    layout(p, d->ndim, d->shape);
    p.nt = d->nt;
    p.ac = acoustic_constants(d->ndim, d->space_order, fwi ? true : d->forward != 0, d->dt,
                              d->spacing);
    p.z0 = p.ac.radius;
    p.z1 = static_cast<int>(p.n[0]) - p.ac.radius;
    p.global_n0 = p.n[0];
    p.own_begin = 0;
    p.own_end = p.n[0];
    p.own_lo = 0;
    p.own_hi = static_cast<int>(p.n[0]);
    p.m = alloc_field(p);
    p.eta = alloc_field(p);
    alloc_points(p, p.src, d->n_src, d->nt);
    alloc_points(p, p.rec, d->n_rec, d->nt);
    choose_geometry(p);
    const int corners = 1 << p.ndim;
    const int64_t fb = field_numel(p) * 4;
    p.arg_names = {d->forward || fwi ? "u" : "v", "m", "eta", "src", "src_ci", "src_w",
                   "rec", "rec_ci", "rec_w"};
    p.arg_bytes = {3 * fb, fb, fb, d->nt * d->n_src * 4, d->n_src * p.ndim * 4,
                   d->n_src * corners * 4, d->nt * d->n_rec * 4, d->n_rec * p.ndim * 4,
                   d->n_rec * corners * 4};
    p.launches_per_step = 3;  // recomputed by launches_per_step_of()
}

void upload_acoustic(Plan& p, void* const* a) {
    const bool fwd = p.ac.forward;
    for (int s = 0; s < 3; ++s)
        if (a[0]) h2d_field(p, p.slot[s], static_cast<const float*>(a[0]) + s * field_numel(p));
    if (a[1]) h2d_field(p, p.m, static_cast<const float*>(a[1]));
    if (a[2]) {
        h2d_field(p, p.eta, static_cast<const float*>(a[2]));
        ++p.eta_gen;
    }
    upload_points(p, p.src, static_cast<const float*>(a[3]), static_cast<const int*>(a[4]),
                  static_cast<const float*>(a[5]), fwd);
    upload_points(p, p.rec, static_cast<const float*>(a[6]), static_cast<const int*>(a[7]),
                  static_cast<const float*>(a[8]), !fwd);
}

void download_acoustic(Plan& p, void* const* a) {
    for (int s = 0; s < 3; ++s)
        if (a[0]) d2h_field(p, static_cast<float*>(a[0]) + s * field_numel(p), p.slot[s]);
    if (a[1]) d2h_field(p, static_cast<float*>(a[1]), p.m);
    if (a[2]) d2h_field(p, static_cast<float*>(a[2]), p.eta);
    if (a[3])
        SF_CUDA(cudaMemcpyAsync(a[3], p.src.series, sizeof(float) * p.nt * p.src.np,
                                cudaMemcpyDeviceToHost, p.stream));
    if (a[6])
        SF_CUDA(cudaMemcpyAsync(a[6], p.rec.series, sizeof(float) * p.nt * p.rec.np,
                                cudaMemcpyDeviceToHost, p.stream));
    // ci / w are read-only for the kernel: nothing to copy back
    SF_CUDA(cudaStreamSynchronize(p.stream));
}

// ---------------------------------------------------------------------------
// sf_plan_invoke with the upload hidden behind the first time steps.
//
// The five fields (three time slots, m, eta) reach the GPU in chunks of whole
// a0 planes on a copy stream. Step k needs u(t) only R planes beyond what it
// updates, so while chunk c+1 is still on the PCIe link the first K steps
// already run on the planes that have arrived, each trailing its predecessor
// by R planes (a time-skewed sweep: step k may update plane z once step k-1
// has finished planes < z + R + 1). Every point is still computed by the same
// kernel from the same inputs, injection and sampling of a step are applied
// to each plane range right after the step's stencil on it, in stream order,
// so the result is bitwise the plain upload-then-run sequence
// (tests/test_gpu_parity.py::test_invoke_overlapped_*). After the last chunk
// the K steps are completed one after the other and steps K..nt run as the
// usual captured graph; the last K2 steps are skewed again so that low planes
// become final first and travel back while the rest finishes. Used where a
// chunk of a step is long against a kernel launch (io_overlap_eligible).
// SF_NO_IO_OVERLAP=1 disables, SF_IO_OVERLAP=1 forces it at any size (tests),
// SF_IO_CHUNK_PLANES / SF_IO_STEPS / SF_IO_TAIL_STEPS override the chunk
// height (multiple of 32), K and K2.
// Rough times the decisions below rest on: a memory-bound time step (20 B per
// interior point at ~5.5 TB/s) and the PCIe link at ~55 GB/s.
double step_seconds_estimate(const Plan& p) {
    const int r = p.ac.radius;
    const double pts = static_cast<double>(p.n[0] - 2 * r) * static_cast<double>(p.n[1] - 2 * r) *
                       static_cast<double>(p.n[2] - 2 * r);
    return pts * 20.0 / 5.5e12;
}

// Chunk height: whole planes, a multiple of 32 (one eta flag word per 32
// planes), about n0 / 16 and at least 64.
int io_chunk_planes(const Plan& p) {
    const int n0 = static_cast<int>(p.n[0]);
    if (const char* e = std::getenv("SF_IO_CHUNK_PLANES")) {
        const int v = std::atoi(e);
        if (v >= 32) return v / 32 * 32;
    }
    return (std::max(64, n0 / 16) + 31) / 32 * 32;
}

bool io_overlap_eligible(const Plan& p, void* const* a, int nargs) {
    bool forced = false;
    if (const char* e = std::getenv("SF_NO_IO_OVERLAP"))
        if (e[0] == '1') return false;
    if (const char* e = std::getenv("SF_IO_OVERLAP")) forced = e[0] == '1';  // tests: any size
    if (p.kind != Plan::ACOUSTIC || p.ndim != 3 || p.slab || p.nccl_comm) return false;
    if (!(p.use_tma && (p.use_vec || p.use_vecq))) return false;
    if (nargs != 9 || !a[0] || !a[1] || !a[2]) return false;
    const int r = p.ac.radius;
    if (!(p.nt >= 1 && p.n[0] > 32 && p.z1 - p.z0 >= 4 * r)) return false;
    if (forced) return true;
    // asynchronous copies need page-locked host buffers (pageable ones are
    // staged synchronously: correct, but nothing would overlap)
    for (int i = 0; i < 3; ++i) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, a[i]) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (at.type != cudaMemoryTypeHost) return false;
    }
    // worth it only where a chunk of a step is long against a launch (the
    // skewed steps are stream launches, not graph nodes): at least three
    // chunks of >= 15 us each (measured e2e: 1024^3 +11 %, 512^3 +9..19 %,
    // 281^3 +5 %)
    const int zc = io_chunk_planes(p);
    return 3 * zc <= p.n[0] && step_seconds_estimate(p) * zc / static_cast<double>(p.n[0]) >= 15e-6;
}

void tile_extent(const Plan& p, int64_t* wx, int64_t* wy) {
    *wx = p.use_vecq ? 64 : 32 * p.tile_nx;
    *wy = p.use_vecq ? 2 * p.vec_warps
          : p.use_vec ? 4 * p.vec_warps * p.vec_rpl / p.tile_nx
                      : p.tile_ty;
}

void h2d_planes(const Plan& p, float* dst, const float* src, int z0, int z1, cudaStream_t st) {
    const int64_t n1 = p.n[1], n2 = p.n[2];
    if (p.pitch == n2) {  // dense rows: one contiguous transfer
        SF_CUDA(cudaMemcpyAsync(dst + static_cast<int64_t>(z0) * p.plane,
                                src + static_cast<int64_t>(z0) * n1 * n2,
                                sizeof(float) * static_cast<size_t>(z1 - z0) * n1 * n2,
                                cudaMemcpyHostToDevice, st));
        return;
    }
    // padded rows: one contiguous transfer into the staging field, then a
    // device repack on the same stream (row-by-row 2D copies over PCIe are
    // several times slower for ~1 KB rows)
    const int64_t rows = static_cast<int64_t>(z1 - z0) * n1;
    SF_CUDA(cudaMemcpyAsync(p.staging, src + static_cast<int64_t>(z0) * n1 * n2,
                            sizeof(float) * rows * n2, cudaMemcpyHostToDevice, st));
    repack_rows_kernel<<<repack_grid(rows), 256, 0, st>>>(dst + static_cast<int64_t>(z0) * p.plane,
                                                         p.pitch, p.staging, n2, rows,
                                                         static_cast<int>(n2));
}

void d2h_planes(const Plan& p, float* dst, const float* src, int z0, int z1, cudaStream_t st) {
    const int64_t n1 = p.n[1], n2 = p.n[2];
    if (p.pitch == n2) {
        SF_CUDA(cudaMemcpyAsync(dst + static_cast<int64_t>(z0) * p.plane,
                                src + static_cast<int64_t>(z0) * p.plane,
                                sizeof(float) * static_cast<size_t>(z1 - z0) * p.plane,
                                cudaMemcpyDeviceToHost, st));
        return;
    }
    const int64_t rows = static_cast<int64_t>(z1 - z0) * n1;
    repack_rows_kernel<<<repack_grid(rows), 256, 0, st>>>(p.staging, n2,
                                                         src + static_cast<int64_t>(z0) * p.plane,
                                                         p.pitch, rows, static_cast<int>(n2));
    SF_CUDA(cudaMemcpyAsync(dst + static_cast<int64_t>(z0) * n1 * n2, p.staging,
                            sizeof(float) * rows * n2, cudaMemcpyDeviceToHost, st));
}

// Returns true when the three slots are already back in host memory (the tail
// ran; false when nt left no steps for it).
bool invoke_overlapped(Plan& p, void* const* a) {
    const bool fwd = p.ac.forward;
    const int r = p.ac.radius, n0 = static_cast<int>(p.n[0]);
    const int zlo = p.z0, zhi = p.z1;
    SF_CUDA(cudaSetDevice(p.device));
    // point sets first (host-side CSR build, small copies on the compute stream)
    upload_points(p, p.src, static_cast<const float*>(a[3]), static_cast<const int*>(a[4]),
                  static_cast<const float*>(a[5]), fwd);
    upload_points(p, p.rec, static_cast<const float*>(a[6]), static_cast<const int*>(a[7]),
                  static_cast<const float*>(a[8]), !fwd);
    const PointSet& inj = fwd ? p.src : p.rec;
    const PointSet& smp = fwd ? p.rec : p.src;
    auto c0_range = [&](const PointSet& s, int* lo, int* hi) {
        *lo = INT32_MAX;
        *hi = -1;
        for (int64_t q = 0; q < s.np; ++q) {
            const int c = s.host_ci[q * 3];
            *lo = std::min(*lo, c);
            *hi = std::max(*hi, c);
        }
    };
    int inj_lo, inj_hi, smp_lo, smp_hi;  // lower corner planes of the point sets
    c0_range(inj, &inj_lo, &inj_hi);
    c0_range(smp, &smp_lo, &smp_hi);

    const int zc = io_chunk_planes(p);
    const int nchunks = (n0 + zc - 1) / zc;
    // steps worth of compute that fit under the upload / the copy back
    const double t_step = step_seconds_estimate(p);
    const double field_bytes = 4.0 * static_cast<double>(p.n[0]) * p.n[1] * p.n[2];
    // (a skewed step costs ~12 us of launch gaps and ramp per chunk on top of its work)
    const double t_chunk = t_step * zc / n0, eff = t_chunk / (t_chunk + 12e-6);
    const int k_up = static_cast<int>(eff * 5.0 * field_bytes / 55e9 / t_step) + 1;
    const int k_down = static_cast<int>(eff * 1.2 * 3.0 * field_bytes / 55e9 / t_step) + 1;
    int K = static_cast<int>(std::min<int64_t>(p.nt, std::min(k_up, 128)));
    if (const char* e = std::getenv("SF_IO_STEPS")) {
        const int v = std::atoi(e);
        if (v >= 1) K = static_cast<int>(std::min<int64_t>(p.nt, v));
    }
    K = std::max(1, std::min(K, (zhi - zlo) / r - 2));

    if (!p.io) SF_CUDA(cudaStreamCreateWithFlags(&p.io, cudaStreamNonBlocking));
    while (static_cast<int>(p.ev_up.size()) < nchunks) {
        cudaEvent_t e;
        SF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p.ev_up.push_back(e);
    }
    // the copies start once whatever used the fields before has finished
    SF_CUDA(cudaEventRecord(p.ev0, p.stream));
    SF_CUDA(cudaStreamWaitEvent(p.io, p.ev0, 0));
    const int64_t fe = field_numel(p);
    for (int c = 0; c < nchunks; ++c) {
        const int a0 = c * zc, a1 = std::min(n0, a0 + zc);
        for (int s = 0; s < 3; ++s)
            h2d_planes(p, p.slot[s], static_cast<const float*>(a[0]) + s * fe, a0, a1, p.io);
        h2d_planes(p, p.m, static_cast<const float*>(a[1]), a0, a1, p.io);
        h2d_planes(p, p.eta, static_cast<const float*>(a[2]), a0, a1, p.io);
        SF_CUDA(cudaEventRecord(p.ev_up[c], p.io));
    }
    ++p.eta_gen;
    const bool flags = eta_flags_wanted(p);
    if (flags) {
        int tx, ty;
        eta_flag_tile(p, &tx, &ty);
        prepare_eta_flags(p, p.eta0, tx, ty);
        p.eta0.gen = p.eta_gen;  // filled chunk by chunk below, before any launch reads them
    }

    // the last K2 steps run skewed the other way round (below): low planes
    // become final first and go back to the host while the rest finishes
    int K2 = static_cast<int>(std::min<int64_t>(p.nt - K, std::min(k_down, 96)));
    if (const char* e = std::getenv("SF_IO_TAIL_STEPS")) {
        const int v = std::atoi(e);
        if (v >= 0) K2 = static_cast<int>(std::min<int64_t>(p.nt - K, v));
    }
    K2 = std::max(0, K2);

    int64_t wx, wy;
    tile_extent(p, &wx, &wy);
    // step k over planes [*front, nf): stencil, then this step's injection
    // into, and sampling on top of, exactly those planes
    auto advance = [&](int64_t k, int* front, int nf) {
        const int f0 = *front;
        if (nf <= f0) return;
        sf_plan::ZRange zr;
        zr.z0 = f0;
        zr.z1 = nf;
        chunk_grid(p, wx, wy, p.resident, &zr.grid, &zr.zchunk, nf - f0);
        const StepSlots st = step_slots(p, k, p.slot);
        launch_stencil(p, st.out, st.cur, st.prev, nullptr, nullptr, &zr);
        // planes outside the stencil's range belong to the first / last range
        const int fa = f0 == zlo ? 0 : f0, fb = nf == zhi ? n0 + 1 : nf;
        if (inj.np > 0 && inj.ncells > 0 && inj_hi + 1 >= fa && inj_lo < fb) {
            launch_inject(p, inj, st.out, st.row, 0, -1, fa, fb);
        }
        if (smp.np > 0 && smp_hi + 1 >= fa && smp_lo + 1 < fb) {
            launch_sample(p, smp, st.out, st.row, std::max(fa, 1), fb);
        }
        *front = nf;
    };
    struct PlainLaunch {  // see g_plain_launches
        PlainLaunch() { g_plain_launches = true; }
        ~PlainLaunch() { g_plain_launches = false; }
    };
    {
        std::vector<int> front(static_cast<size_t>(K), zlo);
        for (int c = 0; c < nchunks; ++c) {
            const int up = std::min(n0, (c + 1) * zc);  // planes [0, up) have arrived
            SF_CUDA(cudaStreamWaitEvent(p.stream, p.ev_up[c], 0));
            if (flags) launch_eta_flags(p, p.eta0, c * zc / 32, (up - c * zc + 31) / 32);
            for (int k = 0; k < K; ++k) {
                // u(t) of step k is valid below `avail`: the upload for k = 0,
                // else what step k-1 has finished (plus the static planes
                // beyond the interior once everything has arrived)
                const int avail = k == 0 ? up : front[k - 1] < zhi ? front[k - 1] : up == n0 ? n0 : zhi;
                const int nf = std::min(zhi, avail - r);
                if (nf <= front[k]) break;  // later steps trail this one
                if (k == 0) {
                    // right behind the flags kernel: a plain launch, so the
                    // producer warp's early flag reads are ordered after it;
                    // the launches that follow may overlap their predecessor
                    PlainLaunch plain;
                    advance(k, &front[k], nf);
                } else {
                    advance(k, &front[k], nf);
                }
            }
        }
        for (int k = 0; k < K; ++k) advance(k, &front[k], zhi);  // complete the skewed steps in order
    }
    run_steps(p, K, p.nt - K2);
    if (K2 == 0) return false;

    // Tail: chunk c of the three slots is final once the last step has
    // finished its planes, which needs step nt-1-i to be r * i planes further.
    // Each pass advances all K2 steps just that far, then the chunk's copy
    // back starts on the copy stream while the next pass runs.
    {
        std::vector<int> front(static_cast<size_t>(K2), zlo);
        float* host_u = static_cast<float*>(a[0]);
        for (int c = 0; c < nchunks; ++c) {
            const int c0 = c * zc, c1 = std::min(n0, c0 + zc);
            for (int j = 0; j < K2; ++j) {
                const int target = c1 >= zhi ? zhi : std::min(zhi, c1 + r * (K2 - 1 - j));
                advance(p.nt - K2 + j, &front[j], target);
            }
            SF_CUDA(cudaEventRecord(p.ev_up[c], p.stream));
            SF_CUDA(cudaStreamWaitEvent(p.io, p.ev_up[c], 0));
            for (int sl = 0; sl < 3; ++sl) d2h_planes(p, host_u + sl * fe, p.slot[sl], c0, c1, p.io);
        }
        SF_CUDA(cudaEventRecord(p.ev_up[0], p.io));
        SF_CUDA(cudaStreamWaitEvent(p.stream, p.ev_up[0], 0));  // the call ends when the copies have
    }
    return true;
}

void upload_any(Plan& p, void* const* a, int nargs) {
    if (nargs != static_cast<int>(p.arg_names.size()))
        throw Status(SF_ERR_SIGNATURE, "expected " + std::to_string(p.arg_names.size()) +
                                           " buffers, got " + std::to_string(nargs));
    SF_CUDA(cudaSetDevice(p.device));
    if (p.kind == Plan::DIFFUSION) {
        if (a[0])
            for (int s = 0; s < 2; ++s)
                h2d_field(p, p.slot[s], static_cast<const float*>(a[0]) + s * field_numel(p));
    } else {
        upload_acoustic(p, a);
    }
}

void download_any(Plan& p, void* const* a, int nargs) {
    if (nargs != static_cast<int>(p.arg_names.size()))
        throw Status(SF_ERR_SIGNATURE, "expected " + std::to_string(p.arg_names.size()) +
                                           " buffers, got " + std::to_string(nargs));
    SF_CUDA(cudaSetDevice(p.device));
    if (p.kind == Plan::DIFFUSION) {
        if (a[0])
            for (int s = 0; s < 2; ++s)
                d2h_field(p, static_cast<float*>(a[0]) + s * field_numel(p), p.slot[s]);
        SF_CUDA(cudaStreamSynchronize(p.stream));
    } else {
        download_acoustic(p, a);
    }
}

void check_kernel_errors(Plan& p) {
    SF_CUDA(cudaGetLastError());
    cudaError_t e = cudaStreamSynchronize(p.stream);
    if (e != cudaSuccess)
        throw Status(SF_ERR_KERNEL, std::string("kernel failed: ") + cudaGetErrorString(e));
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SF_OK;
    } catch (const Status& s) {
        set_error(s.what());
        return s.code;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return SF_ERR_INVALID;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SF_ERR_INVALID;
    }
}

} // namespace
} // namespace sfb

sf_plan::~sf_plan() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (float* s : slot) sfb::dfree(s);
    for (float* s : dscratch) sfb::dfree(s);
    sfb::dfree(staging);
    sfb::dfree(m);
    sfb::dfree(eta);
    sfb::free_points(src);
    sfb::free_points(rec);
    sfb::dfree(fused.tile_start);
    sfb::dfree(fused.cell);
    sfb::dfree(fused.start);
    sfb::dfree(fused.cp);
    sfb::dfree(fused.cw);
    sfb::dfree(fused_adj.tile_start);
    sfb::dfree(fused_adj.cell);
    sfb::dfree(fused_adj.start);
    sfb::dfree(fused_adj.cp);
    sfb::dfree(fused_adj.cw);
    sfb::dfree(eta0.bits);
    sfb::dfree(eta0_grad.bits);
    sfb::dfree(hist);
    sfb::dfree(grad);
    for (float* s : v) sfb::dfree(s);
    for (cudaEvent_t e : ev_up) cudaEventDestroy(e);
    if (io) cudaStreamDestroy(io);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_copy) cudaEventDestroy(ev_copy);
    if (ev_band) cudaEventDestroy(ev_band);
    if (ev_comm) cudaEventDestroy(ev_comm);
    if (comm) cudaStreamDestroy(comm);
    if (nccl_comm) {
        try {
            sfb::nccl().CommDestroy(nccl_comm);
        } catch (...) {
        }
    }
    if (stream) cudaStreamDestroy(stream);
}

using sfb::guard;
using sfb::Status;

namespace sfb {
namespace {

// ---------------------------------------------------------------------------
// GPU autotune (the reference's Operator::autotune, op.cpp:169-221, searches
// CPU cache-blocking plans; here the search space is the stencil kernel
// family, tile shape and pipeline depth).
struct StencilConfig {
    int kind;  // 0 per-thread loads, 1 scalar TMA, 2 vector TMA (ring), 3 queue vector TMA
    int tile_nx, tile_ty, vec_warps, stages;
};

void apply_config(Plan& p, const StencilConfig& c) {
    clear_graphs(p);
    p.use_tma = p.use_vec = p.use_vecq = false;
    p.tile_nx = c.tile_nx;
    p.tile_ty = c.tile_ty;
    p.vec_warps = c.vec_warps;
    // vector ring: tile_ty = 4 * warps * rows-per-lane / tile_nx
    p.vec_rpl = c.kind == 2 ? std::max(1, c.tile_ty * c.tile_nx / (4 * c.vec_warps)) : 1;
    p.stages_override = c.stages;
    if (c.kind >= 1) {
        p.use_vec = c.kind >= 2;
        p.use_vecq = c.kind == 3;
        setup_tma(p);
        p.use_tma = true;
    }
    set_grid(p);
}

StencilConfig current_config(const Plan& p) {
    const bool ring = p.use_vec && !p.use_vecq;
    return {p.use_vecq ? 3 : p.use_vec ? 2 : p.use_tma ? 1 : 0, p.tile_nx,
            ring ? 4 * p.vec_warps * p.vec_rpl / p.tile_nx : p.tile_ty, p.vec_warps,
            p.use_tma ? p.tma_stages : 0};
}

std::vector<StencilConfig> tune_candidates(const Plan& p) {
    std::vector<StencilConfig> out;
    const int r = p.ac.radius;
    for (int nx = 1; nx <= max_tile_nx(r); ++nx)
        for (int ty : {8, 16}) out.push_back({0, nx, ty, 4, 0});
    if (r <= 3)
        for (int nx = 1; nx <= tma_max_nx(r); ++nx)
            for (int st : {2, 3}) out.push_back({1, nx, 8, 4, st});
    if (r <= 4) {
        for (int w : {4, 8})
            for (int st : {2, 3, 4}) out.push_back({2, 2, 2 * w, w, st});
        for (int st : {2, 3, 4}) out.push_back({2, 1, 16, 4, st});
        for (int st : {2, 3, 4}) out.push_back({2, 1, 16, 2, st});  // 2 rows per lane
        for (int st : {2, 3}) out.push_back({2, 2, 16, 4, st});     // 2 rows per lane
        for (int st : {2, 3}) out.push_back({2, 1, 32, 8, st});     // 32 x 32 tiles
        if (r == 4)
            for (int st : {2, 3}) out.push_back({2, 2, 32, 16, st});  // 64 x 32, one CTA per SM
    }
    if (r >= 5)
        for (int w : {4, 8})
            for (int st : {2, 3, 4}) out.push_back({3, 2, 2 * w, w, st});
    return out;
}

} // namespace
} // namespace sfb


extern "C" int sf_plan_autotune(sf_plan* p, int64_t tune_steps, int repeats, sf_tune_entry* entries,
                                int max_entries, int* n_entries) {
    using namespace sfb;
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind != sf_plan::ACOUSTIC || p->ndim != 3 || p->slab)
            throw Status(SF_ERR_INVALID, "autotune tunes single-domain 3D acoustic plans");
        if (tune_steps < 1 || tune_steps > p->nt) throw Status(SF_ERR_INVALID, "tune_steps range");
        if (repeats < 1) repeats = 1;
        NvtxRange nvtx("sf_plan_autotune");
        SF_CUDA(cudaSetDevice(p->device));
        // snapshot what a run modifies: the three slots and both series
        const size_t fbytes = sizeof(float) * (p->slot_elems + field_slack(*p));
        const size_t sbytes = sizeof(float) * p->nt * p->src.np;
        const size_t rbytes = sizeof(float) * p->nt * p->rec.np;
        // snapshot buffers freed, and the plan put back on its original
        // configuration with its state restored, on every exit path
        struct Snap {
            std::vector<float*> bufs;
            ~Snap() {
                for (float* f : bufs) dfree(f);
            }
        } snap_guard;
        std::vector<float*>& snap = snap_guard.bufs;
        auto copy = [&](void* dst, const void* src, size_t n) {
            SF_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, p->stream));
        };
        for (int s = 0; s < 3; ++s) snap.push_back(dalloc<float>(fbytes / sizeof(float)));
        snap.push_back(dalloc<float>(std::max<size_t>(sbytes, 4) / sizeof(float)));
        snap.push_back(dalloc<float>(std::max<size_t>(rbytes, 4) / sizeof(float)));
        auto restore = [&](bool save) {
            for (int s = 0; s < 3; ++s)
                save ? copy(snap[s], p->slot[s], fbytes) : copy(p->slot[s], snap[s], fbytes);
            save ? copy(snap[3], p->src.series, sbytes) : copy(p->src.series, snap[3], sbytes);
            save ? copy(snap[4], p->rec.series, rbytes) : copy(p->rec.series, snap[4], rbytes);
        };
        restore(true);
        const StencilConfig original = current_config(*p);
        StencilConfig best = original;
        float best_ms = -1.0f;
        int n = 0;
        struct Revert {
            sf_plan* p;
            const StencilConfig& cfg;
            std::function<void(bool)>& restore;
            bool armed = true;
            ~Revert() {
                if (!armed) return;
                try {
                    cudaStreamSynchronize(p->stream);
                    clear_graphs(*p);
                    apply_config(*p, cfg);
                    restore(false);
                    cudaStreamSynchronize(p->stream);
                } catch (...) {
                }
            }
        };
        std::function<void(bool)> restore_fn = restore;
        Revert revert{p, original, restore_fn};
        for (const StencilConfig& c : tune_candidates(*p)) {
            try {
                apply_config(*p, c);
            } catch (const Status&) {
                continue;  // does not fit (shared memory) or not compiled
            }
            std::vector<float> t;
            for (int rep = 0; rep < repeats + 1; ++rep) {  // first run warms the graph
                restore(false);
                SF_CUDA(cudaEventRecord(p->ev0, p->stream));
                run_steps(*p, 0, tune_steps);
                SF_CUDA(cudaEventRecord(p->ev1, p->stream));
                check_kernel_errors(*p);
                float ms = 0;
                SF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
                if (rep > 0) t.push_back(ms);
            }
            std::sort(t.begin(), t.end());
            const float med = t[t.size() / 2];
            if (entries && n < max_entries)
                entries[n] = {c.kind, c.tile_nx, c.tile_ty, c.vec_warps, p->use_tma ? p->tma_stages : 0,
                              med};
            ++n;
            if (best_ms < 0 || med < best_ms) {
                best_ms = med;
                best = c;
            }
            clear_graphs(*p);
        }
        apply_config(*p, best);
        restore(false);
        SF_CUDA(cudaStreamSynchronize(p->stream));
        revert.armed = false;
        if (n_entries) *n_entries = n;
    });
}



// ---------------------------------------------------------------------------
// HBM-resident GridFunction I/O in the reference's binary format
// (save_buffer / load_buffer, grid.cpp:213-254): magic "SFG1" | name |
// element id (f32 0, f64 1, i32 2) | ndim | extents | raw little-endian data,
// written straight from (read straight into) the device mirrors.
namespace sfb {
namespace {

struct BufferView {
    std::string name;
    int elem;                      // 0 f32, 2 i32
    std::vector<uint32_t> extents;
};

BufferView buffer_view(const Plan& p, int i) {
    BufferView v;
    v.name = p.arg_names.at(i);
    v.elem = (v.name == "src_ci" || v.name == "rec_ci") ? 2 : 0;
    auto field = [&](int slots) {
        if (slots) v.extents.push_back(static_cast<uint32_t>(slots));
        for (int d = 0; d < p.ndim; ++d) v.extents.push_back(static_cast<uint32_t>(p.n[d]));
    };
    const int corners = 1 << p.ndim;
    if (p.kind == Plan::DIFFUSION) {
        field(2);
        return v;
    }
    switch (i) {
        case 0: field(3); break;
        case 1: case 2: field(0); break;
        case 3: v.extents = {static_cast<uint32_t>(p.nt), static_cast<uint32_t>(p.src.np)}; break;
        case 4: v.extents = {static_cast<uint32_t>(p.src.np), static_cast<uint32_t>(p.ndim)}; break;
        case 5: v.extents = {static_cast<uint32_t>(p.src.np), static_cast<uint32_t>(corners)}; break;
        case 6: v.extents = {static_cast<uint32_t>(p.nt), static_cast<uint32_t>(p.rec.np)}; break;
        case 7: v.extents = {static_cast<uint32_t>(p.rec.np), static_cast<uint32_t>(p.ndim)}; break;
        case 8: v.extents = {static_cast<uint32_t>(p.rec.np), static_cast<uint32_t>(corners)}; break;
        default: throw Status(SF_ERR_INVALID, "argument index out of range");
    }
    return v;
}

int find_arg(const Plan& p, const char* name) {
    for (size_t i = 0; i < p.arg_names.size(); ++i)
        if (p.arg_names[i] == name) return static_cast<int>(i);
    throw Status(SF_ERR_INVALID, std::string("no buffer named ") + name);
}

// host staging of argument i through the plan's own download/upload paths
void transfer_arg(Plan& p, int i, void* host, bool to_host) {
    std::vector<void*> args(p.arg_names.size(), nullptr);
    args[i] = host;
    if (to_host)
        download_any(p, args.data(), static_cast<int>(args.size()));
    else
        upload_any(p, args.data(), static_cast<int>(args.size()));
    if (!to_host) SF_CUDA(cudaStreamSynchronize(p.stream));
}

} // namespace
} // namespace sfb

extern "C" int sf_plan_save_buffer(sf_plan* p, const char* name, const char* path) {
    using namespace sfb;
    if (!p || !name || !path) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind == sf_plan::FWI) throw Status(SF_ERR_INVALID, "FWI plans have no buffers");
        const int i = find_arg(*p, name);
        const BufferView v = buffer_view(*p, i);
        std::vector<char> host(static_cast<size_t>(p->arg_bytes.at(i)));
        // ci / w are not written by the kernels: the device copies are the uploaded ones
        if (i == 4 || i == 5 || i == 7 || i == 8) {
            const PointSet& ps = i < 6 ? p->src : p->rec;
            const void* dev = (i == 4 || i == 7) ? static_cast<const void*>(ps.ci) : ps.w;
            SF_CUDA(cudaMemcpy(host.data(), dev, host.size(), cudaMemcpyDeviceToHost));
        } else {
            transfer_arg(*p, i, host.data(), true);
        }
        FILE* f = std::fopen(path, "wb");
        if (!f) throw Status(SF_ERR_INVALID, std::string("cannot open for write: ") + path);
        auto put = [&](uint32_t x) { std::fwrite(&x, 4, 1, f); };
        put(0x53464731u);
        put(static_cast<uint32_t>(v.name.size()));
        std::fwrite(v.name.data(), 1, v.name.size(), f);
        put(static_cast<uint32_t>(v.elem));
        put(static_cast<uint32_t>(v.extents.size()));
        for (uint32_t e : v.extents) put(e);
        const size_t wrote = std::fwrite(host.data(), 1, host.size(), f);
        std::fclose(f);
        if (wrote != host.size()) throw Status(SF_ERR_INVALID, std::string("short write: ") + path);
    });
}

extern "C" int sf_plan_load_buffer(sf_plan* p, const char* name, const char* path) {
    using namespace sfb;
    if (!p || !name || !path) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind == sf_plan::FWI) throw Status(SF_ERR_INVALID, "FWI plans have no buffers");
        const int i = find_arg(*p, name);
        const BufferView v = buffer_view(*p, i);
        FILE* f = std::fopen(path, "rb");
        if (!f) throw Status(SF_ERR_INVALID, std::string("cannot open for read: ") + path);
        auto get = [&]() {
            uint32_t x = 0;
            if (std::fread(&x, 4, 1, f) != 1) x = 0xFFFFFFFFu;
            return x;
        };
        auto fail = [&](const std::string& m) {
            std::fclose(f);
            throw Status(SF_ERR_INVALID, m + " in " + path);
        };
        if (get() != 0x53464731u) fail("bad magic");
        const uint32_t nlen = get();
        if (nlen > 4096) fail("bad name length");
        std::string fname(nlen, '\0');
        if (std::fread(fname.data(), 1, nlen, f) != nlen) fail("short read");
        if (get() != static_cast<uint32_t>(v.elem)) fail("element type mismatch");
        if (get() != v.extents.size()) fail("rank mismatch");
        for (uint32_t e : v.extents)
            if (get() != e) fail("shape mismatch");
        std::vector<char> host(static_cast<size_t>(p->arg_bytes.at(i)));
        if (std::fread(host.data(), 1, host.size(), f) != host.size()) fail("short read");
        std::fclose(f);
        transfer_arg(*p, i, host.data(), false);
    });
}

// Text dumps (dump_csv, grid.cpp:256-273; save_series_text, sparse.cpp:215-227):
// values are written as `std::ostream << double` does by default, i.e. printf
// "%g" (six significant digits) of the f32 value widened to double.
namespace sfb {
void put_g(FILE* f, float x) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%g", static_cast<double>(x));
    std::fputs(buf, f);
}
}  // namespace sfb

extern "C" int sf_plan_dump_csv(sf_plan* p, const char* name, const char* path, long slot) {
    using namespace sfb;
    if (!p || !name || !path) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind == sf_plan::FWI) throw Status(SF_ERR_INVALID, "FWI plans have no buffers");
        const int i = find_arg(*p, name);
        const BufferView v = buffer_view(*p, i);
        const bool field = p->kind == sf_plan::DIFFUSION || i <= 2;
        const bool timed = p->kind == sf_plan::DIFFUSION || i == 0;
        if (!field || p->ndim != 2) throw Status(SF_ERR_INVALID, "csv dump supports 2D grids only");
        const long slots = timed ? static_cast<long>(v.extents[0]) : 1;
        if (timed && (slot < 0 || slot >= slots))
            throw Status(SF_ERR_INVALID, "slot out of range");
        std::vector<float> host(static_cast<size_t>(p->arg_bytes.at(i)) / 4);
        transfer_arg(*p, i, host.data(), true);
        const long n0 = p->n[0], n1 = p->n[1];
        const float* base = host.data() + (timed ? slot * n0 * n1 : 0);
        FILE* f = std::fopen(path, "w");
        if (!f) throw Status(SF_ERR_INVALID, std::string("cannot open for write: ") + path);
        for (long a = 0; a < n0; ++a) {
            for (long b = 0; b < n1; ++b) {
                if (b) std::fputc(',', f);
                put_g(f, base[a * n1 + b]);
            }
            std::fputc('\n', f);
        }
        if (std::fclose(f) != 0) throw Status(SF_ERR_INVALID, std::string("short write: ") + path);
    });
}

extern "C" int sf_plan_save_series_text(sf_plan* p, const char* name, const char* path) {
    using namespace sfb;
    if (!p || !name || !path) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind != sf_plan::ACOUSTIC) throw Status(SF_ERR_INVALID, "no sparse series in this plan");
        const int i = find_arg(*p, name);
        if (i != 3 && i != 6) throw Status(SF_ERR_INVALID, std::string(name) + " is not a series");
        const BufferView v = buffer_view(*p, i);
        const long nt = v.extents[0], np = v.extents[1];
        std::vector<float> host(static_cast<size_t>(nt * np));
        if (!host.empty()) transfer_arg(*p, i, host.data(), true);
        FILE* f = std::fopen(path, "w");
        if (!f) throw Status(SF_ERR_INVALID, std::string("cannot open for write: ") + path);
        for (long t = 0; t < nt; ++t) {
            for (long q = 0; q < np; ++q) {
                if (q) std::fputc(' ', f);
                put_g(f, host[t * np + q]);
            }
            std::fputc('\n', f);
        }
        if (std::fclose(f) != 0) throw Status(SF_ERR_INVALID, std::string("short write: ") + path);
    });
}

extern "C" int sf_plan_eta_skip_fraction(sf_plan* p, double* fraction) {
    return sfb::guard([&] {
        if (!p || !fraction) throw sfb::Status(SF_ERR_INVALID, "null argument");
        *fraction = 0.0;
        const sf_plan::EtaFlags& f = p->eta0;
        if (!f.bits || f.gen != p->eta_gen || p->ndim != 3) return;
        std::vector<uint32_t> bits(static_cast<size_t>(f.ntx) * f.nty * f.words);
        SF_CUDA(cudaStreamSynchronize(p->stream));
        SF_CUDA(cudaMemcpy(bits.data(), f.bits, bits.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        const int64_t r = p->ac.radius;
        auto overlap = [&](int64_t b, int64_t e, int64_t n) {
            return std::max<int64_t>(0, std::min(e, n - r) - std::max(b, r));
        };
        double skipped = 0.0, total = 0.0;
        for (int ty = 0; ty < f.nty; ++ty)
            for (int tx = 0; tx < f.ntx; ++tx) {
                const double pts = static_cast<double>(overlap(int64_t(tx) * f.tx, int64_t(tx + 1) * f.tx, p->n[2])) *
                                   static_cast<double>(overlap(int64_t(ty) * f.ty, int64_t(ty + 1) * f.ty, p->n[1]));
                for (int z = p->z0; z < p->z1; ++z) {
                    total += pts;
                    const uint32_t w = bits[(static_cast<size_t>(ty) * f.ntx + tx) * f.words + z / 32];
                    if ((w >> (z % 32)) & 1u) skipped += pts;
                }
            }
        *fraction = total > 0 ? skipped / total : 0.0;
    });
}

extern "C" int sf_selftest_reciprocal(int device, unsigned long long* mismatches) {
    using namespace sfb;
    if (!mismatches) return SF_ERR_INVALID;
    return guard([&] {
        SF_CUDA(cudaSetDevice(device));
        unsigned long long* d = dalloc<unsigned long long>(1);
        SF_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
        const uint32_t chunk = 1u << 30;  // float bit patterns per launch
        for (int mode = 0; mode < 2; ++mode)
            for (uint64_t first = 0; first < (1ull << 32); first += chunk)
                rcp4_check_kernel<<<chunk / 4 / 256, 256>>>(static_cast<uint32_t>(first), chunk, mode, d);
        SF_CUDA(cudaGetLastError());
        SF_CUDA(cudaMemcpy(mismatches, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        dfree(d);
    });
}

namespace sfb {
namespace {
// medium.cu reports MediumError; map it onto the status codes
template <typename F>
int medium_guard(F&& f) {
    return guard([&] {
        try {
            f();
        } catch (const sfb::MediumError& e) {
            throw sfb::Status(e.code == 1 ? SF_ERR_OOM : e.code == 2 ? SF_ERR_CUDA : SF_ERR_INVALID,
                              e.what());
        }
    });
}
}  // namespace
}  // namespace sfb

extern "C" {

const char* sf_last_error(void) { return sfb::g_error.c_str(); }

int sf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int sf_acoustic_plan_create(const sf_acoustic_desc* d, int device, sf_plan** out) {
    if (!out) return SF_ERR_INVALID;
    *out = nullptr;
    auto p = std::make_unique<sf_plan>();
    p->kind = sf_plan::ACOUSTIC;
    int rc = guard([&] {
        sfb::setup_acoustic(*p, d, device, false);
        for (int s = 0; s < 3; ++s) p->slot[s] = sfb::alloc_field(*p);
        sfb::enable_tma(*p);
        SF_CUDA(cudaStreamSynchronize(p->stream));
    });
    if (rc == SF_OK) *out = p.release();
    return rc;
}

int sf_diffusion_plan_create(const sf_diffusion_desc* d, int device, sf_plan** out) {
    if (!out || !d) return SF_ERR_INVALID;
    *out = nullptr;
    auto p = std::make_unique<sf_plan>();
    p->kind = sf_plan::DIFFUSION;
    int rc = guard([&] {
        if (d->order < 2 || d->order > 16 || d->order % 2)
            throw Status(SF_ERR_INVALID, "order must be even in [2, 16]");
        if (d->nx < d->order + 1 || d->ny < d->order + 1 || d->nt < 0)
            throw Status(SF_ERR_INVALID, "grid too small for the order");
        if (d->alpha_den == 0 || d->dx_den == 0 || d->alpha_num <= 0 || d->dx_num <= 0)
            throw Status(SF_ERR_INVALID, "alpha and dx must be positive rationals");
        sfb::init_device(*p, device);
        const int64_t shape[2] = {d->nx, d->ny};
        sfb::layout(*p, 2, shape);
        p->nt = d->nt;
        p->nslots = 2;
        p->dc = sfb::diffusion_constants(sfb::Rat::make(d->alpha_num, d->alpha_den),
                                         sfb::Rat::make(d->dx_num, d->dx_den), d->order);
        for (int s = 0; s < 2; ++s) p->slot[s] = sfb::alloc_field(*p);
        for (int s = 0; s < 2; ++s) p->dscratch[s] = sfb::alloc_field(*p);
        if (const char* env = std::getenv("SF_DIFFUSION_TB")) p->diffusion_tb = env[0] != '0';
        if (p->diffusion_tb) {
            if (const char* env = std::getenv("SF_TB_RV")) p->tb_rv = std::atoi(env) == 2 ? 2 : 1;
            if (const char* env = std::getenv("SF_TB_TILE")) {
                const int t = std::atoi(env);
                if (p->dc.radius == 1 && (t == 48 || t == 56 || t == 64 || t == 72 || t == 80 || t == 96))
                    p->tb_tile = t;
            }
            const uint32_t box = static_cast<uint32_t>(sfb::diffusion_box(p->dc.radius, p->tb_tile));
            for (int s = 0; s < 2; ++s) {
                sfb::make_map_2d(&p->tm_dx[s], *p, p->slot[s], box);
                sfb::make_map_2d(&p->tm_dy[s], *p, p->dscratch[s], box);
            }
        }
        p->arg_names = {"u"};
        p->arg_bytes = {2 * d->nx * d->ny * 4};
        p->launches_per_step = 1;
        SF_CUDA(cudaStreamSynchronize(p->stream));
    });
    if (rc == SF_OK) *out = p.release();
    return rc;
}

void sf_plan_destroy(sf_plan* p) { delete p; }

// Plans whose folded constants come from elsewhere (the C-source front end
// sf-cuda-cc lifts them from the reference's generated kernel): same layout
// as sf_acoustic_constants' output.
int sf_acoustic_plan_create_ex(const sf_acoustic_desc* d, const float* c, const int* tsel,
                               int device, sf_plan** out) {
    if (!c || !tsel) return SF_ERR_INVALID;
    int rc = sf_acoustic_plan_create(d, device, out);
    if (rc != SF_OK) return rc;
    sf_plan* p = *out;
    rc = guard([&] {
        const bool fwd = d->forward != 0;
        const int want[3] = {0, fwd ? 2 : 3, fwd ? 3 : 2};
        for (int k = 0; k < 3; ++k)
            if (tsel[k] != want[k])
                throw Status(SF_ERR_INVALID, "time terms are not in the emitted order");
        p->ac.ce = c[0];
        p->ac.cm = c[1];
        for (int k = 0; k < 3; ++k) p->ac.tc[k] = c[2 + k];
        p->ac.c0 = c[5];
        for (int j = 0; j < 8; ++j) p->ac.cj[j] = j < p->ac.radius ? c[6 + j] : 0.0f;
        p->ac.src_scale = c[14];
        for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
        p->graphs.clear();
    });
    if (rc != SF_OK) {
        delete p;
        *out = nullptr;
    }
    return rc;
}

int sf_diffusion_plan_create_ex(const sf_diffusion_desc* d, float c0, int has_c0, const float* cj,
                                int device, sf_plan** out) {
    if (!cj) return SF_ERR_INVALID;
    int rc = sf_diffusion_plan_create(d, device, out);
    if (rc != SF_OK) return rc;
    (*out)->dc.c0 = c0;
    (*out)->dc.has_c0 = has_c0 != 0;
    for (int j = 0; j < 8; ++j) (*out)->dc.cj[j] = j < (*out)->dc.radius ? cj[j] : 0.0f;
    return SF_OK;
}

int sf_acoustic_plan_create_slab(const sf_acoustic_desc* d, const sf_slab_desc* sl, int device,
                                 sf_plan** out) {
    if (!out || !d || !sl) return SF_ERR_INVALID;
    *out = nullptr;
    auto p = std::make_unique<sf_plan>();
    p->kind = sf_plan::ACOUSTIC;
    int rc = guard([&] {
        if (d->ndim != 3) throw Status(SF_ERR_INVALID, "slab decomposition is 3D");
        const int64_t r = d->space_order / 2;
        const int64_t n0 = d->shape[0];
        if (sl->own_begin < 0 || sl->own_end > sl->global_n0 || sl->own_end - sl->own_begin < r ||
            sl->plane0 != std::max<int64_t>(sl->own_begin - r, 0) ||
            sl->plane0 + n0 != std::min<int64_t>(sl->own_end + r, sl->global_n0))
            throw Status(SF_ERR_INVALID,
                         "slab: shape[0] must be the owned planes plus r-deep halos, owned >= r");
        sfb::setup_acoustic(*p, d, device, false);
        for (int s = 0; s < 3; ++s) p->slot[s] = sfb::alloc_field(*p);
        p->slab = true;
        p->global_n0 = sl->global_n0;
        p->plane0 = sl->plane0;
        p->own_begin = sl->own_begin;
        p->own_end = sl->own_end;
        p->own_lo = static_cast<int>(sl->own_begin - sl->plane0);
        p->own_hi = static_cast<int>(sl->own_end - sl->plane0);
        p->has_lower = sl->own_begin > 0;
        p->has_upper = sl->own_end < sl->global_n0;
        p->z0 = static_cast<int>(std::max<int64_t>(sl->own_begin, r) - sl->plane0);
        p->z1 = static_cast<int>(std::min<int64_t>(sl->own_end, sl->global_n0 - r) - sl->plane0);
        SF_CUDA(cudaEventCreateWithFlags(&p->ev_copy, cudaEventDisableTiming));
        SF_CUDA(cudaEventCreateWithFlags(&p->ev_band, cudaEventDisableTiming));
        SF_CUDA(cudaEventCreateWithFlags(&p->ev_comm, cudaEventDisableTiming));
        SF_CUDA(cudaStreamCreateWithFlags(&p->comm, cudaStreamNonBlocking));
        if (const char* env = std::getenv("SF_NO_OVERLAP")) p->overlap_disabled = env[0] == '1';
        sfb::choose_geometry(*p);
        sfb::enable_tma(*p);
        SF_CUDA(cudaStreamSynchronize(p->stream));
    });
    if (rc == SF_OK) *out = p.release();
    return rc;
}

int sf_slab_chain_run(sf_plan* const* plans, int nplans, int64_t b, int64_t e) {
    return guard([&] {
        if (!plans || nplans < 1) throw Status(SF_ERR_INVALID, "no plans");
        for (int i = 0; i < nplans; ++i) {
            const sf_plan* p = plans[i];
            if (!p || !p->slab || p->kind != sf_plan::ACOUSTIC)
                throw Status(SF_ERR_INVALID, "chain needs acoustic slab plans");
            if (p->nt != plans[0]->nt || p->ac.radius != plans[0]->ac.radius ||
                p->plane != plans[0]->plane || p->ac.forward != plans[0]->ac.forward)
                throw Status(SF_ERR_INVALID, "chain plans disagree");
            if (i > 0 && plans[i - 1]->own_end != p->own_begin)
                throw Status(SF_ERR_INVALID, "chain slabs must be adjacent and ordered");
        }
        if (b < 0 || e > plans[0]->nt || b > e) throw Status(SF_ERR_INVALID, "step range");
        for (int i = 0; i < nplans; ++i) {  // all-zero eta boxes of each slab (its own planes)
            SF_CUDA(cudaSetDevice(plans[i]->device));
            sfb::ensure_eta_flags(*plans[i]);
            // the stencil's TMA producer reads the flag words before its
            // griddepcontrol.wait: the first (PDL) launch of the chain must not
            // overlap the flags kernel, so finish it here
            SF_CUDA(cudaStreamSynchronize(plans[i]->stream));
        }
        sfb::NvtxRange r("sf_slab_chain_run: time loop");
        for (int64_t k = b; k < e; ++k) sfb::chain_step(plans, nplans, k);
        for (int i = 0; i < nplans; ++i) sfb::check_kernel_errors(*plans[i]);
    });
}

int sf_nccl_unique_id(void* out, int bytes) {
    return guard([&] {
        if (bytes < 128) throw Status(SF_ERR_INVALID, "need 128 bytes");
        sfb::NcclId id;
        sfb::nccl_check(sfb::nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, id.internal, 128);
    });
}

int sf_plan_attach_nccl(sf_plan* p, const void* id, int nranks, int rank) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        if (!p->slab) throw Status(SF_ERR_INVALID, "NCCL exchange needs a slab plan");
        if (rank < 0 || rank >= nranks) throw Status(SF_ERR_INVALID, "rank out of range");
        SF_CUDA(cudaSetDevice(p->device));
        sfb::NcclId nid;
        std::memcpy(nid.internal, id, 128);
        void* comm = nullptr;
        sfb::nccl_check(sfb::nccl().CommInitRank(&comm, nranks, nid, rank), "ncclCommInitRank");
        p->nccl_comm = comm;
        p->nccl_rank = rank;
        p->nccl_nranks = nranks;
        for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
        p->graphs.clear();
    });
}

int sf_plan_num_args(const sf_plan* p) { return p ? static_cast<int>(p->arg_names.size()) : 0; }

const char* sf_plan_arg_name(const sf_plan* p, int i) {
    if (!p || i < 0 || i >= static_cast<int>(p->arg_names.size())) return nullptr;
    return p->arg_names[i].c_str();
}

int64_t sf_plan_arg_bytes(const sf_plan* p, int i) {
    if (!p || i < 0 || i >= static_cast<int>(p->arg_bytes.size())) return -1;
    return p->arg_bytes[i];
}

int sf_plan_upload(sf_plan* p, void* const* args, int nargs) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        sfb::NvtxRange r("sf_plan_upload");
        sfb::upload_any(*p, args, nargs);
    });
}

int sf_plan_download(sf_plan* p, void* const* args, int nargs) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        sfb::NvtxRange r("sf_plan_download");
        sfb::download_any(*p, args, nargs);
    });
}

int sf_plan_run(sf_plan* p, int64_t b, int64_t e) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind == sf_plan::FWI) throw Status(SF_ERR_INVALID, "use sf_fwi_gradient");
        if (b < 0 || e > p->nt || b > e) throw Status(SF_ERR_INVALID, "step range out of bounds");
        SF_CUDA(cudaSetDevice(p->device));
        sfb::NvtxRange r("sf_plan_run: time loop");
        sfb::run_steps(*p, b, e);
        SF_CUDA(cudaGetLastError());
    });
}

int sf_plan_synchronize(sf_plan* p) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] { sfb::check_kernel_errors(*p); });
}

int sf_plan_invoke(sf_plan* p, void* const* args, int nargs) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        if (p->kind == sf_plan::FWI) throw Status(SF_ERR_INVALID, "use sf_fwi_gradient");
        for (int i = 0; i < nargs; ++i)
            if (!args[i]) throw Status(SF_ERR_SIGNATURE, "null buffer for " + p->arg_names.at(i));
        sfb::NvtxRange whole("sf_plan_invoke");
        bool field_back = false;
        if (sfb::io_overlap_eligible(*p, args, nargs)) {
            sfb::NvtxRange r("time loop with the upload / download overlapped by its first / last steps");
            try {
                field_back = sfb::invoke_overlapped(*p, args);
            } catch (...) {
                // asynchronous copies may still reference the caller's buffers
                if (p->io) cudaStreamSynchronize(p->io);
                cudaStreamSynchronize(p->stream);
                throw;
            }
            sfb::check_kernel_errors(*p);
        } else {
            {
                sfb::NvtxRange r("upload (H2D + repack)");
                sfb::upload_any(*p, args, nargs);
            }
            sfb::NvtxRange r("time loop");
            sfb::run_steps(*p, 0, p->nt);
            sfb::check_kernel_errors(*p);
        }
        sfb::NvtxRange r("download (repack + D2H)");
        // only what the kernel writes comes back (the generated Operator
        // stores into the field and the sampled series; m, eta, the injected
        // series, ci and w are read-only, so the host copies already match)
        std::vector<void*> out(args, args + nargs);
        if (p->kind == sf_plan::ACOUSTIC)
            for (int i = 1; i < nargs; ++i)
                if (i != (p->ac.forward ? 6 : 3)) out[i] = nullptr;
        if (field_back) out[0] = nullptr;
        sfb::download_any(*p, out.data(), nargs);
    });
}

int sf_acoustic_apply(sf_plan* p, float* u, float* m, float* eta, float* src, int* src_ci,
                      float* src_w, float* rec, int* rec_ci, float* rec_w) {
    if (!p || p->kind != sf_plan::ACOUSTIC) {
        sfb::set_error("not an acoustic plan");
        return SF_ERR_SIGNATURE;
    }
    void* a[9] = {u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w};
    return sf_plan_invoke(p, a, 9);
}

int sf_diffusion_apply(sf_plan* p, float* u) {
    if (!p || p->kind != sf_plan::DIFFUSION) {
        sfb::set_error("not a diffusion plan");
        return SF_ERR_SIGNATURE;
    }
    void* a[1] = {u};
    return sf_plan_invoke(p, a, 1);
}

int sf_plan_time(sf_plan* p, float* total_ms, float* stencil_ms, int64_t* launches) {
    if (!p) return SF_ERR_INVALID;
    return guard([&] {
        SF_CUDA(cudaSetDevice(p->device));
        sfb::run_steps(*p, 0, p->nt);  // make sure the graph exists (warm)
        SF_CUDA(cudaStreamSynchronize(p->stream));
        SF_CUDA(cudaEventRecord(p->ev0, p->stream));
        sfb::run_steps(*p, 0, p->nt);
        SF_CUDA(cudaEventRecord(p->ev1, p->stream));
        sfb::check_kernel_errors(*p);
        float ms = 0;
        SF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
        if (total_ms) *total_ms = ms;
        if (launches)
            *launches = p->kind == sf_plan::DIFFUSION ? sfb::diffusion_launches(*p, p->nt)
                                                      : sfb::launches_per_step_of(*p) * p->nt +
                                                            (sfb::fused_sparse_active(*p) ? 1 : 0);
        if (stencil_ms) {
            // same steps with only the stencil launches: their summed duration
            sfb::run_steps(*p, sfb::kStencilOnly, sfb::kStencilOnly);
            SF_CUDA(cudaStreamSynchronize(p->stream));
            SF_CUDA(cudaEventRecord(p->ev0, p->stream));
            sfb::run_steps(*p, sfb::kStencilOnly, sfb::kStencilOnly);
            SF_CUDA(cudaEventRecord(p->ev1, p->stream));
            sfb::check_kernel_errors(*p);
            SF_CUDA(cudaEventElapsedTime(stencil_ms, p->ev0, p->ev1));
        }
    });
}

int sf_fwi_plan_create(const sf_acoustic_desc* d, int device, sf_plan** out) {
    if (!out) return SF_ERR_INVALID;
    *out = nullptr;
    auto p = std::make_unique<sf_plan>();
    p->kind = sf_plan::FWI;
    int rc = guard([&] {
        if (d && d->ndim != 3) throw Status(SF_ERR_INVALID, "FWI gradient is 3D only");
        sfb::setup_acoustic(*p, d, device, true);
        p->ac_fwd = p->ac;
        p->ac_adj = sfb::acoustic_constants(3, d->space_order, false, d->dt, d->spacing);
        const int64_t levels = d->nt + 2;
        p->hist = sfb::dalloc<float>(
            static_cast<size_t>(levels * p->slot_elems + sfb::field_slack(*p)));
        for (int s = 0; s < 3; ++s) p->v[s] = sfb::alloc_field(*p);
        p->grad = sfb::alloc_field(*p);
        sfb::enable_tma(*p);
        p->arg_names.clear();
        p->arg_bytes.clear();
        SF_CUDA(cudaStreamSynchronize(p->stream));
    });
    if (rc == SF_OK) *out = p.release();
    return rc;
}

int sf_fwi_gradient(sf_plan* p, const float* m, const float* eta, const float* src,
                    const int* src_ci, const float* src_w, const int* rec_ci, const float* rec_w,
                    const float* residual, float* rec_out, float* grad_out, float* v_out,
                    float* src_adj_out) {
    if (!p || p->kind != sf_plan::FWI) return SF_ERR_INVALID;
    return guard([&] {
        if (!m || !eta || !src || !src_ci || !src_w || !rec_ci || !rec_w || !residual)
            throw Status(SF_ERR_SIGNATURE, "null input buffer");
        SF_CUDA(cudaSetDevice(p->device));
        sfb::NvtxRange whole("sf_fwi_gradient");
        sfb::h2d_field(*p, p->m, m);
        sfb::h2d_field(*p, p->eta, eta);
        ++p->eta_gen;
        // forward: src injects, rec samples
        sfb::upload_points(*p, p->src, src, src_ci, src_w, true);
        sfb::upload_points(*p, p->rec, nullptr, rec_ci, rec_w, true);
        {
            sfb::NvtxRange r("FWI forward sweep (history)");
            sfb::run_steps(*p, sfb::kFwiForward, sfb::kFwiForward);
            sfb::check_kernel_errors(*p);
        }
        if (rec_out)
            SF_CUDA(cudaMemcpyAsync(rec_out, p->rec.series, sizeof(float) * p->nt * p->rec.np,
                                    cudaMemcpyDeviceToHost, p->stream));
        // adjoint: residual injected at receivers, source positions sampled
        SF_CUDA(cudaStreamSynchronize(p->stream));
        SF_CUDA(cudaMemcpyAsync(p->rec.series, residual, sizeof(float) * p->nt * p->rec.np,
                                cudaMemcpyHostToDevice, p->stream));
        {
            sfb::NvtxRange r("FWI adjoint + gradient sweep");
            sfb::run_steps(*p, sfb::kFwiAdjoint, sfb::kFwiAdjoint);
            sfb::check_kernel_errors(*p);
        }
        if (grad_out) sfb::d2h_field(*p, grad_out, p->grad);
        if (v_out)
            for (int s = 0; s < 3; ++s)
                sfb::d2h_field(*p, v_out + s * sfb::field_numel(*p), p->v[s]);
        if (src_adj_out)
            SF_CUDA(cudaMemcpyAsync(src_adj_out, p->src.series, sizeof(float) * p->nt * p->src.np,
                                    cudaMemcpyDeviceToHost, p->stream));
        SF_CUDA(cudaStreamSynchronize(p->stream));
    });
}

int sf_fwi_time(sf_plan* p, float* fwd_ms, float* adj_ms) {
    if (!p || p->kind != sf_plan::FWI) return SF_ERR_INVALID;
    return guard([&] {
        SF_CUDA(cudaSetDevice(p->device));
        SF_CUDA(cudaEventRecord(p->ev0, p->stream));
        sfb::run_steps(*p, sfb::kFwiForward, sfb::kFwiForward);
        SF_CUDA(cudaEventRecord(p->ev1, p->stream));
        sfb::check_kernel_errors(*p);
        SF_CUDA(cudaEventElapsedTime(fwd_ms, p->ev0, p->ev1));
        SF_CUDA(cudaEventRecord(p->ev0, p->stream));
        sfb::run_steps(*p, sfb::kFwiAdjoint, sfb::kFwiAdjoint);
        SF_CUDA(cudaEventRecord(p->ev1, p->stream));
        sfb::check_kernel_errors(*p);
        SF_CUDA(cudaEventElapsedTime(adj_ms, p->ev0, p->ev1));
    });
}

int sf_interpolation_weights(int ndim, const double* coord, double spacing,
                             const int64_t* extents, int32_t* cell, float* w) {
    if (ndim < 1 || ndim > 3) return SF_ERR_INVALID;
    return sfb::interpolation_weights(ndim, coord, spacing, extents, cell, w)
               ? SF_OK
               : SF_ERR_OUT_OF_DOMAIN;
}

double sf_stable_dt(int ndim, int order, double spacing, double v_top, double v_bottom) {
    try {
        return sfb::stable_dt(ndim, order, spacing, v_top, v_bottom);
    } catch (const std::exception& e) {
        sfb::set_error(e.what());
        return -1.0;
    }
}

double sf_ricker(double f0, double t, double t0) { return sfb::ricker(f0, t, t0); }

int sf_build_medium(int ndim, const int64_t* shape, int boundary_width, double spacing,
                    double v_top, double v_bottom, const double* v_field, double v_min, float* m,
                    float* eta) {
    if (ndim < 2 || ndim > 3 || !shape || !m || !eta) return SF_ERR_INVALID;
    sfb::build_medium(ndim, shape, boundary_width, spacing, v_top, v_bottom, v_field, v_min, m,
                      eta);
    return SF_OK;
}


int sf_smooth_extrema(const sf_smooth_medium_desc* d, int device, double* lo, double* hi) {
    if (!d || !lo || !hi) return SF_ERR_INVALID;
    return sfb::medium_guard([&] {
        SF_CUDA(cudaSetDevice(device));
        sfb::smooth_medium_run(*d, 0, lo, hi, nullptr, nullptr, 0, 0, nullptr);
    });
}

int sf_smooth_medium(const sf_smooth_medium_desc* d, double lo, double hi, int device, float* m,
                     float* eta) {
    if (!d || !m || !eta) return SF_ERR_INVALID;
    return sfb::medium_guard([&] {
        SF_CUDA(cudaSetDevice(device));
        if (d->shape[0] < 1 || d->shape[1] < 1 || d->shape[2] < 1 || d->a0_end <= d->a0_begin)
            throw sfb::Status(SF_ERR_INVALID, "smooth medium: empty range");
        const int64_t n12 = d->shape[1] * d->shape[2];
        const size_t n = static_cast<size_t>((d->a0_end - d->a0_begin) * n12);
        float *dm = nullptr, *de = nullptr;
        SF_CUDA(cudaMalloc(&dm, sizeof(float) * n));
        std::unique_ptr<float, decltype(&cudaFree)> gm(dm, &cudaFree);
        SF_CUDA(cudaMalloc(&de, sizeof(float) * n));
        std::unique_ptr<float, decltype(&cudaFree)> ge(de, &cudaFree);
        sfb::smooth_medium_run(*d, 1, &lo, &hi, dm, de, d->shape[2], n12, nullptr);
        SF_CUDA(cudaMemcpy(m, dm, sizeof(float) * n, cudaMemcpyDeviceToHost));
        SF_CUDA(cudaMemcpy(eta, de, sizeof(float) * n, cudaMemcpyDeviceToHost));
    });
}

int sf_plan_set_smooth_medium(sf_plan* p, const sf_smooth_medium_desc* d, double lo, double hi) {
    if (!p || !d) return SF_ERR_INVALID;
    return sfb::medium_guard([&] {
        if (p->kind == sf_plan::DIFFUSION || p->ndim != 3 || !p->m || !p->eta)
            throw sfb::Status(SF_ERR_INVALID, "smooth medium needs a 3D acoustic or FWI plan");
        if (d->shape[1] != p->n[1] || d->shape[2] != p->n[2] || d->shape[0] != p->global_n0)
            throw sfb::Status(SF_ERR_INVALID, "smooth medium: global shape does not match the plan");
        SF_CUDA(cudaSetDevice(p->device));
        sf_smooth_medium_desc dd = *d;
        dd.a0_begin = p->plane0;
        dd.a0_end = p->plane0 + p->n[0];
        sfb::smooth_medium_run(dd, 1, &lo, &hi, p->m, p->eta, p->pitch, p->plane, p->stream);
        ++p->eta_gen;
    });
}

int sf_acoustic_constants(int ndim, int order, int forward, double dt, double spacing,
                          float* out, int* tsel) {
    return guard([&] {
        sfb::AcousticConstants c = sfb::acoustic_constants(ndim, order, forward != 0, dt, spacing);
        std::fill(out, out + 15, 0.0f);
        out[0] = c.ce;
        out[1] = c.cm;
        for (int k = 0; k < 3; ++k) {
            out[2 + k] = c.tc[k];
            tsel[k] = c.tsel[k];
        }
        out[5] = c.c0;
        for (int j = 0; j < c.radius; ++j) out[6 + j] = c.cj[j];
        out[14] = c.src_scale;
    });
}

int sf_diffusion_constants(int order, int64_t an, int64_t ad, int64_t dn, int64_t dd, float* c0,
                           int* has_c0, float* cj) {
    return guard([&] {
        sfb::DiffusionConstants c =
            sfb::diffusion_constants(sfb::Rat::make(an, ad), sfb::Rat::make(dn, dd), order);
        *c0 = c.c0;
        *has_c0 = c.has_c0;
        for (int j = 0; j < 8; ++j) cj[j] = c.cj[j];
    });
}

} // extern "C"
