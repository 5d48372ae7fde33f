// libptyger runtime: context, C ABI entry points, CUDA-graph capture of one CG iteration and
// the NCCL plumbing for world > 1 (band exchange of partial gradients + fp64 allreduces of the
// DY and LS scalars).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host.h"
#include "internal.h"
#include "p2p.h"

using namespace pty;

namespace {

thread_local std::string g_last_error;

// ---------------- NCCL, loaded on demand (world == 1 never touches it) ----------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

NcclApi* nccl_api(std::string& err) {
    static NcclApi api;
    static bool tried = false;
    if (tried) {
        if (!api.ok) err = "NCCL library could not be loaded (set PTYGER_NCCL_LIB)";
        return api.ok ? &api : nullptr;
    }
    tried = true;
    const char* cands[] = {getenv("PTYGER_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* c : cands) {
        if (!c) continue;
        h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        err = "NCCL library could not be loaded (set PTYGER_NCCL_LIB)";
        return nullptr;
    }
#define LD(name, sym)                                                  \
    api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, sym));   \
    if (!api.name) {                                                   \
        err = std::string("NCCL symbol missing: ") + sym;              \
        return nullptr;                                                \
    }
    LD(GetUniqueId, "ncclGetUniqueId");
    LD(CommInitRank, "ncclCommInitRank");
    LD(CommDestroy, "ncclCommDestroy");
    LD(AllReduce, "ncclAllReduce");
    LD(Broadcast, "ncclBroadcast");
    LD(Send, "ncclSend");
    LD(Recv, "ncclRecv");
    LD(GroupStart, "ncclGroupStart");
    LD(GroupEnd, "ncclGroupEnd");
    LD(GetErrorString, "ncclGetErrorString");
#undef LD
    api.ok = true;
    return &api;
}

// Device buffers come from the device's default stream-ordered memory pool with the release
// threshold raised to "never": a context created after another one was destroyed (e.g. one
// reconstruction problem after another) reuses the mapped pages instead of paying cudaMalloc's
// page-mapping cost again.  Allocations / zero fills are on the legacy stream; init
// synchronises it before the context's own (non-blocking) stream uses the buffers.
void pool_setup(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

template <typename T>
T* dalloc(size_t count, std::string& err, bool zero = true) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMallocAsync(&p, count * sizeof(T), 0) != cudaSuccess) {
        cudaGetLastError();
        err = "cudaMallocAsync of " + std::to_string(count * sizeof(T)) + " bytes failed";
        return nullptr;
    }
    if (zero) cudaMemsetAsync(p, 0, count * sizeof(T), 0);
    return static_cast<T*>(p);
}

}  // namespace

struct ptyger_ctx {
    ptyger_config cfg{};
    SolverCfg sc{};
    int64_t H = 0, W = 0, n = 0;
    int N = 0;
    int sms = 148;
    // partition
    std::vector<int32_t> frame_rank;
    std::vector<int64_t> rows;   // P*6
    int64_t st_lo = 0, st_hi = 0, SH = 0;
    std::vector<int64_t> local_global;  // storage index -> global frame index
    Geometry geo{};
    // device
    float2 *psi = nullptr, *g[2] = {nullptr, nullptr}, *eta = nullptr, *u = nullptr, *v = nullptr,
           *probe = nullptr, *probe_s = nullptr, *full = nullptr, *recv[2] = {nullptr, nullptr};
    float* d = nullptr;
    int2* pos = nullptr;
    int* order = nullptr;
    int* tile_ptr = nullptr;
    int* entries = nullptr;
    float2* frac = nullptr;      // per storage frame fractional offsets (subpixel mode only)
    float* illum = nullptr;      // I = diag(G^H G) over the storage rows (object-grid LS moments, sc.qg)
    bool subpx = false;
    int ntx = 0, nty = 0;
    double *part_adj = nullptr, *part_fr = nullptr, *part_el = nullptr, *scratch = nullptr;
    int band_grid = 0;
    DevState* st = nullptr;
    ptyger_trace* d_tr = nullptr;
    int tr_cap = 0;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    cudaEvent_t ev_it[2] = {nullptr, nullptr};
    float last_ms = 0.f;
    int grid_fr = 0, grid_el = 0;
    int parts_ls = 0;    // per-CTA partial rows written by the LS pass-0 frame kernel(s)
    int ls_side = 0;     // N = 256: CTAs of the side LS kernel (c256_ls_side), 0 = none
    int m_host = 0;
    int pending_iters = 0;   // iterations launched by ptyger_cg_launch, not yet waited for
    int64_t launches_per_iter = 0, last_launches = 0;
    bool failed_numeric = false;
    // bands: [0] with rank-1, [1] with rank+1 (storage-local rows)
    int64_t band_lo[2] = {0, 0}, band_rows[2] = {0, 0};
    // peer-memory transport (cfg.transport == PTYGER_TRANSPORT_P2P, world > 1)
    bool p2p = false, connected = true;
    unsigned char* win = nullptr;        // own exchange window (cudaMalloc: IPC-exportable)
    P2PView pv{};
    uint64_t gather_epoch = 1;           // host mirror of the gather channel's epoch (buffer parity)
    // nccl
    NcclApi* nc = nullptr;
    ncclComm_t comm = nullptr;
    std::string err;
};

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            err = std::string(#call) + ": " + cudaGetErrorString(e_);                            \
            return PTYGER_E_CUDA;                                                                 \
        }                                                                                         \
    } while (0)

#define NK(call)                                                                                  \
    do {                                                                                          \
        ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess) {                                                                  \
            err = std::string(#call) + ": " + c->nc->GetErrorString(r_);                          \
            return PTYGER_E_NCCL;                                                                 \
        }                                                                                         \
    } while (0)

#define LK(call)                                                                                  \
    do {                                                                                          \
        if ((call) != 0) {                                                                        \
            err = std::string("kernel launch failed: ") + #call + ": " +                          \
                  cudaGetErrorString(cudaGetLastError());                                         \
            return PTYGER_E_CUDA;                                                                 \
        }                                                                                         \
    } while (0)

static ptyger_status set_err(ptyger_ctx* c, ptyger_status s, const std::string& m) {
    if (c)
        c->err = m;
    else
        g_last_error = m;
    return s;
}

// fp64 sum over ranks, in place on the device (NCCL or the peer-memory mailbox)
static int allreduce(ptyger_ctx* c, double* buf, int count, cudaStream_t s) {
    if (c->p2p) return launch_p2p_allreduce(buf, count, c->pv, c->st, s);
    return c->nc->AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, s) == ncclSuccess ? 0 : -1;
}

// ------------------------------------------------------------------------------------------
// One iteration as a sequence of launches on c->stream (captured into a graph).
// parity p: gcur = g[p], gprev = g[1-p].
// ------------------------------------------------------------------------------------------
static int enqueue_iteration(ptyger_ctx* c, int p, std::string& err, int64_t& launches) {
    const bool multi = c->cfg.world > 1;
    float2* gcur = c->g[p];
    float2* gprev = c->g[1 - p];
    cudaStream_t s = c->stream;
    const Geometry& g = c->geo;
    const SolverCfg& sc = c->sc;
    const float eps = (float)sc.eps;
    launches = 0;
    LK(launch_begin_iter(c->st, s)); ++launches;   // stage stamp 0
    // GRAD stage (Alg.1 648-649)
    LK(launch_grad(g, c->u, c->v, c->d, c->probe, c->probe_s, c->st, eps, c->grid_fr, s));
    ++launches;
    LK(launch_adj(g, c->v, c->tile_ptr, c->entries, c->ntx, c->nty, gcur, gprev, c->eta, c->part_adj, c->st, s,
                  (multi && c->p2p) ? &c->pv : nullptr));
    ++launches;
    int nparts = c->ntx * c->nty;
    if (multi) {
        LK(launch_stamp(c->st, 5, s));   // adjoint done, band exchange next
        ++launches;
    }
    if (multi && c->p2p) {
        // band exchange fused into k_adj (its band tiles stored into the neighbours' windows and its
        // last tile raised the flags); wait for the neighbours' bands, then add them
        LK(launch_p2p_wait_band(c->pv, c->st, c->band_rows[0] > 0, c->band_rows[1] > 0, s));
        launches += 1;
        for (int b = 0; b < 2; ++b) {
            if (c->band_rows[b] <= 0) continue;
            LK(launch_band_add(gcur, c->recv[b], c->band_lo[b], c->band_rows[b], c->W, gprev, c->eta, g.own_lo, g.own_hi,
                               c->part_adj + (int64_t)nparts * NDY, c->band_grid, s));
            ++launches;
            nparts += c->band_grid;
        }
    } else if (multi) {
        // band exchange of partial gradients with the two neighbours (replaces the paper's
        // pattern duplication + border exchange, R#15)
        NK(c->nc->GroupStart());
        const int peers[2] = {c->cfg.rank - 1, c->cfg.rank + 1};
        for (int b = 0; b < 2; ++b) {
            if (c->band_rows[b] <= 0) continue;
            const size_t cnt = (size_t)(c->band_rows[b] * c->W * 2);
            NK(c->nc->Send(gcur + c->band_lo[b] * c->W, cnt, ncclFloat32, peers[b], c->comm, s));
            NK(c->nc->Recv(c->recv[b], cnt, ncclFloat32, peers[b], c->comm, s));
        }
        NK(c->nc->GroupEnd());
        for (int b = 0; b < 2; ++b) {
            if (c->band_rows[b] <= 0) continue;
            LK(launch_band_add(gcur, c->recv[b], c->band_lo[b], c->band_rows[b], c->W, gprev, c->eta, g.own_lo, g.own_hi,
                               c->part_adj + (int64_t)nparts * NDY, c->band_grid, s));
            ++launches;
            nparts += c->band_grid;
        }
    }
    LK(launch_stamp(c->st, 1, s));   // GRAD stage done
    ++launches;
    const P2PView* fuse = (multi && c->p2p) ? &c->pv : nullptr;   // reduce + allreduce in one kernel
    // DIR stage (Alg.1 651-656) rides on the DY reduction unless an NCCL allreduce sits in between
    const bool fuse_dir = !(multi && !c->p2p);
    const PickArgs pkd = {2, 0, 0, 0, sc};
    LK(launch_reduce(c->part_adj, nparts, NDY, &c->st->dy[0], s, c->st, 0, 0, fuse, fuse_dir ? &pkd : nullptr));
    ++launches;
    if (multi && !c->p2p) LK(allreduce(c, &c->st->dy[0], NDY, s));
    // DIR stage (Alg.1 651-656)
    if (!fuse_dir) {
        LK(launch_dir(c->st, sc, s));
        ++launches;
    }
    LK(launch_eta(g, gcur, c->eta, sc.qg ? c->psi : nullptr, c->illum, c->st, c->part_el, c->grid_el, s)); ++launches;
    // ||eta||^2 and the object-grid moments: summed over ranks here with the peer-memory transport (NCCL:
    // with the pass-0 LS vector)
    LK(launch_reduce(c->part_el, c->grid_el, 4, &c->st->ls_pass[LS_ETA], s, c->st, 0, 0, fuse)); ++launches;
    LK(launch_stamp(c->st, 2, s));   // DIR stage done
    ++launches;
    // LS stage (Alg.1 659-668).  Pass 0 computes v = G eta and screens trials 0..K-1; every pass
    // is followed by an exact re-evaluation that runs only when the screening left it undecided;
    // further passes (trials pK..pK+K-1) run only while nothing was accepted.
    LK(launch_ls(g, c->eta, c->probe, c->probe_s, c->pos, c->order, c->u, c->v, c->d, sc, c->part_fr, c->grid_fr, c->st, s));
    launches += c->ls_side > 0 ? 2 : 1;   // N = 256: + the side kernel on the SMs the clusters leave idle
    // pass 0 evaluates keff trials (adaptive on the device, >= KMIN), later passes K each
    const int rest = sc.max_shrinks > KMIN ? sc.max_shrinks - KMIN : 0;
    const int k1 = ls_k1(sc);
    const int npass = 1 + (rest > 0 ? 1 : 0) + (rest > k1 ? (rest - k1 + sc.K - 1) / sc.K : 0);
    const int wscreen = LSP;
    for (int pass = 0; pass < npass; ++pass) {
        const bool fused = pass == 0;
        if (!fused) {
            LK(launch_lsx(g, c->u, c->v, c->d, sc, pass, false, c->part_el, c->grid_el, c->st, s));
            ++launches;
        }
        // the decision step rides on the reduction kernel unless an NCCL allreduce sits in between
        const bool fuse_pick = !(multi && !c->p2p);
        const PickArgs pk0 = {1, pass, 0, 0, sc}, pk1 = {1, pass, 1, pass == npass - 1, sc};
        LK(launch_reduce(fused ? c->part_fr : c->part_el, fused ? c->parts_ls : c->grid_el, wscreen,
                         &c->st->ls_pass[0], s, c->st, pass == 0 ? 0 : 1, pass, fuse, fuse_pick ? &pk0 : nullptr));
        ++launches;
        if (multi && !c->p2p) LK(allreduce(c, &c->st->ls_pass[0], LSW, s));
        if (!fuse_pick) {
            LK(launch_pick(c->st, sc, pass, 0, 0, s));
            ++launches;
        }
        LK(launch_lsx(g, c->u, c->v, c->d, sc, pass, true, c->part_el, c->grid_el, c->st, s)); ++launches;
        LK(launch_reduce(c->part_el, c->grid_el, LSP, &c->st->ls_pass[0], s, c->st, 2, pass, fuse,
                         fuse_pick ? &pk1 : nullptr));
        ++launches;
        if (multi && !c->p2p) LK(allreduce(c, &c->st->ls_pass[0], KC, s));
        if (!fuse_pick) {
            LK(launch_pick(c->st, sc, pass, 1, pass == npass - 1, s));
            ++launches;
        }
    }
    LK(launch_stamp(c->st, 3, s));   // LS stage done
    ++launches;
    // Update stage (Alg.1 672)
    LK(launch_upd(g, c->psi, c->eta, c->st, c->grid_el, s)); ++launches;
    LK(launch_stamp(c->st, 4, s));   // Update done: stage ms into the trace entry
    ++launches;
    return 0;
}

static int build_graphs_on(ptyger_ctx* c, std::string& err);

// Captured on a private stream, so the context stream may still be busy with the uploads and
// the d validation while the graphs are built (the graphs are launched on c->stream later).
static int build_graphs(ptyger_ctx* c, std::string& err) {
    cudaStream_t cap = nullptr, own = c->stream;
    CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    c->stream = cap;
    const int rc = build_graphs_on(c, err);
    c->stream = own;
    cudaStreamDestroy(cap);
    return rc;
}

static int build_graphs_on(ptyger_ctx* c, std::string& err) {
    for (int p = 0; p < 2; ++p) {
        if (c->graph[p]) {
            cudaGraphExecDestroy(c->graph[p]);
            c->graph[p] = nullptr;
        }
        cudaGraph_t gr = nullptr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int64_t launches = 0;
        const int rc = enqueue_iteration(c, p, err, launches);
        cudaGraph_t tmp = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(c->stream, &tmp);
        if (rc) {
            if (tmp) cudaGraphDestroy(tmp);
            return rc;
        }
        if (ce != cudaSuccess) {
            err = std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce);
            return PTYGER_E_CUDA;
        }
        gr = tmp;
        CK(cudaGraphInstantiate(&c->graph[p], gr, 0));
        cudaGraphDestroy(gr);
        c->launches_per_iter = launches;
    }
    return 0;
}

// u = G psi and F(psi) (by definition) -> st->F, gamma = 0
static int run_forward(ptyger_ctx* c, std::string& err) {
    const Geometry& g = c->geo;
    LK(launch_fwd(g, c->psi, c->probe, c->pos, c->order, c->d, c->u, c->part_fr, c->grid_fr, (float)c->sc.eps, c->stream));
    LK(launch_reduce(c->part_fr, c->grid_fr, 1, c->scratch, c->stream));
    if (c->cfg.world > 1 && allreduce(c, c->scratch, 1, c->stream) != 0) {
        err = "allreduce(F0) failed";
        return c->p2p ? PTYGER_E_CUDA : PTYGER_E_NCCL;
    }
    LK(launch_set_F(c->st, c->scratch, c->sc.K, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

static void free_ctx(ptyger_ctx* c) {
    if (!c) return;
    for (int p = 0; p < 2; ++p)
        if (c->graph[p]) cudaGraphExecDestroy(c->graph[p]);
    if (c->p2p) c->full = c->recv[0] = c->recv[1] = nullptr;   // inside the exchange window
    void* ptrs[] = {c->psi, c->g[0], c->g[1], c->eta, c->u, c->v, c->probe, c->probe_s, c->full, c->recv[0], c->recv[1], c->d,
                    c->pos, c->order, c->frac, c->tile_ptr, c->entries, c->part_adj, c->part_fr, c->part_el, c->scratch, c->st,
                    c->d_tr, c->illum};
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (void* p : ptrs)
        if (p) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    for (int i = 0; i < 2; ++i)
        if (c->ev_it[i]) cudaEventDestroy(c->ev_it[i]);
    if (c->comm && c->nc) c->nc->CommDestroy(c->comm);
    if (c->p2p) {
        for (int r = 0; r < c->pv.world; ++r)
            if (r != c->cfg.rank && c->pv.win[r]) cudaIpcCloseMemHandle(c->pv.win[r]);
        if (c->win) cudaFree(c->win);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

extern "C" {

void ptyger_config_default(ptyger_config* cfg) {
    if (!cfg) return;
    cfg->gamma0 = 1.0;
    cfg->tau = 0.5;
    cfg->t = 0.0;
    cfg->eps = 1e-16;
    cfg->max_shrinks = 32;
    cfg->direction = PTYGER_DIR_DY;
    cfg->ls_batch = 16;
    cfg->estimator = PTYGER_EST_ML;
    cfg->device = 0;
    cfg->rank = 0;
    cfg->world = 1;
    cfg->transport = PTYGER_TRANSPORT_P2P;
    cfg->nccl_id = nullptr;
}

const char* ptyger_version(void) { return "ptyger-b200 0.1 (sm_100a)"; }

const char* ptyger_last_error(const ptyger_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

int64_t ptyger_kernel_launches(const ptyger_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

ptyger_status ptyger_round_positions(const float* raw, int64_t n, int32_t* out) {
    if (!raw || !out || n < 0) return set_err(nullptr, PTYGER_E_ARG, "round_positions: null pointer or n < 0");
    round_positions(raw, n, out);
    return PTYGER_OK;
}

ptyger_status ptyger_partition(const int32_t* scan, int64_t n, int64_t H, int32_t N, int32_t P,
                               int32_t* frame_rank, int64_t* rows) {
    if (!scan || !frame_rank || !rows) return set_err(nullptr, PTYGER_E_ARG, "partition: null pointer");
    std::vector<int32_t> rk;
    std::vector<int64_t> rw;
    std::string err;
    const int rc = partition(scan, n, H, N, P, rk, rw, err);
    if (rc) return set_err(nullptr, (ptyger_status)rc, err);
    std::memcpy(frame_rank, rk.data(), sizeof(int32_t) * n);
    std::memcpy(rows, rw.data(), sizeof(int64_t) * rw.size());
    return PTYGER_OK;
}

ptyger_status ptyger_nccl_unique_id(void* out128) {
    std::string err;
    NcclApi* api = nccl_api(err);
    if (!api) return set_err(nullptr, PTYGER_E_NCCL, err);
    ncclUniqueId id;
    ncclResult_t r = api->GetUniqueId(&id);
    if (r != ncclSuccess) return set_err(nullptr, PTYGER_E_NCCL, api->GetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
    return PTYGER_OK;
}

ptyger_status ptyger_fft2(const float* in, float* out, int32_t N, int64_t batch, int32_t inverse, void* stream) {
    if (!in || !out || batch < 0) return set_err(nullptr, PTYGER_E_ARG, "fft2: null pointer or batch < 0");
    if (N != 16 && N != 32 && N != 64 && N != 128 && N != 256)
        return set_err(nullptr, PTYGER_E_ARG, "fft2: N must be 16, 32, 64, 128 or 256");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(nullptr, PTYGER_E_CUDA, "fft2: no CUDA device");
    }
    if (batch == 0) return PTYGER_OK;
    const int rc = launch_fft2(reinterpret_cast<const float2*>(in), reinterpret_cast<float2*>(out), N, batch,
                               inverse != 0, (cudaStream_t)stream);
    if (rc) return set_err(nullptr, PTYGER_E_CUDA, std::string("fft2 launch: ") + cudaGetErrorString(cudaGetLastError()));
    return PTYGER_OK;
}

// fr: nullptr, or 2n fractional offsets (row, col) in [0, 1) of bilinear windows at the integer
// corners scan (ptyger_init_subpixel, R#22); all-zero offsets take the integer path unchanged.
// PTYGER_INIT_TRACE=1: wall-clock milestones of ptyger_init on stderr (where init time goes)
static void init_trace(const char* what) {
    static const bool on = getenv("PTYGER_INIT_TRACE") && atoi(getenv("PTYGER_INIT_TRACE")) == 1;
    static std::chrono::steady_clock::time_point t0;
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    if (what[0] == '^') t0 = t;
    fprintf(stderr, "[ptyger init] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
}

static ptyger_status init_impl(ptyger_ctx* c, const float* object, const float* probe, const int32_t* scan,
                               const float* intensities, const float* fr = nullptr) {
    init_trace("^start");
    std::string& err = c->err;
    const ptyger_config& cfg = c->cfg;
    const int N = c->N;
    const int64_t H = c->H, W = c->W, n = c->n;
    if (fr)
        for (int64_t i = 0; i < 2 * n; ++i)
            if (fr[i] != 0.0f) c->subpx = true;
    // the LS trials' non-log part from the object grid (G^H G = diag(I)): Poisson ML, integer positions
    c->sc.qg = (c->sc.est == PTYGER_EST_ML && !c->subpx) ? 1 : 0;
    // ---- partition (host) ----
    const int foot = N + (c->subpx ? 1 : 0);
    const int rc = partition(scan, n, H, N, cfg.world, c->frame_rank, c->rows, err, foot);
    init_trace("partition");
    if (rc) return (ptyger_status)rc;
    const int me = cfg.rank;
    const int64_t* R = &c->rows[6 * me];
    c->st_lo = R[4];
    c->st_hi = R[5];
    c->SH = c->st_hi - c->st_lo;
    for (int64_t j = 0; j < n; ++j)
        if (c->frame_rank[j] == me) c->local_global.push_back(j);
    const int64_t nl = (int64_t)c->local_global.size();
    // bands (storage-local)
    if (cfg.world > 1) {
        if (me > 0) {
            const int64_t lo = R[2], hi = c->rows[6 * (me - 1) + 3];
            if (hi > lo) { c->band_lo[0] = lo - c->st_lo; c->band_rows[0] = hi - lo; }
        }
        if (me + 1 < cfg.world) {
            const int64_t lo = c->rows[6 * (me + 1) + 2], hi = R[3];
            if (hi > lo) { c->band_lo[1] = lo - c->st_lo; c->band_rows[1] = hi - lo; }
        }
    }
    Geometry& g = c->geo;
    g.N = N;
    g.W = W;
    g.SH = c->SH;
    g.own_lo = R[0] - c->st_lo;
    g.own_hi = R[1] - c->st_lo;
    g.band_lo0 = c->band_lo[0];
    g.band_hi0 = c->band_lo[0] + c->band_rows[0];
    g.band_lo1 = c->band_lo[1];
    g.band_hi1 = c->band_lo[1] + c->band_rows[1];
    g.n_local = nl;
    g.est = cfg.estimator;
    // local positions and canonical processing order
    std::vector<int32_t> lpos(2 * nl);
    std::vector<int32_t> sub(2 * nl);
    for (int64_t i = 0; i < nl; ++i) {
        const int64_t j = c->local_global[i];
        lpos[2 * i] = (int32_t)(scan[2 * j] - c->st_lo);
        lpos[2 * i + 1] = scan[2 * j + 1];
        sub[2 * i] = scan[2 * j];
        sub[2 * i + 1] = scan[2 * j + 1];
    }
    // canonical order and tile lists are built on the host AFTER the big uploads are issued (below)
    std::vector<int32_t> ord, tptr, ent;

    // ---- device ----
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        err = "no CUDA device (libptyger has no CPU fallback)";
        return PTYGER_E_CUDA;
    }
    if (cfg.device < 0 || cfg.device >= ndev) {
        err = "config.device out of range";
        return PTYGER_E_ARG;
    }
    CK(cudaSetDevice(cfg.device));
    pool_setup(cfg.device);
    init_trace("device set");
    CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, cfg.device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->p2p = cfg.world > 1 && cfg.transport == PTYGER_TRANSPORT_P2P;
    if (cfg.world > 1 && !c->p2p) {
        c->nc = nccl_api(err);
        if (!c->nc) return PTYGER_E_NCCL;
        ncclUniqueId id;
        std::memcpy(&id, cfg.nccl_id, sizeof(id));
        NK(c->nc->CommInitRank(&c->comm, cfg.world, id, cfg.rank));
    }
    const int64_t obj = c->SH * W;
    const int64_t NN = (int64_t)N * N;
#define AL(ptr, T, cnt)                                  \
    do {                                                 \
        ptr = dalloc<T>((size_t)(cnt), err);             \
        if (!ptr) return PTYGER_E_OOM;                   \
    } while (0)
    AL(c->psi, float2, obj);
    AL(c->g[0], float2, obj);
    AL(c->g[1], float2, obj);
    AL(c->eta, float2, obj);
    // u is written by k_fwd, d by the upload, v by the first LS pass before any read: no zero fill
#define ALN(ptr, T, cnt)                                       \
    do {                                                       \
        ptr = dalloc<T>((size_t)(cnt), err, false);            \
        if (!ptr) return PTYGER_E_OOM;                         \
    } while (0)
    ALN(c->u, float2, nl * NN);
    ALN(c->v, float2, nl * NN);
    ALN(c->d, float, nl * NN);
#undef ALN
    AL(c->probe, float2, NN);
    AL(c->pos, int2, nl);
    AL(c->order, int, nl);
    if (c->subpx) AL(c->frac, float2, nl);
    c->grid_fr = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms, nl));
    c->grid_el = c->sms * 8;
    c->band_grid = c->sms * 2;
    // N = 256: the LS pass runs on clusters of four CTAs (large config: 96.7 -> 71.6 ms against the
    // v-slot transpose kernel); the GRAD pass keeps the v-slot kernel (kernels_n256.cu)
    c->parts_ls = N == 256 ? c256_ls_parts(nl, c->sc.side) : c->grid_fr;
    c->ls_side = N == 256 ? c256_ls_side(nl, c->sc.side) : 0;
    if (c->parts_ls <= 0) {
        err = "cluster LS kernel setup failed";
        return PTYGER_E_CUDA;
    }
    AL(c->probe_s, float2, NN);
    AL(c->part_fr, double, (int64_t)std::max(c->grid_fr, c->parts_ls) * LSW);
    AL(c->part_el, double, (int64_t)c->grid_el * LSW);
    AL(c->scratch, double, 64);
    AL(c->st, DevState, 1);
    if (c->p2p) {
        // exchange window layout, identical arithmetic on every rank (p2p.h)
        P2PView& v = c->pv;
        v.world = cfg.world;
        v.rank = cfg.rank;
        v.off_flags = 0;
        v.off_mail = 4096;
        v.off_full = v.off_mail + (int64_t)2 * P2P_MAX_RANKS * P2P_MBW * 8;
        v.full_elems = H * W;
        auto up = [](int64_t x) { return (x + 255) / 256 * 256; };
        int64_t my_bytes = 0;
        for (int r = 0; r < cfg.world; ++r) {
            const int64_t* Rr = &c->rows[6 * r];
            int64_t b0 = 0, b1 = 0;
            if (r > 0) b0 = std::max<int64_t>(0, c->rows[6 * (r - 1) + 3] - Rr[2]);
            if (r + 1 < cfg.world) b1 = std::max<int64_t>(0, Rr[3] - c->rows[6 * (r + 1) + 2]);
            v.off_recv0[r] = up(v.off_full + 2 * H * W * 8);
            v.off_recv1[r] = up(v.off_recv0[r] + b0 * W * 8);
            if (r == cfg.rank) my_bytes = up(v.off_recv1[r] + b1 * W * 8);
        }
        void* wp = nullptr;
        if (cudaMalloc(&wp, (size_t)my_bytes) != cudaSuccess) {
            cudaGetLastError();
            err = "cudaMalloc of the " + std::to_string(my_bytes) + "-byte exchange window failed";
            return PTYGER_E_OOM;
        }
        CK(cudaMemset(wp, 0, (size_t)my_bytes));
        c->win = static_cast<unsigned char*>(wp);
        v.win[cfg.rank] = c->win;
        c->full = reinterpret_cast<float2*>(c->win + v.off_full);
        c->recv[0] = c->band_rows[0] > 0 ? reinterpret_cast<float2*>(c->win + v.off_recv0[cfg.rank]) : nullptr;
        c->recv[1] = c->band_rows[1] > 0 ? reinterpret_cast<float2*>(c->win + v.off_recv1[cfg.rank]) : nullptr;
    } else {
        for (int b = 0; b < 2; ++b)
            if (c->band_rows[b] > 0) AL(c->recv[b], float2, c->band_rows[b] * W);
        if (cfg.world > 1) AL(c->full, float2, H * W);
    }
#undef AL
    CK(cudaStreamSynchronize(0));  // pool allocations and zero fills (legacy stream) are done
    init_trace("allocations");
    // Uploads are asynchronous (from pinned host memory the DMA of d overlaps the host work and the
    // graph capture below; pageable sources are staged before each call returns, so the host
    // vectors below may go out of scope).  d first, contiguous runs of local frames, on an upload
    // stream of its own: the small pageable copies on the context stream below would otherwise
    // block the host until the whole d DMA ahead of them had drained (measured: init 39-54 ms for
    // a 29.5 ms DMA of d at the paper config).  The context stream joins it before validating d.
    cudaStream_t up = nullptr;
    cudaEvent_t up_done = nullptr;
    CK(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&up_done, cudaEventDisableTiming));
    struct UpGuard {
        cudaStream_t& s;
        cudaEvent_t& e;
        ~UpGuard() {
            if (s) cudaStreamSynchronize(s);   // error paths: no DMA into d may outlive init
            if (e) cudaEventDestroy(e);
            if (s) cudaStreamDestroy(s);
        }
    } up_guard{up, up_done};
    // local frames [i0, i1) of d in contiguous runs.  Host-to-device copies drain in issue order,
    // and a pageable copy returns only once it is staged, i.e. after everything issued before it:
    // so half of d goes first (its DMA, 15 ms at paper scale, covers the host work below: 6-12 ms
    // measured), then psi, the small tables and the transform u_0 = G psi_0, then the rest of d
    // while that transform runs.
    auto issue_d = [&](int64_t i0, int64_t i1) -> cudaError_t {
        for (int64_t i = i0; i < i1;) {
            int64_t k = i;
            while (k + 1 < i1 && c->local_global[k + 1] == c->local_global[k] + 1) ++k;
            const int64_t j0 = c->local_global[i];
            const cudaError_t e = cudaMemcpyAsync(c->d + i * NN, intensities + j0 * NN, sizeof(float) * NN * (k - i + 1),
                                                  cudaMemcpyDefault, up);
            if (e != cudaSuccess) return e;
            i = k + 1;
        }
        return cudaSuccess;
    };
    const int64_t d_first = nl / 2;
    CK(issue_d(0, d_first));
    init_trace("d upload (1/2) issued");
    CK(cudaMemcpyAsync(c->psi, object + 2 * c->st_lo * W, sizeof(float2) * obj, cudaMemcpyDefault, c->stream));
    CK(cudaMemcpyAsync(c->probe, probe, sizeof(float2) * NN, cudaMemcpyDefault, c->stream));
    // probe / N (exact: N is a power of two) carries the unitary FFT scale of the frame kernels
    LK(launch_scale_c(c->probe, c->probe_s, NN, 1.0f / (float)N, c->stream));
    // host work while the DMA runs: canonical processing order and the tile -> frame lists
    {
        std::vector<int64_t> ord64;
        canonical_order(sub.data(), nl, N, ord64);
        ord.assign(ord64.begin(), ord64.end());
        build_tiles(lpos, ord, foot, c->SH, W, c->ntx, c->nty, tptr, ent);
        c->tile_ptr = dalloc<int>(tptr.size(), err, false);
        c->entries = dalloc<int>(ent.size(), err, false);
        if (!c->tile_ptr || !c->entries) return PTYGER_E_OOM;
        c->part_adj = dalloc<double>(((int64_t)c->ntx * c->nty + 2 * c->band_grid) * NDY, err);
        if (!c->part_adj) return PTYGER_E_OOM;
        CK(cudaStreamSynchronize(0));   // the pool allocations above (legacy stream) are done
    }
    init_trace("order + tiles built");
    std::vector<int2> p2(nl);
    for (int64_t i = 0; i < nl; ++i) p2[i] = make_int2(lpos[2 * i], lpos[2 * i + 1]);
    CK(cudaMemcpyAsync(c->pos, p2.data(), sizeof(int2) * nl, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->order, ord.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, c->stream));
    std::vector<float2> fl;
    if (c->subpx) {
        fl.resize(nl);
        for (int64_t i = 0; i < nl; ++i) {
            const int64_t j = c->local_global[i];
            fl[i] = make_float2(fr[2 * j], fr[2 * j + 1]);
        }
        CK(cudaMemcpyAsync(c->frac, fl.data(), sizeof(float2) * nl, cudaMemcpyHostToDevice, c->stream));
        c->geo.frac = c->frac;
    }
    CK(cudaMemcpyAsync(c->tile_ptr, tptr.data(), sizeof(int) * tptr.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->entries, ent.data(), sizeof(int) * ent.size(), cudaMemcpyHostToDevice, c->stream));
    if (c->sc.qg) {
        c->illum = dalloc<float>((size_t)(c->SH * W), err, false);
        if (!c->illum) return PTYGER_E_OOM;
        LK(launch_illum(c->geo, c->probe, c->tile_ptr, c->entries, c->ntx, c->nty, c->illum, c->stream));
    }
    init_trace("small uploads issued");
    unsigned long long* bad = dalloc<unsigned long long>(1, err, false);
    if (!bad) return PTYGER_E_OOM;
    {
        const unsigned long long init = ~0ull;
        CK(cudaMemcpyAsync(bad, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    }
    DevState hs;
    std::memset(&hs, 0, sizeof(hs));
    hs.tk_start[0] = hs.tk_start[1] = ~0ull;   // disarmed frame-kernel timers
    for (int ch = 0; ch < 4; ++ch) hs.p2p_epoch[ch] = 1;   // peer flags start at 0
    CK(cudaMemcpyAsync(c->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
    auto check_bad = [&]() -> ptyger_status {
        unsigned long long hb = 0;
        CK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        cudaFreeAsync(bad, 0);
        if (hb != ~0ull) {
            err = "intensities: frame " + std::to_string(c->local_global[(int64_t)hb]) +
                  " has a negative or non-finite value";
            return PTYGER_E_DATA;
        }
        return PTYGER_OK;
    };
    // u_0 = G psi_0 needs no d: the transform runs while the rest of d is in flight (F(psi_0) below)
    if (!c->p2p)
        LK(launch_fwd(c->geo, c->psi, c->probe, c->pos, c->order, nullptr, c->u, c->part_fr, c->grid_fr,
                      (float)c->sc.eps, c->stream));
    CK(issue_d(d_first, nl));
    CK(cudaEventRecord(up_done, up));
    init_trace("d upload issued");
    if (c->p2p) {   // the forward pass and the graphs need the peers: ptyger_ipc_connect
        CK(cudaStreamWaitEvent(c->stream, up_done, 0));   // d has landed
        LK(launch_validate_d(c->d, nl * NN, NN, bad, c->stream));
        const ptyger_status rs = check_bad();
        if (rs != PTYGER_OK) return rs;
        c->connected = false;
        return PTYGER_OK;
    }
    int rc2 = build_graphs(c, err);   // host-side capture + instantiation overlaps the uploads
    init_trace("graphs built");
    if (rc2) {
        cudaStreamSynchronize(c->stream);
        cudaFreeAsync(bad, 0);
        return (ptyger_status)rc2;
    }
    // d has landed: check it and form F(psi_0) (Eq.2) from u_0 and d in one pass
    CK(cudaStreamWaitEvent(c->stream, up_done, 0));
    // grid: 4 CTAs of 512 per SM (part_fr holds >= grid_fr * LSW >= that many partials)
    const int f0_grid = (int)std::min<int64_t>((int64_t)c->grid_fr * 4, std::max<int64_t>(1, nl * NN / 2048));
    LK(launch_f0_validate(c->u, c->d, nl * NN, NN, bad, c->part_fr, f0_grid, (float)c->sc.eps, c->geo.est,
                          c->stream));
    LK(launch_reduce(c->part_fr, f0_grid, 1, c->scratch, c->stream));
    if (cfg.world > 1 && allreduce(c, c->scratch, 1, c->stream) != 0) {
        cudaStreamSynchronize(c->stream);
        cudaFreeAsync(bad, 0);
        err = "allreduce(F0) failed";
        return PTYGER_E_NCCL;
    }
    LK(launch_set_F(c->st, c->scratch, c->sc.K, c->stream));
    const ptyger_status rs = check_bad();
    init_trace("F0 + d check done");
    return rs;
}

static ptyger_status create_ctx(ptyger_ctx** out, const ptyger_config* cfg_in, const float* object, int64_t H,
                                int64_t W, const float* probe, int32_t N, const int32_t* scan, int64_t n,
                                const float* intensities, const float* fr) {
    if (!out) return set_err(nullptr, PTYGER_E_ARG, "init: out is NULL");
    *out = nullptr;
    ptyger_config cfg;
    if (cfg_in)
        cfg = *cfg_in;
    else
        ptyger_config_default(&cfg);
    if (!object || !probe || !scan || !intensities) return set_err(nullptr, PTYGER_E_ARG, "init: null input array");
    if (!(cfg.gamma0 > 0) || !(cfg.tau > 0 && cfg.tau < 1) || !(cfg.eps > 0) || cfg.max_shrinks < 1 ||
        cfg.max_shrinks > SMAX || cfg.ls_batch < KMIN || cfg.ls_batch > KC || cfg.direction < 0 ||
        cfg.direction > PTYGER_DIR_GD || cfg.estimator < 0 || cfg.estimator > PTYGER_EST_LS || cfg.world < 1 ||
        cfg.rank < 0 || cfg.rank >= cfg.world ||
        (cfg.world > 1 && cfg.transport == PTYGER_TRANSPORT_NCCL && !cfg.nccl_id) ||
        (cfg.transport == PTYGER_TRANSPORT_P2P && cfg.world > P2P_MAX_RANKS) ||
        (cfg.transport != PTYGER_TRANSPORT_NCCL && cfg.transport != PTYGER_TRANSPORT_P2P) || !std::isfinite(cfg.t))
        return set_err(nullptr, PTYGER_E_ARG,
                       "init: bad config (need gamma0>0, 0<tau<1, eps>0, 1<=max_shrinks<=64, 4<=ls_batch<=16, "
                       "direction in {0,1,2}, 0<=rank<world, nccl_id when world>1)");
    if (N != 16 && N != 32 && N != 64 && N != 128 && N != 256)
        return set_err(nullptr, PTYGER_E_ARG, "init: N must be 16, 32, 64, 128 or 256");
    if (H < N || W < N) return set_err(nullptr, PTYGER_E_DATA, "init: object smaller than the probe");
    if (n < 1) return set_err(nullptr, PTYGER_E_DATA, "init: need at least one scan position");
    for (int64_t j = 0; j < n; ++j) {
        const int64_t r = scan[2 * j], cc = scan[2 * j + 1];
        // a bilinear window with a nonzero fraction also reads the row / column after the window
        const int64_t er = fr && fr[2 * j] != 0.0f ? 1 : 0, ec = fr && fr[2 * j + 1] != 0.0f ? 1 : 0;
        if (r < 0 || r + er > H - N || cc < 0 || cc + ec > W - N)
            return set_err(nullptr, PTYGER_E_DATA,
                           "init: scan position of frame " + std::to_string(j) + " (" + std::to_string(r) + ", " +
                               std::to_string(cc) + ") puts the window outside the object");
    }
    ptyger_ctx* c = new ptyger_ctx();
    c->cfg = cfg;
    c->sc.gamma0 = cfg.gamma0;
    c->sc.tau = cfg.tau;
    c->sc.t = cfg.t;
    c->sc.eps = cfg.eps;
    c->sc.max_shrinks = cfg.max_shrinks;
    c->sc.direction = cfg.direction;
    c->sc.K = cfg.ls_batch;
    // margin of the adaptive pass-0 trial count over the previous k* (experiments: PTYGER_KEFF_ADD)
    c->sc.kadd = getenv("PTYGER_KEFF_ADD") ? atoi(getenv("PTYGER_KEFF_ADD")) : 3;
    if (c->sc.kadd < 0) c->sc.kadd = 0;
    // N = 256: share of the frames (per mille) for the LS side kernel on the SMs the clusters leave idle
    c->sc.side = getenv("PTYGER_C256_SIDE") ? atoi(getenv("PTYGER_C256_SIDE")) : 110;
    c->sc.est = cfg.estimator;
    if (cfg.direction == PTYGER_DIR_GD) c->sc.max_shrinks = 1;   // Eq.4: one fixed step gamma0
    c->H = H;
    c->W = W;
    c->N = N;
    c->n = n;
    const ptyger_status s = init_impl(c, object, probe, scan, intensities, fr);
    if (s != PTYGER_OK) {
        g_last_error = c->err;
        free_ctx(c);
        return s;
    }
    *out = c;
    return PTYGER_OK;
}

ptyger_status ptyger_init(ptyger_ctx** out, const ptyger_config* cfg_in, const float* object, int64_t H, int64_t W,
                          const float* probe, int32_t N, const int32_t* scan, int64_t n, const float* intensities) {
    return create_ctx(out, cfg_in, object, H, W, probe, N, scan, n, intensities, nullptr);
}

// Fractional positions (R#22): integer corner floor(x) (exact in double) and fraction x - floor(x)
// (exact in float32: x and floor(x) share the exponent range).
static ptyger_status split_positions(const float* scan_f, int64_t n, std::vector<int32_t>& base,
                                     std::vector<float>& frac) {
    base.resize(2 * n);
    frac.resize(2 * n);
    for (int64_t i = 0; i < 2 * n; ++i) {
        const double x = (double)scan_f[i];
        if (!std::isfinite(x) || x < 0.0 || x > 2.0e9)
            return set_err(nullptr, PTYGER_E_DATA,
                           "init_subpixel: scan position of frame " + std::to_string(i / 2) + " is negative or not finite");
        const double f = std::floor(x);
        base[i] = (int32_t)f;
        frac[i] = (float)(x - f);
    }
    return PTYGER_OK;
}

ptyger_status ptyger_init_subpixel(ptyger_ctx** out, const ptyger_config* cfg, const float* object, int64_t H,
                                   int64_t W, const float* probe, int32_t N, const float* scan, int64_t n,
                                   const float* intensities) {
    if (!out) return set_err(nullptr, PTYGER_E_ARG, "init: out is NULL");
    if (!scan) return set_err(nullptr, PTYGER_E_ARG, "init: null input array");
    if (n < 1) return set_err(nullptr, PTYGER_E_DATA, "init: need at least one scan position");
    std::vector<int32_t> base;
    std::vector<float> frac;
    const ptyger_status s = split_positions(scan, n, base, frac);
    if (s != PTYGER_OK) return s;
    return create_ctx(out, cfg, object, H, W, probe, N, base.data(), n, intensities, frac.data());
}

ptyger_status ptyger_partition_subpixel(const float* scan, int64_t n, int64_t H, int32_t N, int32_t P,
                                        int32_t* frame_rank, int64_t* rows) {
    if (!scan || !frame_rank || !rows) return set_err(nullptr, PTYGER_E_ARG, "partition: null pointer");
    std::vector<int32_t> base;
    std::vector<float> frac;
    ptyger_status s = split_positions(scan, n, base, frac);
    if (s != PTYGER_OK) return s;
    bool sub = false;
    for (float f : frac) sub |= f != 0.0f;
    std::vector<int32_t> rk;
    std::vector<int64_t> rw;
    std::string err;
    const int rc = partition(base.data(), n, H, N, P, rk, rw, err, N + (sub ? 1 : 0));
    if (rc) return set_err(nullptr, (ptyger_status)rc, err);
    std::memcpy(frame_rank, rk.data(), sizeof(int32_t) * n);
    std::memcpy(rows, rw.data(), sizeof(int64_t) * rw.size());
    return PTYGER_OK;
}

static ptyger_status check_numeric(ptyger_ctx* c) {
    DevState hs;
    std::string& err = c->err;
    CK(cudaMemcpy(&hs, c->st, sizeof(hs), cudaMemcpyDeviceToHost));
    if (hs.numeric_error) {
        const char* stage = hs.numeric_error == 1 ? "DIR (non-finite ||grad||^2)"
                            : hs.numeric_error == 2 ? "LS (non-finite DeltaF)"
                                                    : "LS (non-finite F)";
        c->failed_numeric = true;
        return set_err(c, PTYGER_E_NUMERIC,
                       "numeric failure at iteration " + std::to_string(hs.err_iter) + " in stage " + stage +
                           "; psi holds the last good iterate");
    }
    return PTYGER_OK;
}

ptyger_status ptyger_cg_launch(ptyger_ctx* c, int32_t n_iter) {
    if (!c) return set_err(nullptr, PTYGER_E_ARG, "cg_launch: ctx is NULL");
    std::string& err = c->err;
    if (n_iter < 0) return set_err(c, PTYGER_E_ARG, "cg_launch: n_iter < 0");
    if (c->failed_numeric) return set_err(c, PTYGER_E_NUMERIC, "context is in a numeric-failure state; call set_state");
    if (!c->connected) return set_err(c, PTYGER_E_STATE, "P2P context not connected (ptyger_ipc_connect)");
    if (c->pending_iters) return set_err(c, PTYGER_E_STATE, "cg_launch: previous launch not waited for");
    if (n_iter == 0) return PTYGER_OK;
    CK(cudaSetDevice(c->cfg.device));
    if (c->tr_cap < n_iter) {
        CK(cudaStreamSynchronize(c->stream));
        if (c->d_tr) cudaFreeAsync(c->d_tr, 0);
        c->d_tr = dalloc<ptyger_trace>((size_t)n_iter, err);
        if (!c->d_tr) return PTYGER_E_OOM;
        CK(cudaStreamSynchronize(0));
        c->tr_cap = n_iter;
    }
    struct { int idx, cap; ptyger_trace* p; } hdr = {0, c->tr_cap, c->d_tr};
    CK(cudaMemcpyAsync(&c->st->trace_idx, &hdr, sizeof(int) * 2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(&c->st->trace_ptr, &hdr.p, sizeof(hdr.p), cudaMemcpyHostToDevice, c->stream));
    if (!c->ev_it[0]) {
        CK(cudaEventCreate(&c->ev_it[0]));
        CK(cudaEventCreate(&c->ev_it[1]));
    }
    CK(cudaEventRecord(c->ev_it[0], c->stream));
    for (int i = 0; i < n_iter; ++i) {
        CK(cudaGraphLaunch(c->graph[c->m_host & 1], c->stream));
        c->m_host += 1;
    }
    CK(cudaEventRecord(c->ev_it[1], c->stream));
    c->last_launches = c->launches_per_iter * n_iter;
    c->pending_iters = n_iter;
    return PTYGER_OK;
}

ptyger_status ptyger_cg_wait(ptyger_ctx* c, ptyger_trace* traces) {
    if (!c) return set_err(nullptr, PTYGER_E_ARG, "cg_wait: ctx is NULL");
    std::string& err = c->err;
    const int n_iter = c->pending_iters;
    if (n_iter == 0) return PTYGER_OK;
    c->pending_iters = 0;
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaEventElapsedTime(&c->last_ms, c->ev_it[0], c->ev_it[1]));
    if (traces) CK(cudaMemcpy(traces, c->d_tr, sizeof(ptyger_trace) * n_iter, cudaMemcpyDeviceToHost));
    return check_numeric(c);
}

ptyger_status ptyger_cg_iterate(ptyger_ctx* c, int32_t n_iter, ptyger_trace* traces) {
    const ptyger_status s = ptyger_cg_launch(c, n_iter);
    if (s != PTYGER_OK) return s;
    return ptyger_cg_wait(c, traces);
}

void* ptyger_stream(const ptyger_ctx* c) { return c ? (void*)c->stream : nullptr; }

// full H*W array of a per-rank storage buffer (collective when world > 1)
static ptyger_status gather_rows(ptyger_ctx* c, const float2* src, float* out) {
    std::string& err = c->err;
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaStreamSynchronize(c->stream));
    if (c->cfg.world == 1) {
        CK(cudaMemcpy(out, src, sizeof(float2) * c->H * c->W, cudaMemcpyDeviceToHost));
        return PTYGER_OK;
    }
    const int64_t* R = &c->rows[6 * c->cfg.rank];
    if (c->p2p) {
        if (!c->connected) return set_err(c, PTYGER_E_STATE, "P2P context not connected (ptyger_ipc_connect)");
        const int64_t par = (int64_t)(c->gather_epoch & 1);
        LK(launch_p2p_gather(src, c->st_lo, R[0], R[1], c->W, c->pv, c->st, c->band_grid, c->stream));
        c->gather_epoch += 1;
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaMemcpy(out, c->full + par * c->H * c->W, sizeof(float2) * c->H * c->W, cudaMemcpyDeviceToHost));
        return PTYGER_OK;
    }
    CK(cudaMemcpyAsync(c->full + R[0] * c->W, src + (R[0] - c->st_lo) * c->W, sizeof(float2) * (R[1] - R[0]) * c->W,
                       cudaMemcpyDeviceToDevice, c->stream));
    NK(c->nc->GroupStart());
    for (int r = 0; r < c->cfg.world; ++r) {
        const int64_t lo = c->rows[6 * r], hi = c->rows[6 * r + 1];
        if (hi <= lo) continue;
        NK(c->nc->Broadcast(c->full + lo * c->W, c->full + lo * c->W, (size_t)((hi - lo) * c->W * 2), ncclFloat32, r,
                            c->comm, c->stream));
    }
    NK(c->nc->GroupEnd());
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(out, c->full, sizeof(float2) * c->H * c->W, cudaMemcpyDeviceToHost));
    return PTYGER_OK;
}

ptyger_status ptyger_get_object(ptyger_ctx* c, float* out) {
    if (!c || !out) return set_err(c, PTYGER_E_ARG, "get_object: null pointer");
    return gather_rows(c, c->psi, out);
}

ptyger_status ptyger_get_gradient(ptyger_ctx* c, float* out) {
    if (!c || !out) return set_err(c, PTYGER_E_ARG, "get_gradient: null pointer");
    if (c->m_host == 0) {
        std::memset(out, 0, sizeof(float2) * c->H * c->W);
        return PTYGER_OK;
    }
    return gather_rows(c, c->g[(c->m_host - 1) & 1], out);
}

ptyger_status ptyger_get_farfield(ptyger_ctx* c, float* out) {
    if (!c || !out) return set_err(c, PTYGER_E_ARG, "get_farfield: null pointer");
    std::string& err = c->err;
    CK(cudaSetDevice(c->cfg.device));
    // u lags psi by the last accepted gamma v (R#11): fold it in first (bit-identical to k_grad's fold)
    LK(launch_fold(c->geo, c->u, c->v, c->st, c->grid_el, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(out, c->u, sizeof(float2) * c->geo.n_local * c->N * c->N, cudaMemcpyDeviceToHost));
    return PTYGER_OK;
}

ptyger_status ptyger_get_state(ptyger_ctx* c, float* psi, float* g_prev, float* eta_prev, double* F, int32_t* m) {
    if (!c) return set_err(nullptr, PTYGER_E_ARG, "get_state: ctx is NULL");
    std::string& err = c->err;
    ptyger_status s;
    if (psi && (s = ptyger_get_object(c, psi)) != PTYGER_OK) return s;
    if (g_prev && (s = ptyger_get_gradient(c, g_prev)) != PTYGER_OK) return s;
    if (eta_prev && (s = gather_rows(c, c->eta, eta_prev)) != PTYGER_OK) return s;
    DevState hs;
    CK(cudaMemcpy(&hs, c->st, sizeof(hs), cudaMemcpyDeviceToHost));
    if (F) *F = hs.F;
    if (m) *m = c->m_host;
    return PTYGER_OK;
}

ptyger_status ptyger_set_state(ptyger_ctx* c, const float* psi, const float* g_prev, const float* eta_prev,
                               int32_t m) {
    if (!c || !psi || m < 0) return set_err(c, PTYGER_E_ARG, "set_state: null ctx/psi or m < 0");
    if (c->cfg.world != 1) return set_err(c, PTYGER_E_STATE, "set_state: only for world == 1");
    if (m > 0 && (!g_prev || !eta_prev)) return set_err(c, PTYGER_E_ARG, "set_state: m > 0 needs g_prev and eta_prev");
    std::string& err = c->err;
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaStreamSynchronize(c->stream));
    const size_t bytes = sizeof(float2) * c->H * c->W;
    CK(cudaMemcpy(c->psi, psi, bytes, cudaMemcpyDefault));
    if (m > 0) {
        CK(cudaMemcpy(c->g[(m - 1) & 1], g_prev, bytes, cudaMemcpyDefault));
        CK(cudaMemcpy(c->eta, eta_prev, bytes, cudaMemcpyDefault));
    } else {
        CK(cudaMemset(c->g[0], 0, bytes));
        CK(cudaMemset(c->g[1], 0, bytes));
        CK(cudaMemset(c->eta, 0, bytes));
    }
    DevState hs;
    std::memset(&hs, 0, sizeof(hs));
    hs.m = m;
    hs.tk_start[0] = hs.tk_start[1] = ~0ull;
    for (int ch = 0; ch < 4; ++ch) hs.p2p_epoch[ch] = 1;
    CK(cudaMemcpy(c->st, &hs, sizeof(hs), cudaMemcpyHostToDevice));
    c->m_host = m;
    c->failed_numeric = false;
    const int rc = run_forward(c, err);
    return (ptyger_status)rc;
}

ptyger_status ptyger_get_ls_partials(ptyger_ctx* c, double* dF, double* bound, int32_t K, int32_t* n_eval) {
    if (!c || !dF || K < 0) return set_err(c, PTYGER_E_ARG, "get_ls_partials: bad arguments");
    std::string& err = c->err;
    CK(cudaStreamSynchronize(c->stream));
    DevState hs;
    CK(cudaMemcpy(&hs, c->st, sizeof(hs), cudaMemcpyDeviceToHost));
    for (int k = 0; k < K; ++k) {
        dF[k] = k < SMAX ? hs.ls_hist[k] : NAN;
        if (bound) bound[k] = k < SMAX ? hs.ls_bnd[k] : NAN;
    }
    if (n_eval) *n_eval = hs.n_eval;
    return PTYGER_OK;
}

float ptyger_last_iterate_ms(const ptyger_ctx* c) { return c ? c->last_ms : 0.f; }

ptyger_status ptyger_fp32_peak(int32_t device, int32_t paired, double* tflops) {
    if (!tflops) return set_err(nullptr, PTYGER_E_ARG, "fp32_peak: null pointer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || device < 0 || device >= ndev) {
        cudaGetLastError();
        return set_err(nullptr, PTYGER_E_CUDA, "fp32_peak: no such CUDA device");
    }
    const double t = measure_fp32_peak(device, paired != 0);
    if (t <= 0) return set_err(nullptr, PTYGER_E_CUDA, "fp32_peak: microbenchmark launch failed");
    *tflops = t;
    return PTYGER_OK;
}

ptyger_status ptyger_kernel_times(ptyger_ctx* c, double* ms, int32_t* count, int32_t reset) {
    if (!c || !ms || !count) return set_err(c, PTYGER_E_ARG, "kernel_times: null pointer");
    std::string& err = c->err;
    CK(cudaSetDevice(c->cfg.device));
    LK(launch_timers(c->st, c->scratch, reset != 0, c->stream));
    double h[4];
    CK(cudaMemcpyAsync(h, c->scratch, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    ms[0] = h[0];
    ms[1] = h[1];
    count[0] = (int32_t)h[2];
    count[1] = (int32_t)h[3];
    return PTYGER_OK;
}

ptyger_status ptyger_ipc_handle(ptyger_ctx* c, void* out64) {
    if (!c || !out64) return set_err(c, PTYGER_E_ARG, "ipc_handle: null pointer");
    if (!c->p2p) return set_err(c, PTYGER_E_STATE, "ipc_handle: not a P2P-transport context");
    std::string& err = c->err;
    CK(cudaSetDevice(c->cfg.device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->win));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(out64, &h, sizeof(h));
    return PTYGER_OK;
}

ptyger_status ptyger_ipc_connect(ptyger_ctx* c, const void* handles) {
    if (!c || !handles) return set_err(c, PTYGER_E_ARG, "ipc_connect: null pointer");
    if (!c->p2p || c->connected) return set_err(c, PTYGER_E_STATE, "ipc_connect: not a pending P2P context");
    std::string& err = c->err;
    CK(cudaSetDevice(c->cfg.device));
    for (int r = 0; r < c->cfg.world; ++r) {
        if (r == c->cfg.rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const unsigned char*>(handles) + 64 * r, 64);
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            err = "cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " + cudaGetErrorString(e);
            return PTYGER_E_CUDA;
        }
        c->pv.win[r] = static_cast<unsigned char*>(p);
    }
    c->connected = true;
    int rc = run_forward(c, err);
    if (rc) return (ptyger_status)rc;
    rc = build_graphs(c, err);
    if (rc) return (ptyger_status)rc;
    return PTYGER_OK;
}

void ptyger_destroy(ptyger_ctx* c) { free_ctx(c); }

}  // extern "C"
