// km_api.cu — C-ABI runtime for the B200-native MTI k-means hot path (include/kmeans_b200.h).
//
// Host side of one iteration, all on the context stream:
//   [re-bucket rows]           if AUTO and rows reassigned since the last sort > fraction * n
//   k_prep                     S1 geometry/drift
//   k_assign                   S2+S3 fused; iteration 1: dense
//                              pass, re-bucket, reduction pass (S0)
//   ncclAllReduce (world > 1)  one fp64 sum of [sums | counts] + one int64 sum of the counters
//                              ("merge global state")
//   k_update                   S4; then one D2H of the counters and a stream sync for the stop test
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only; the library is loaded with dlopen when world > 1

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/kmeans_b200.h"
#include "km_kernels.cuh"

namespace {

thread_local std::string g_err;
thread_local size_t *g_track = nullptr;   // device bytes of the context being created

km_status fail(km_status s, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define KM_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? KM_ENOMEM : KM_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                 \
    } while (0)

#define KM_TRY(call)                              \
    do {                                          \
        km_status s_ = (call);                    \
        if (s_ != KM_OK) return s_;               \
    } while (0)

// ---- NCCL, loaded on demand ---------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi *nccl()
{
    static NcclApi api;
    static bool tried = false;
    if (tried) return api.ok ? &api : nullptr;
    tried = true;
    const char *env = getenv("KM_NCCL_LIB");
    const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *nm : names)
        if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return nullptr;
#define SYM(f, s) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, s))
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(AllReduce, "ncclAllReduce");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.GroupStart &&
             api.GroupEnd && api.CommDestroy && api.GetErrorString;
    return api.ok ? &api : nullptr;
}

struct HostStat {
    unsigned long long local[8];   // changed, dists, clause1, refined, walk_steps (this rank)
    int empty;                     // follows the counters in device scratch: one copy for both
    int pad;
    unsigned long long global[8];  // after allreduce (world 1: = local)
};

// clause-1 rate above which the walk stages only the rows that fail clause 1 (SKIP1): C5 (0.29 ->
// 0.42), C2 (0.16 -> 0.46) and C1 (0.45) use it, C3 (<= 0.04) and C4 (<= 0.01) do not
constexpr double kSkip1Rate = 0.15;

int pad_dim(int d)
{
    for (int p : {4, 8, 16, 32, 64})
        if (d <= p) return p;
    return -1;
}

int next_pow2(int v)
{
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace

struct km_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int64_t n = 0;
    int d = 0, DP = 0, k = 0, prune = KM_PRUNE_MTI, rank = 0, world = 1, num_sms = 148;
    int64_t n_global = 0;
    bool csmem = false;
    // row data (ping-pong for re-bucketing)
    float *X[2] = {nullptr, nullptr};
    int32_t *a[2] = {nullptr, nullptr};
    float *u[2] = {nullptr, nullptr};
    int32_t *perm[2] = {nullptr, nullptr};
    int cur = 0;
    // sort scratch
    uint32_t *keys = nullptr, *hist = nullptr, *totals = nullptr, *base = nullptr, *lohist = nullptr;
    int32_t *qmap = nullptr;
    int Q = 1, NB = 0, ntiles = 0, tile_rows = 32768;
    int ks = 0;                     // NL row stride
    // centroid state
    double *C = nullptr, *Cprev = nullptr;
    float *Cneg = nullptr, *f = nullptr, *s = nullptr;
    uint64_t *NL = nullptr;
    // tensor-core MTI engine: per-cluster B operand blocks, column metadata, NL ranks
    float *Bop = nullptr;
    float4 *Bmeta = nullptr;
    // walk engine: per-cluster candidate rows and H
    float4 *Wblk = nullptr;
    float *Wcc = nullptr, *WH = nullptr;
    float2 *Wmeta = nullptr;
    bool wh_smem = false;
    int wpad = 0, whs = 0, wbits = 0, walk_grid = 0;
    bool use_walk = false;
    unsigned long long *defer = nullptr;   // deferred distance-count entries (n_alloc)
    int *dcount = nullptr;                 // per 128-row tile
    bool use_tc = false;
    int tc_nmax = 0, tc_cols = 0, tc_grid = 0;
    int64_t n_alloc = 0;            // rows allocated (n rounded up to the 128-row tile)
    // per-iteration scratch (zeroed by one memset): acc | counters | empty, eps_bits, work[2]
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    double *acc = nullptr;          // k x (DP+1) reduced sums | counts (allreduce buffer)
    double *S = nullptr;            // k x (DP+1) running sums | counts (delta passes add to it)
    double *acc_part = nullptr;     // grid x k x (DP+1) per-CTA partials
    int part_grid = 0;
    int nslab = 0;                  // number of partial slabs (= SM count)
    unsigned long long *counters = nullptr, *counters_g = nullptr;
    int *empty = nullptr, *work = nullptr;
    unsigned *eps_bits = nullptr;
    double *sse_buf = nullptr;
    double *exact_P = nullptr;      // exact-order sums: per 64 Ki-row block x cluster partials (B12)
    bool perm_identity = true;      // stored rows still in caller order (no re-bucketing yet)
    HostStat *hstat = nullptr;
    int grid_assign[4] = {0, 0, 0, 0};
    float g_up = 1.f, g_dn = 1.f;
    int t = 0;
    int64_t changed_since_sort = 0;
    int last_sort_t = 0;            // iteration of the last re-bucketing
    bool spherical = false;         // sk-means (rows and centroids on the unit sphere)
    int resort_policy = KM_RESORT_AUTO;
    float resort_fraction = 0.10f;
    // Elkan TI baseline (KM_PRUNE_TI): k x n_alloc lower bounds (centroid-major), H in index order
    bool use_ti = false;
    float *L = nullptr, *Hm = nullptr;
    int ti_grid = 0;
    size_t dev_bytes = 0;           // device memory held by the context
    double resum_moves = 4.0;       // full re-summation once moves since the last one > this * n_global
    int64_t moves_since_full = 0;   // global moves applied as deltas since the last full reduction
    std::vector<km_iter_stats> stats;
    cudaEvent_t ev[7] = {};
    ncclComm_t comm = nullptr;
    bool comm_on = false;           // allreduce runs (world > 1, or force_comm)
    // CUDA graph of one iteration t >= 2 (S1-S4 + allreduce + counter copy), one per row buffer
    bool use_graph = true;
    cudaGraphExec_t gexec[4] = {nullptr, nullptr, nullptr, nullptr};   // [row buffer][skip1]
    int64_t glaunches[4] = {0, 0, 0, 0};   // kernels in each graph
    // NEXT-2: the walk reads only the rows that fail clause 1, chosen when the last pass's
    // clause-1 rate exceeded kSkip1Rate (global counts: the same choice on every rank)
    bool skip1 = false;
    // screen engine (km_screen.cu): k_screen decides the rows that stay, k_resolve the queued rest
    bool use_screen = false;        // CUDA-core screen (k_screen) or, with use_tc, tensor screen
    int *qrow = nullptr, *qcnt = nullptr;   // per 32-row group: queued rows, count
    int16_t *nlrank = nullptr;      // tensor screen: k x k neighbour-list positions
    // column-chunked tensor-core screen (km_tcc.cu)
    bool use_tcc = false;
    float *Bc = nullptr;
    float *Mh = nullptr, *Mx = nullptr;
    int tcc_nch = 0, tcc_nmeta = 0;
    alignas(64) unsigned char tmap[2][128];   // TMA tensor maps of the two row buffers
    int screen_grid = 0, resolve_grid = 0;
    int64_t launches = 0;
};

namespace {

km_status prep(km_ctx *c)
{
    km::PrepParams p;
    p.C = c->C;
    p.Cprev = c->Cprev;
    p.k = c->k;
    p.d = c->d;
    p.DP = c->DP;
    p.sortN = std::max(2, next_pow2(c->k));
    p.ks = c->ks;
    p.Cneg = c->Cneg;
    p.f = c->f;
    p.s = c->s;
    p.NL = c->NL;
    p.eps_bits = c->eps_bits;
    KM_CUDA(km::launch_prep(p, c->st));
    c->launches += 1;
    if (c->use_walk) {
        KM_CUDA(km::launch_prep_walk(c->C, c->NL, c->k, c->d, c->DP, c->ks, c->wpad, c->whs, c->Wblk, c->Wcc, c->Wmeta, c->WH,
                                     c->st));
        c->launches += 1;
    }
    if (c->use_ti) {
        KM_CUDA(km::launch_prep_ti(c->NL, c->k, c->ks, c->Hm, c->st));
        c->launches += 1;
    }
    if (c->use_tcc) {
        KM_CUDA(km::launch_prep_tcc(c->C, c->NL, c->k, c->d, c->DP, c->ks, c->tcc_nch, c->tcc_nmeta, c->Bc, c->Mh,
                                    c->Mx, c->nlrank, c->st));
        c->launches += 1;
    }
    if (c->use_tc) {
        KM_CUDA(km::launch_prep_tc(c->C, c->NL, c->k, c->d, c->DP, c->ks, c->tc_nmax, c->Bop, c->Bmeta,
                                   c->use_screen ? c->nlrank : nullptr, c->st));
        c->launches += 1;
    }
    return KM_OK;
}

km::AssignParams assign_params(km_ctx *c, int work_slot)
{
    km::AssignParams p;
    p.X = c->X[c->cur];
    p.a = c->a[c->cur];
    p.u = c->u[c->cur];
    p.n = c->n;
    p.d = c->d;
    p.k = c->k;
    p.Cneg = c->Cneg;
    p.C64 = c->C;
    p.NL = c->NL;
    p.ks = c->ks;
    p.f = c->f;
    p.s = c->s;
    p.eps = reinterpret_cast<const float *>(c->eps_bits);
    p.g_up = c->g_up;
    p.g_dn = c->g_dn;
    p.count_changed = c->t > 1;
    p.acc = c->acc_part;
    p.nslab = c->nslab;
    p.counters = c->counters;
    p.work = c->work + work_slot;
    p.Bop = c->Bop;
    p.Bmeta = c->Bmeta;
    p.nmax = c->tc_nmax;
    p.tmem_cols = c->tc_cols;
    p.tile_chunk = 16;
    p.defer = c->defer;
    p.dcount = c->dcount;
    p.nmeta = c->use_tc ? km::tc_nmeta_host(c->tc_nmax) : 0;
    p.Wblk = c->Wblk;
    p.WH = c->WH;
    p.Wcc = c->Wcc;
    p.Wmeta = c->Wmeta;
    p.wh_smem = c->wh_smem ? 1 : 0;
    p.whs = c->whs;
    p.wpad = c->wpad;
    p.wbits = c->wbits;
    p.qrow = c->qrow;
    p.qcnt = c->qcnt;
    p.rank = c->nlrank;
    p.Bc = c->Bc;
    p.Mh = c->Mh;
    p.Mx = c->Mx;
    p.tcc_nch = c->tcc_nch;
    return p;
}

km_status launch_assign(km_ctx *c, int mode, int work_slot)
{
    km::AssignParams p = assign_params(c, work_slot);
    if (c->use_ti && (mode == km::MODE_MTI_REDUCE || mode == km::MODE_DENSE)) {
        KM_CUDA(km::launch_ti(c->DP, c->csmem, mode == km::MODE_DENSE, p, c->L, c->Hm, c->ti_grid, c->st));
    } else if (mode == km::MODE_MTI_REDUCE && c->use_tcc) {
        KM_CUDA(km::launch_tcc(c->DP, c->csmem, p, c->num_sms, c->tmap[c->cur], c->st));
        KM_CUDA(km::launch_resolve(c->DP, c->csmem, p, c->resolve_grid, c->st));
        c->launches += 1;
    } else if (mode == km::MODE_MTI_REDUCE && (c->use_tc || c->use_walk)) {
        if (c->use_tc) {
            KM_CUDA(km::launch_mti_tc(c->DP, c->csmem, p, c->tc_grid, c->use_screen, c->st));
            if (c->use_screen) {
                KM_CUDA(km::launch_resolve(c->DP, c->csmem, p, c->resolve_grid, c->st));
                c->launches += 1;
            }
        }
        else if (c->use_screen) {
            KM_CUDA(km::launch_screen(c->DP, c->csmem, p, c->screen_grid, c->resolve_grid, c->skip1, c->qrow, c->qcnt,
                                      c->n_alloc, c->st));
            c->launches += 1;
        } else KM_CUDA(km::launch_walk(c->DP, c->csmem, p, c->walk_grid, c->skip1, c->st));
        if (!c->use_screen && (c->use_tc || !c->wh_smem)) {   // deferred distance counts (misfit rows)
            KM_CUDA(km::launch_mti_count(c->defer, c->dcount, c->n_alloc / 128, c->counters, c->NL, c->ks, c->k,
                                         c->num_sms, c->st));
            c->launches += 1;
        }
    }
    else
        KM_CUDA(km::launch_assign(mode, c->DP, c->csmem, p, c->grid_assign[mode], c->st));
    c->launches += 1;
    if (mode != km::MODE_DENSE) {
        KM_CUDA(km::launch_partials_reduce(c->acc_part, c->nslab,
                                           (int64_t)c->k * (c->DP + 1), c->acc, c->st));
        c->launches += 1;
    }
    return KM_OK;
}

km_status resort(km_ctx *c)
{
    km::SortParams p;
    const int o = c->cur, nw = 1 - c->cur;
    p.X = c->X[o]; p.a = c->a[o]; p.u = c->u[o]; p.perm = c->perm[o];
    p.X2 = c->X[nw]; p.a2 = c->a[nw]; p.u2 = c->u[nw]; p.perm2 = c->perm[nw];
    p.keys = c->keys; p.hist = c->hist; p.totals = c->totals; p.base = c->base;
    p.NL = c->NL; p.s = c->s; p.ks = c->ks;
    p.lohist = c->lohist;
    p.qmap = c->qmap;
    p.n = c->n; p.k = c->k; p.DP = c->DP;
    p.Q = c->prune == KM_PRUNE_MTI ? c->Q : 1;
    p.NB = c->k * p.Q;
    p.ntiles = c->ntiles;
    p.tile_rows = c->tile_rows;
    int l = 0;
    KM_CUDA(km::launch_sort(p, c->st, &l));
    c->launches += l;
    c->cur = nw;
    c->perm_identity = false;
    c->changed_since_sort = 0;
    c->last_sort_t = c->t;
    return KM_OK;
}

// c->acc = this rank's per-cluster sums | counts of the current assignment in the exact order of
// reading B12 (caller row order, 64 Ki-row blocks merged in block order): bit-reproducible.
// Scratch: keys (inverse permutation), the idle row buffer's a (caller-order assignments).
km_status exact_sums(km_ctx *c)
{
    int l = 0;
    KM_CUDA(km::launch_exact_sums(c->X[c->cur], c->a[c->cur], c->perm[c->cur], c->n, c->DP, c->k,
                                  reinterpret_cast<int32_t *>(c->keys), c->a[1 - c->cur], c->exact_P, c->acc,
                                  c->perm_identity, c->st, &l));
    c->launches += l;
    return KM_OK;
}

km_status allreduce(km_ctx *c)
{
    if (!c->comm_on) return KM_OK;   // global counters = local (iterate copies them once)
    NcclApi *N = nccl();
    if (!N) return fail(KM_ENCCL, "libnccl.so.2 not loadable");
    ncclResult_t r;
    N->GroupStart();
    r = N->AllReduce(c->acc, c->acc, (size_t)c->k * (c->DP + 1), ncclFloat64, ncclSum, c->comm, c->st);
    if (r == ncclSuccess)
        r = N->AllReduce(c->counters, c->counters_g, 8, ncclUint64, ncclSum, c->comm, c->st);
    ncclResult_t r2 = N->GroupEnd();
    if (r != ncclSuccess) return fail(KM_ENCCL, "ncclAllReduce: %s", N->GetErrorString(r));
    if (r2 != ncclSuccess) return fail(KM_ENCCL, "ncclGroupEnd: %s", N->GetErrorString(r2));
    return KM_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b)
{
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) ms = 0.f;
    return ms;
}

// event record that becomes an event node when the stream is being captured
cudaError_t rec_event(cudaEvent_t e, cudaStream_t st)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t err = cudaStreamIsCapturing(st, &cs);
    if (err != cudaSuccess) return err;
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                                               : cudaEventRecord(e, st);
}

// Everything of one iteration after any re-bucketing: S1 prep, S2+S3 pass, allreduce, S4 update,
// copy of the counters to pinned host memory.  t >= 2 only.  Graph-capturable.  full: after the
// pass, re-derive the per-cluster sums from every row (instead of adding this pass's moves).
km_status enqueue_body(km_ctx *c, bool full = false)
{
    cudaEvent_t *ev = c->ev;
    KM_CUDA(cudaMemsetAsync(c->scratch, 0, c->scratch_bytes, c->st));
    KM_CUDA(cudaMemsetAsync(c->acc_part, 0, (size_t)c->nslab * c->k * (c->DP + 1) * sizeof(double), c->st));
    KM_TRY(prep(c));
    KM_CUDA(rec_event(ev[2], c->st));
    KM_TRY(launch_assign(c, c->prune != KM_PRUNE_NONE ? km::MODE_MTI_REDUCE : km::MODE_DENSE_REDUCE, 0));
    KM_CUDA(rec_event(ev[3], c->st));
    if (full) KM_TRY(exact_sums(c));   // re-derive the sums from every row (exact order, B12)
    KM_CUDA(rec_event(ev[4], c->st));
    KM_TRY(allreduce(c));
    KM_CUDA(rec_event(ev[5], c->st));
    // the walk, tensor-core and TI passes reduce only the rows that moved (S += acc, reading B5);
    // the knori- and legacy passes reduce every row (S = acc)
    const int delta = (c->use_walk || c->use_tc || c->use_tcc || c->use_ti) && !full ? 1 : 0;
    KM_CUDA(km::launch_update(c->acc, c->S, delta, c->C, c->Cprev, c->k, c->d, c->DP,
                              c->empty, c->spherical ? 1 : 0, c->st));
    c->launches += 1;
    static_assert(offsetof(HostStat, empty) == 8 * sizeof(unsigned long long), "HostStat layout");
    KM_CUDA(cudaMemcpyAsync(c->hstat->local, c->counters, 8 * sizeof(unsigned long long) + 2 * sizeof(int),
                            cudaMemcpyDeviceToHost, c->st));
    if (c->comm_on)
        KM_CUDA(cudaMemcpyAsync(c->hstat->global, c->counters_g, 8 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, c->st));
    KM_CUDA(rec_event(ev[6], c->st));
    return KM_OK;
}

// replay (capturing on first use) the graph of the body for the current row buffer
km_status launch_body_graph(km_ctx *c)
{
    const int g = c->cur * 2 + (c->skip1 ? 1 : 0);
    if (!c->gexec[g]) {
        const int64_t l0 = c->launches;
        KM_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
        km_status s = enqueue_body(c);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(c->st, &graph);
        if (s != KM_OK) { if (graph) cudaGraphDestroy(graph); return s; }
        KM_CUDA(e);
        e = cudaGraphInstantiate(&c->gexec[g], graph, 0);
        cudaGraphDestroy(graph);
        KM_CUDA(e);
        c->glaunches[g] = c->launches - l0;
        c->launches = l0;
    }
    KM_CUDA(cudaGraphLaunch(c->gexec[g], c->st));
    c->launches += c->glaunches[g];
    return KM_OK;
}

km_status iterate(km_ctx *c, int64_t *changed_out, int64_t *dists_out)
{
    KM_CUDA(cudaSetDevice(c->device));
    cudaEvent_t *ev = c->ev;
    const bool first = c->t == 0;
    c->t += 1;
    km_iter_stats rec;
    memset(&rec, 0, sizeof rec);
    KM_CUDA(cudaEventRecord(ev[0], c->st));
    // re-bucket before the pass when the layout has drifted (u and NL of the previous pass)
    bool sorted_now = false;
    if (!first) {
        bool need = false;
        if (c->resort_policy == KM_RESORT_ALWAYS) need = true;
        else if (c->resort_policy == KM_RESORT_AUTO)
            // the bucket keys of iteration 1 come from the Forgy centroids' H; by iteration 3 the
            // centroids have settled, so the first re-bucketing is never later than t = 3
            need = (double)c->changed_since_sort > (double)c->resort_fraction * (double)c->n ||
                   (c->t == 3 && c->last_sort_t == 1);
        if (need) {
            KM_TRY(resort(c));
            sorted_now = true;
        }
    }
    KM_CUDA(cudaEventRecord(ev[1], c->st));
    if (first) {
        // S0: dense pass, re-bucketing, full reduction of the sorted rows, update (S = acc)
        KM_CUDA(cudaMemsetAsync(c->scratch, 0, c->scratch_bytes, c->st));
        KM_CUDA(cudaMemsetAsync(c->acc_part, 0, (size_t)c->nslab * c->k * (c->DP + 1) * sizeof(double), c->st));
        KM_TRY(prep(c));
        KM_CUDA(cudaEventRecord(ev[2], c->st));
        KM_TRY(launch_assign(c, km::MODE_DENSE, 0));
        KM_CUDA(cudaEventRecord(ev[3], c->st));
        // the full reduction first, while the rows are still in caller order (no permutation to
        // invert: reading B12's order is the stored order), then the first re-bucketing
        KM_TRY(exact_sums(c));
        if (c->resort_policy != KM_RESORT_NEVER) {
            KM_TRY(resort(c));
            sorted_now = true;
        }
        KM_CUDA(cudaEventRecord(ev[4], c->st));
        KM_TRY(allreduce(c));
        KM_CUDA(cudaEventRecord(ev[5], c->st));
        KM_CUDA(km::launch_update(c->acc, c->S, 0, c->C, c->Cprev, c->k, c->d, c->DP, c->empty,
                                  c->spherical ? 1 : 0, c->st));
        c->launches += 1;
        KM_CUDA(cudaMemcpyAsync(c->hstat->local, c->counters, 8 * sizeof(unsigned long long) + 2 * sizeof(int),
                                cudaMemcpyDeviceToHost, c->st));
        if (c->comm_on)
            KM_CUDA(cudaMemcpyAsync(c->hstat->global, c->counters_g, 8 * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, c->st));
        KM_CUDA(cudaEventRecord(ev[6], c->st));
    } else {
        // the decision uses global counts only, so every rank takes it in the same iteration
        const bool full = (c->use_walk || c->use_tc || c->use_tcc || c->use_ti) && c->resum_moves >= 0.0 &&
                          (double)c->moves_since_full > c->resum_moves * (double)c->n_global;
        if (full) {
            KM_TRY(enqueue_body(c, true));
            c->moves_since_full = 0;
        } else if (c->use_graph) {
            KM_TRY(launch_body_graph(c));
        } else {
            KM_TRY(enqueue_body(c));
        }
    }
    KM_CUDA(cudaStreamSynchronize(c->st));
    HostStat *h = c->hstat;
    if (!c->comm_on) memcpy(h->global, h->local, sizeof h->global);
    if (first) {
        rec.changed = c->n_global;
        rec.dists = c->n_global * (int64_t)c->k;
        c->changed_since_sort = 0;
    } else {
        rec.changed = (int64_t)h->global[0];
        rec.dists = (int64_t)h->global[1];
        c->changed_since_sort += (int64_t)h->local[0];
        c->moves_since_full += rec.changed;
    }
    rec.clause1 = (int64_t)h->global[2];
    c->skip1 = (double)rec.clause1 > kSkip1Rate * (double)c->n_global;
    rec.refined = (int64_t)h->global[3];
    rec.walk_steps = (int64_t)h->global[4];
    rec.fallbacks = (int64_t)h->global[5];
    rec.empty = h->empty;
    rec.resorted = sorted_now;
    rec.ms_assign = elapsed(ev[2], ev[3]);
    rec.ms_sort = first ? elapsed(ev[3], ev[4]) : elapsed(ev[0], ev[1]);
    rec.ms_comm = c->comm_on ? elapsed(ev[4], ev[5]) : 0.f;
    rec.ms_iter = elapsed(ev[0], ev[6]);
    c->stats.push_back(rec);
    if (changed_out) *changed_out = rec.changed;
    if (dists_out) *dists_out = rec.dists;
    return KM_OK;
}

void free_all(km_ctx *c)
{
    for (int i = 0; i < 2; ++i) {
        cudaFree(c->X[i]); cudaFree(c->a[i]); cudaFree(c->u[i]); cudaFree(c->perm[i]);
    }
    cudaFree(c->keys); cudaFree(c->hist); cudaFree(c->totals); cudaFree(c->base); cudaFree(c->lohist); cudaFree(c->qmap);
    cudaFree(c->C); cudaFree(c->Cprev); cudaFree(c->Cneg); cudaFree(c->f); cudaFree(c->s);
    cudaFree(c->NL); cudaFree(c->Bop); cudaFree(c->Bmeta); cudaFree(c->defer); cudaFree(c->dcount); cudaFree(c->Wblk); cudaFree(c->WH); cudaFree(c->Wcc); cudaFree(c->Wmeta); cudaFree(c->scratch); cudaFree(c->sse_buf); cudaFree(c->exact_P); cudaFree(c->qrow); cudaFree(c->qcnt); cudaFree(c->nlrank); cudaFree(c->Bc); cudaFree(c->Mh); cudaFree(c->Mx);
    cudaFree(c->counters_g); cudaFree(c->S); cudaFree(c->acc_part); cudaFree(c->L); cudaFree(c->Hm);
    if (c->hstat) cudaFreeHost(c->hstat);
    for (auto &e : c->ev) if (e) cudaEventDestroy(e);
    for (auto &g : c->gexec) if (g) cudaGraphExecDestroy(g);
    if (c->comm) { NcclApi *N = nccl(); if (N) N->CommDestroy(c->comm); }
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
}

template <typename T>
km_status dalloc(T **p, size_t count)
{
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();   // not sticky: clear it so later launches do not report it
        return fail(KM_ENOMEM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    }
    if (g_track) *g_track += std::max<size_t>(count, 1) * sizeof(T);
    return KM_OK;
}

km_status create(int64_t n, int32_t d, int32_t k, const float *points, const double *C0,
                 const km_options *o, km_ctx *c)
{
    c->device = o->device;
    KM_CUDA(cudaSetDevice(c->device));
    c->n = n; c->d = d; c->k = k; c->DP = pad_dim(d);
    c->prune = o->prune; c->rank = o->rank; c->world = o->world;
    c->n_global = o->n_global > 0 ? o->n_global : n * (int64_t)o->world;
    c->resort_policy = o->resort_policy;
    c->use_ti = o->prune == KM_PRUNE_TI;
    if (c->use_ti) c->resort_policy = KM_RESORT_NEVER;   // n x k bounds stay with the caller's rows
    c->resort_fraction = o->resort_fraction > 0.f ? o->resort_fraction : 0.10f;
    c->spherical = o->spherical != 0;
    KM_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    if (o->stream) {
        c->st = static_cast<cudaStream_t>(o->stream);
    } else {
        KM_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    for (auto &e : c->ev) KM_CUDA(cudaEventCreate(&e));
    const int DP = c->DP;
    c->csmem = (size_t)k * DP * sizeof(float) <= 48 * 1024;
    // exact-mode gamma = (DP + 3) 2^-24 on the distance scale
    const double gamma = (DP + 3) * std::ldexp(1.0, -24);
    c->g_up = std::nextafter((float)(1.0 + gamma), 2.0f);
    c->g_dn = std::nextafter((float)(1.0 - gamma), 0.0f);
    // buffers
    // rows padded to whole 128-row tiles (the tensor-core kernel bulk-copies whole tiles);
    // padding rows are zero and never valid
    c->n_alloc = (n + 127) / 128 * 128;
    for (int i = 0; i < 2; ++i) {
        KM_TRY(dalloc(&c->X[i], (size_t)c->n_alloc * DP));
        KM_TRY(dalloc(&c->a[i], (size_t)c->n_alloc));
        KM_TRY(dalloc(&c->u[i], (size_t)c->n_alloc));
        KM_TRY(dalloc(&c->perm[i], (size_t)c->n_alloc));
        KM_CUDA(cudaMemsetAsync(c->X[i], 0, (size_t)c->n_alloc * DP * sizeof(float), c->st));
        KM_CUDA(cudaMemsetAsync(c->a[i], 0, (size_t)c->n_alloc * sizeof(int32_t), c->st));
        KM_CUDA(cudaMemsetAsync(c->u[i], 0, (size_t)c->n_alloc * sizeof(float), c->st));
    }
    // prefix classes per cluster: up to 32 while k*Q <= KM_NB_MAX bucket cursors (scatter smem)
    // (k = 100 and k = 1000: 32 classes of equal population)
    c->Q = std::max(1, std::min(32, KM_NB_MAX / k));
    const int NBmax = k * c->Q;
    c->ntiles = (int)((n + c->tile_rows - 1) / c->tile_rows);
    KM_TRY(dalloc(&c->keys, (size_t)n));
    KM_TRY(dalloc(&c->exact_P, (size_t)km::exact_blocks(n) * k * (DP + 1)));
    KM_TRY(dalloc(&c->hist, (size_t)NBmax * c->ntiles));
    KM_TRY(dalloc(&c->totals, (size_t)NBmax));
    KM_TRY(dalloc(&c->lohist, (size_t)k + 1));
    KM_TRY(dalloc(&c->qmap, (size_t)k + 1));
    KM_TRY(dalloc(&c->base, (size_t)NBmax));
    KM_TRY(dalloc(&c->C, (size_t)k * d));
    KM_TRY(dalloc(&c->Cprev, (size_t)k * d));
    KM_TRY(dalloc(&c->Cneg, (size_t)k * DP));
    KM_TRY(dalloc(&c->f, (size_t)k));
    KM_TRY(dalloc(&c->s, (size_t)k));
    c->ks = (k + 1) & ~1;
    KM_TRY(dalloc(&c->NL, (size_t)(k + 1) * c->ks));   // + one spare row (prefetch slack)
    KM_CUDA(cudaMemset(c->NL, 0, (size_t)(k + 1) * c->ks * sizeof(uint64_t)));
    const size_t acc_bytes = (size_t)k * (DP + 1) * sizeof(double);
    c->scratch_bytes = acc_bytes + 8 * sizeof(unsigned long long) + 8 * sizeof(int);
    KM_TRY(dalloc(reinterpret_cast<char **>(&c->scratch), c->scratch_bytes));
    c->acc = static_cast<double *>(c->scratch);
    c->counters = reinterpret_cast<unsigned long long *>(static_cast<char *>(c->scratch) + acc_bytes);
    int *ints = reinterpret_cast<int *>(c->counters + 8);
    c->empty = ints + 0;
    c->eps_bits = reinterpret_cast<unsigned *>(ints + 1);
    c->work = ints + 2;   // two work counters
    KM_TRY(dalloc(&c->counters_g, 8));
    KM_TRY(dalloc(&c->S, (size_t)k * (DP + 1)));
    KM_TRY(dalloc(&c->sse_buf, 1));
    KM_CUDA(cudaMallocHost(&c->hstat, sizeof(HostStat)));
    // points -> private padded copy
    float *X0 = c->X[0];
    const cudaMemcpyKind kind = o->points_on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    if (DP == d) {
        // one linear copy (a pitched copy of 32-byte rows runs far below the link bandwidth)
        KM_CUDA(cudaMemcpyAsync(X0, points, (size_t)n * d * sizeof(float), kind, c->st));
    } else {
        // linear copy into the second buffer, then pad d -> DP on the device
        KM_CUDA(cudaMemcpyAsync(c->X[1], points, (size_t)n * d * sizeof(float), kind, c->st));
        KM_CUDA(km::launch_pad_rows(c->X[1], X0, n, d, DP, c->st));
        c->launches += 1;
    }
    KM_CUDA(km::launch_iota(c->perm[0], n, c->st));
    c->launches += 1;
    std::vector<double> C0n;
    if (c->spherical) {
        // sk-means: rows onto the unit sphere on the device, initial centroids here (same steps)
        KM_CUDA(cudaMemsetAsync(c->work, 0, sizeof(int), c->st));
        KM_CUDA(km::launch_normalize_rows(X0, n, d, DP, c->work, c->st));
        c->launches += 1;
        int flag = 0;
        KM_CUDA(cudaMemcpyAsync(&flag, c->work, sizeof(int), cudaMemcpyDeviceToHost, c->st));
        KM_CUDA(cudaStreamSynchronize(c->st));
        if (flag) return fail(KM_EARG, "spherical: a point has zero norm");
        C0n.assign(C0, C0 + (size_t)k * d);
        for (int c_ = 0; c_ < k; ++c_) {
            double ss = 0.0;
            for (int j = 0; j < d; ++j) ss += C0n[(size_t)c_ * d + j] * C0n[(size_t)c_ * d + j];
            if (!(ss > 0.0)) return fail(KM_EARG, "spherical: init_centroids row %d has zero norm", c_);
            const double nrm = std::sqrt(ss);
            for (int j = 0; j < d; ++j) C0n[(size_t)c_ * d + j] /= nrm;
        }
        C0 = C0n.data();
    }
    KM_CUDA(cudaMemcpyAsync(c->C, C0, (size_t)k * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    KM_CUDA(cudaMemcpyAsync(c->Cprev, C0, (size_t)k * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    KM_CUDA(cudaStreamSynchronize(c->st));   // C0n is host memory of this scope
    if (o->check_finite) {
        for (int64_t i = 0; i < (int64_t)k * d; ++i)
            if (!std::isfinite(C0[i])) return fail(KM_ENONFINITE, "init_centroids[%lld] is not finite", (long long)i);
        KM_CUDA(cudaMemsetAsync(c->work, 0, sizeof(int), c->st));
        KM_CUDA(km::launch_check_finite(X0, (int64_t)n * DP, c->work, c->st));
        c->launches += 1;
        int flag = 0;
        KM_CUDA(cudaMemcpyAsync(&flag, c->work, sizeof(int), cudaMemcpyDeviceToHost, c->st));
        KM_CUDA(cudaStreamSynchronize(c->st));
        if (flag) return fail(KM_ENONFINITE, "points contain NaN or Inf");
    }
    for (int m = 0; m < 4; ++m) {
        c->grid_assign[m] = km::assign_grid(m, DP, c->csmem, k, c->num_sms);
        c->part_grid = std::max(c->part_grid, c->grid_assign[m]);
    }
    // AUTO (measured on B200 at full size): the column-chunked
    // tensor-core screen k_tcc when d pads to 32 and k >= kAutoTccK (C5, k = 1000: 11.1 vs 24.5 ms
    // per pass: a quarter of its active rows need nearly the whole neighbour list, the dense-
    // survivor regime the tensor cores serve), the CUDA-core walk otherwise (C3 1.56 vs 5.26 ms,
    // C4 6.27 vs 7.76 ms); k = 1 or another prune mode: the default engines, as for the walk
    constexpr int kAutoTccK = 512;
    const bool auto_tcc = o->engine == KM_ENGINE_AUTO && DP == 32 && k >= kAutoTccK &&
                          km::tcc_smem(DP, c->csmem, k) != 0;
    if ((o->engine == KM_ENGINE_TENSOR_CHUNKED || auto_tcc) && c->prune == KM_PRUNE_MTI && !c->use_ti && k >= 2) {
        if (!km::tc_supported(DP))
            return fail(KM_EARG, "tensor_chunked engine needs d padded to 8, 16 or 32 (d=%d)", d);
        if (km::tcc_smem(DP, c->csmem, k) == 0)
            return fail(KM_EARG, "tensor_chunked engine: shared memory for d=%d k=%d exceeds one SM", d, k);
        c->use_tcc = true;
        c->use_screen = true;
        c->tcc_nch = km::tcc_nch_host(k);
        c->tcc_nmeta = km::tcc_nmeta_host(k);
        KM_TRY(dalloc(&c->Bc, (size_t)k * c->tcc_nch * 128 * km::tcc_ka_host(DP)));
        KM_TRY(dalloc(&c->Mh, (size_t)k * km::tcc_hrow_host(k)));
        KM_TRY(dalloc(&c->Mx, (size_t)k * c->tcc_nmeta));
        KM_TRY(dalloc(&c->nlrank, (size_t)k * k));
        KM_TRY(dalloc(&c->qrow, (size_t)c->n_alloc));
        KM_TRY(dalloc(&c->qcnt, (size_t)(c->n_alloc / 32)));
        c->resolve_grid = km::resolve_grid(DP, c->csmem, k, c->num_sms);
        c->part_grid = std::max(c->part_grid, std::max(c->resolve_grid, c->num_sms));
        for (int b = 0; b < 2; ++b) {
            const int r = km::tcc_make_tmap(c->tmap[b], c->X[b], c->n_alloc, DP);
            if (r != 0) return fail(KM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", r);
        }
    }
    const bool want_tc = o->engine == KM_ENGINE_TENSOR || o->engine == KM_ENGINE_TENSOR_SCREEN;
    c->use_tc = km::tc_supported(DP) && c->prune == KM_PRUNE_MTI && k >= 2 && !c->use_ti && want_tc;
    if (want_tc && !km::tc_supported(DP))
        return fail(KM_EARG, "tensor engine needs d padded to 8, 16 or 32 (d=%d)", d);
    // the tensor-core kernel handles rows outside the tile's cluster without extra walks, so
    // re-bucketing only pays when the layout is badly mixed
    if (c->use_tc) {
        c->tc_nmax = std::min(256, std::max(16, (k - 1 + 15) & ~15));   // columns: NL[A] prefix
        if (km::tc_plan(DP, c->csmem, k, c->tc_nmax, c->num_sms, &c->tc_grid, &c->tc_cols) == 0) {
            if (want_tc)
                return fail(KM_EARG, "tensor engine: shared memory for d=%d k=%d exceeds one SM", d, k);
            c->use_tc = false;
        }
    }
    if (c->use_tc) {
        const int KT = km::tc_kt_host(DP);
        KM_TRY(dalloc(&c->Bop, (size_t)k * c->tc_nmax * KT));
        KM_TRY(dalloc(&c->Bmeta, (size_t)k * km::tc_nmeta_host(c->tc_nmax)));
        c->part_grid = std::max(c->part_grid, c->tc_grid);
        if (o->engine == KM_ENGINE_TENSOR_SCREEN) {
            c->use_screen = true;
            c->resolve_grid = km::resolve_grid(DP, c->csmem, k, c->num_sms);
            KM_TRY(dalloc(&c->qrow, (size_t)c->n_alloc));
            KM_TRY(dalloc(&c->qcnt, (size_t)(c->n_alloc / 32)));
            KM_TRY(dalloc(&c->nlrank, (size_t)k * k));
            c->part_grid = std::max(c->part_grid, c->resolve_grid);
        }
    }
    // CUDA-core engine: the centred expansion-form walk (k_walk); KM_ENGINE_CUDA_CORE with a
    // compile-time -DKM_LEGACY_WALK keeps the direct-form lane walk of k_assign (A/B builds only)
    if (c->use_ti) {
        // Elkan's O(nk) lower-bound matrix: fp32, centroid-major
        const size_t lbytes = (size_t)k * c->n_alloc * sizeof(float);
        if (dalloc(&c->L, (size_t)k * c->n_alloc) != KM_OK)
            return fail(KM_ENOMEM, "TI lower-bound matrix: k x n = %d x %lld fp32 = %.1f GB does not fit on the device",
                        k, (long long)c->n_alloc, lbytes / 1e9);
        KM_TRY(dalloc(&c->Hm, (size_t)k * k));
        c->ti_grid = km::ti_grid(DP, c->csmem, k, c->num_sms);
        c->part_grid = std::max(c->part_grid, c->ti_grid);
    }
#ifdef KM_LEGACY_WALK
    c->use_walk = false;
#else
    c->use_walk = !c->use_tc && !c->use_tcc && !c->use_ti && c->prune == KM_PRUNE_MTI && k >= 2 && km::walk_supported(DP);
#endif
    if (c->use_walk) {
        c->wpad = (k + 1) & ~1;                    // k-1 neighbours + >= 1 dummy row, even
        c->wbits = 1;
        while ((1 << c->wbits) < c->wpad) ++c->wbits;
        c->whs = 16;
        while (c->whs < c->wpad) c->whs <<= 1;
        c->wh_smem = c->whs <= 256 && (size_t)k * c->whs * sizeof(float) <= 56 * 1024;
        if (!c->wh_smem && c->whs < 256) c->whs = 256;
        KM_TRY(dalloc(&c->Wblk, (size_t)k * (c->wpad / 2) * (DP / 2)));
        KM_TRY(dalloc(&c->Wcc, (size_t)k * c->wpad));
        KM_TRY(dalloc(&c->Wmeta, (size_t)k * c->wpad));
        KM_TRY(dalloc(&c->WH, (size_t)k * c->whs));
        c->walk_grid = km::walk_grid(DP, c->csmem, k, c->whs, c->wh_smem, c->num_sms);
        c->part_grid = std::max(c->part_grid, c->walk_grid);
        c->use_screen = o->engine == KM_ENGINE_SCREEN;
        if (c->use_screen) {
            km::screen_grids(DP, c->csmem, k, c->whs, c->wh_smem, c->num_sms, &c->screen_grid, &c->resolve_grid);
            KM_TRY(dalloc(&c->qrow, (size_t)c->n_alloc));
            KM_TRY(dalloc(&c->qcnt, (size_t)(c->n_alloc / 32)));
            c->part_grid = std::max(c->part_grid, std::max(c->screen_grid, c->resolve_grid));
        }
    }
    if (c->use_tc || c->use_walk) {
        KM_TRY(dalloc(&c->defer, (size_t)c->n_alloc));
        KM_TRY(dalloc(&c->dcount, (size_t)(c->n_alloc / 32)));
        KM_CUDA(cudaMemsetAsync(c->dcount, 0, (size_t)(c->n_alloc / 32) * sizeof(int), c->st));
    }
    // engines that handle rows outside the warp's / tile's cluster by the triangle bound only
    // re-bucket when the layout is badly mixed
    if ((c->use_tc || c->use_tcc || c->use_walk) && !(o->resort_fraction > 0.f)) c->resort_fraction = 0.25f;
    c->nslab = std::min(c->part_grid, c->num_sms);
    KM_TRY(dalloc(&c->acc_part, (size_t)c->nslab * k * (DP + 1)));
    c->use_graph = o->no_graph == 0;
    c->resum_moves = o->resum_moves == 0.f ? 4.0 : (double)o->resum_moves;
    c->comm_on = c->world > 1 || o->force_comm != 0;
    if (c->comm_on) {
        NcclApi *N = nccl();
        if (!N) return fail(KM_ENCCL, "libnccl.so.2 not loadable (world=%d)", c->world);
        ncclUniqueId id;
        memcpy(id.internal, o->nccl_unique_id, sizeof(id.internal));
        ncclResult_t r = N->CommInitRank(&c->comm, c->world, id, c->rank);
        if (r != ncclSuccess) return fail(KM_ENCCL, "ncclCommInitRank: %s", N->GetErrorString(r));
    }
    KM_CUDA(cudaStreamSynchronize(c->st));
    return KM_OK;
}

}  // namespace

extern "C" {

void kmeans_default_options(km_options *o)
{
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->prune = KM_PRUNE_MTI;
    o->world = 1;
    o->resort_policy = KM_RESORT_AUTO;
    o->resort_fraction = 0.f;      // auto
}

km_status kmeans_nccl_unique_id(uint8_t out[128])
{
    if (!out) return fail(KM_EARG, "out is NULL");
    NcclApi *N = nccl();
    if (!N) return fail(KM_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    ncclResult_t r = N->GetUniqueId(&id);
    if (r != ncclSuccess) return fail(KM_ENCCL, "ncclGetUniqueId: %s", N->GetErrorString(r));
    memcpy(out, id.internal, 128);
    return KM_OK;
}

km_status kmeans_create(int64_t n_local, int32_t d, int32_t k, const float *points,
                        const double *init_centroids, const km_options *opt, km_ctx **out)
{
    g_err.clear();
    if (!out) return fail(KM_EARG, "out is NULL");
    *out = nullptr;
    km_options o;
    if (opt) o = *opt; else kmeans_default_options(&o);
    if (o.world < 1) o.world = 1;
    const int64_t ng = o.n_global > 0 ? o.n_global : n_local * (int64_t)o.world;
    if (n_local < 1 || n_local > 0x7fffffffLL) return fail(KM_EARG, "n_local=%lld out of range", (long long)n_local);
    if (d < 1 || d > 64) return fail(KM_EARG, "d=%d out of range [1, 64]", d);
    if (k < 1 || k > 4096 || k > ng) return fail(KM_EARG, "k=%d out of range [1, min(4096, n_global=%lld)]", k, (long long)ng);
    if (!points || !init_centroids) return fail(KM_EARG, "points/init_centroids is NULL");
    if (reinterpret_cast<uintptr_t>(points) % 4) return fail(KM_EARG, "points not 4-byte aligned");
    if (o.rank < 0 || o.rank >= o.world) return fail(KM_EARG, "rank=%d world=%d", o.rank, o.world);
    if (o.prune != KM_PRUNE_MTI && o.prune != KM_PRUNE_NONE && o.prune != KM_PRUNE_TI) return fail(KM_EARG, "prune=%d", o.prune);
    if (o.resort_policy < 0 || o.resort_policy > 2) return fail(KM_EARG, "resort_policy=%d", o.resort_policy);
    o.n_global = ng;
    km_ctx *c = new km_ctx();
    g_track = &c->dev_bytes;
    km_status s = create(n_local, d, k, points, init_centroids, &o, c);
    g_track = nullptr;
    if (s != KM_OK) {
        std::string keep = g_err;
        free_all(c);
        delete c;
        g_err = keep;
        return s;
    }
    *out = c;
    return KM_OK;
}

km_status kmeans_iterate(km_ctx *c, int64_t *changed, int64_t *dists)
{
    g_err.clear();
    if (!c) return fail(KM_EARG, "ctx is NULL");
    return iterate(c, changed, dists);
}

// C_T re-derived from exact-order sums of a_T (reading B12); C_prev (the centroids of the last
// pass) is kept, so iterating further stays sound.  No-op before the first iteration.
km_status finalize(km_ctx *c)
{
    KM_CUDA(cudaSetDevice(c->device));
    if (c->t == 0) return KM_OK;
    KM_CUDA(cudaMemsetAsync(c->scratch, 0, c->scratch_bytes, c->st));
    KM_TRY(exact_sums(c));
    KM_TRY(allreduce(c));
    KM_CUDA(km::launch_update(c->acc, c->S, 2, c->C, c->Cprev, c->k, c->d, c->DP, c->empty,
                              c->spherical ? 1 : 0, c->st));
    c->launches += 1;
    KM_CUDA(cudaStreamSynchronize(c->st));
    c->moves_since_full = 0;
    return KM_OK;
}

km_status kmeans_finalize(km_ctx *c)
{
    g_err.clear();
    if (!c) return fail(KM_EARG, "ctx is NULL");
    return finalize(c);
}

km_status kmeans_run(km_ctx *c, int32_t max_iters, int64_t tol, int32_t *iterations, int64_t *dists_total)
{
    g_err.clear();
    if (!c) return fail(KM_EARG, "ctx is NULL");
    if (max_iters < 0) return fail(KM_EARG, "max_iters=%d", max_iters);
    int it = 0;
    int64_t tot = 0;
    for (; it < max_iters;) {
        int64_t ch = 0, ds = 0;
        km_status s = iterate(c, &ch, &ds);
        if (s != KM_OK) return s;
        ++it;
        tot += ds;
        if (ch <= tol) break;
    }
    if (it > 0) KM_TRY(finalize(c));
    if (iterations) *iterations = it;
    if (dists_total) *dists_total = tot;
    return KM_OK;
}

km_status kmeans_get_assignments(km_ctx *c, int32_t *out, int32_t out_is_device)
{
    g_err.clear();
    if (!c || !out) return fail(KM_EARG, "NULL argument");
    if (c->t == 0) return fail(KM_ESTATE, "no assignment pass has run yet");
    KM_CUDA(cudaSetDevice(c->device));
    // scratch: the idle row buffer's a (dead until the next re-bucketing overwrites it whole); no
    // allocation on the read-back path (a lazy cudaMalloc here cost 5-30 ms of the e2e run)
    int32_t *tmp = c->a[1 - c->cur];
    KM_CUDA(km::launch_unpermute(c->a[c->cur], c->perm[c->cur], c->n, tmp, c->st));
    c->launches += 1;
    KM_CUDA(cudaMemcpyAsync(out, tmp, (size_t)c->n * sizeof(int32_t),
                            out_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
    KM_CUDA(cudaStreamSynchronize(c->st));
    return KM_OK;
}

km_status kmeans_get_bounds(km_ctx *c, float *out, int32_t out_is_device)
{
    g_err.clear();
    if (!c || !out) return fail(KM_EARG, "NULL argument");
    if (c->t == 0) return fail(KM_ESTATE, "no assignment pass has run yet");
    if (c->prune == KM_PRUNE_NONE) return fail(KM_ESTATE, "no bounds are kept with KM_PRUNE_NONE");
    KM_CUDA(cudaSetDevice(c->device));
    // u is 4-byte data in the context's row order: the int32 unpermute moves its bits
    int32_t *tmp = c->a[1 - c->cur];
    KM_CUDA(km::launch_unpermute(reinterpret_cast<const int32_t *>(c->u[c->cur]), c->perm[c->cur], c->n, tmp,
                                 c->st));
    c->launches += 1;
    KM_CUDA(cudaMemcpyAsync(out, tmp, (size_t)c->n * sizeof(float),
                            out_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
    KM_CUDA(cudaStreamSynchronize(c->st));
    return KM_OK;
}

km_status kmeans_get_centroids(km_ctx *c, double *out)
{
    g_err.clear();
    if (!c || !out) return fail(KM_EARG, "NULL argument");
    KM_CUDA(cudaSetDevice(c->device));
    KM_CUDA(cudaMemcpyAsync(out, c->C, (size_t)c->k * c->d * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    KM_CUDA(cudaStreamSynchronize(c->st));
    return KM_OK;
}

km_status kmeans_set_centroids(km_ctx *c, const double *cent)
{
    g_err.clear();
    if (!c || !cent) return fail(KM_EARG, "NULL argument");
    KM_CUDA(cudaSetDevice(c->device));
    KM_CUDA(cudaMemcpyAsync(c->C, cent, (size_t)c->k * c->d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    if (c->t == 0)   // before iteration 1 there is no previous pass: drift reference = C
        KM_CUDA(cudaMemcpyAsync(c->Cprev, cent, (size_t)c->k * c->d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    KM_CUDA(cudaStreamSynchronize(c->st));
    return KM_OK;
}

km_status kmeans_sse(km_ctx *c, double *out)
{
    g_err.clear();
    if (!c || !out) return fail(KM_EARG, "NULL argument");
    if (c->t == 0) return fail(KM_ESTATE, "no assignment pass has run yet");
    KM_CUDA(cudaSetDevice(c->device));
    KM_CUDA(cudaMemsetAsync(c->sse_buf, 0, sizeof(double), c->st));
    KM_CUDA(km::launch_sse(c->X[c->cur], c->a[c->cur], c->C, c->n, c->d, c->DP, c->sse_buf, c->st));
    c->launches += 1;
    if (c->comm_on) {
        NcclApi *N = nccl();
        if (!N) return fail(KM_ENCCL, "libnccl.so.2 not loadable");
        ncclResult_t r = N->AllReduce(c->sse_buf, c->sse_buf, 1, ncclFloat64, ncclSum, c->comm, c->st);
        if (r != ncclSuccess) return fail(KM_ENCCL, "ncclAllReduce: %s", N->GetErrorString(r));
    }
    KM_CUDA(cudaMemcpyAsync(out, c->sse_buf, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    KM_CUDA(cudaStreamSynchronize(c->st));
    return KM_OK;
}

km_status kmeans_get_stats(km_ctx *c, km_iter_stats *out, int32_t cap, int32_t *count)
{
    g_err.clear();
    if (!c) return fail(KM_EARG, "ctx is NULL");
    const int32_t m = (int32_t)c->stats.size();
    if (count) *count = m;
    if (out && cap > 0) memcpy(out, c->stats.data(), sizeof(km_iter_stats) * (size_t)std::min(cap, m));
    return KM_OK;
}

int64_t kmeans_launch_count(const km_ctx *c) { return c ? c->launches : 0; }

int64_t kmeans_device_bytes(const km_ctx *c) { return c ? (int64_t)c->dev_bytes : 0; }

const char *kmeans_engine(const km_ctx *c)
{
    if (!c) return "";
    if (c->prune == KM_PRUNE_NONE) return "k_assign_dense";
    if (c->use_ti) return "k_ti";
    if (c->use_tcc) return "k_tcc";
    if (c->use_tc && c->use_screen) return "k_mti_tc_screen";
    return c->use_tc ? "k_mti_tc" : (c->use_walk ? (c->use_screen ? "k_screen" : "k_walk") : "k_assign");
}

void kmeans_destroy(km_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->st) cudaStreamSynchronize(c->st);
    free_all(c);
    delete c;
}

const char *kmeans_last_error(void) { return g_err.c_str(); }

const char *kmeans_version(void) { return "kmeans_b200 0.1.0 (sm_100a)"; }

km_status kmeans_seed_plusplus(int64_t n, int32_t d, int32_t k, const float *points, int32_t points_on_host,
                               int64_t first_index, const double *uniforms, int32_t device, void *stream,
                               int64_t *chosen, double *centroids)
{
    g_err.clear();
    if (n < 1 || d < 1 || k < 1 || k > n) return fail(KM_EARG, "n=%lld d=%d k=%d", (long long)n, d, k);
    if (!points || !chosen || !centroids || (k > 1 && !uniforms)) return fail(KM_EARG, "NULL argument");
    if (first_index < 0 || first_index >= n) return fail(KM_EARG, "first_index=%lld", (long long)first_index);
    for (int m = 0; m + 1 < k; ++m)
        if (!(uniforms[m] >= 0.0 && uniforms[m] < 1.0)) return fail(KM_EARG, "uniforms[%d] not in [0,1)", m);
    KM_CUDA(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    float *Xd = nullptr, *crow = nullptr;
    double *D2 = nullptr;
    char *scratch = nullptr;
    int64_t *dsel = nullptr;
    auto cleanup = [&]() {
        if (points_on_host) cudaFree(Xd);
        cudaFree(crow); cudaFree(D2); cudaFree(scratch); cudaFree(dsel);
    };
    km_status s = KM_OK;
    do {
        if (points_on_host) {
            if ((s = dalloc(&Xd, (size_t)n * d)) != KM_OK) break;
            if (cudaMemcpyAsync(Xd, points, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, st) != cudaSuccess) {
                s = fail(KM_ECUDA, "copy of the points"); break;
            }
        } else {
            Xd = const_cast<float *>(points);
        }
        if ((s = dalloc(&crow, (size_t)d)) != KM_OK) break;
        if ((s = dalloc(&D2, (size_t)n)) != KM_OK) break;
        if ((s = dalloc(&scratch, km::seed_scratch_bytes(n))) != KM_OK) break;
        if ((s = dalloc(&dsel, (size_t)1)) != KM_OK) break;
        cudaError_t e = km::seed_plusplus(Xd, n, d, d, k, first_index, uniforms, D2, scratch, crow, dsel, chosen, st);
        if (e == cudaErrorInvalidValue) { s = fail(KM_EARG, "fewer than k distinct rows"); break; }
        if (e == cudaErrorNotSupported) { s = fail(KM_EARG, "a D^2 outside the exact fixed point (non-fp32 data)"); break; }
        if (e != cudaSuccess) { s = fail(KM_ECUDA, "seed_plusplus: %s", cudaGetErrorString(e)); break; }
        std::vector<float> row((size_t)d);
        for (int m = 0; m < k; ++m) {
            if (cudaMemcpy(row.data(), Xd + chosen[m] * d, (size_t)d * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) {
                s = fail(KM_ECUDA, "copy of a chosen row"); break;
            }
            for (int j = 0; j < d; ++j) centroids[(size_t)m * d + j] = (double)row[j];
        }
    } while (false);
    cudaStreamSynchronize(st);
    cleanup();
    return s;
}

}  // extern "C"
