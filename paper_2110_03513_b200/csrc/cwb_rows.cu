// cwb_rows.cu -- row sharding (include/cwb.h "row sharding"):
// the communicator of a context and the restriction of its index vectors to the
// rank's row block.  The per-iteration kernels and the all-reduce points are in
// cwb_iter.cu (cwb_train_rows / cwb_find_best_rows).
//
// NCCL is loaded with dlopen("libnccl.so.2") on first use: in a process that has
// already imported torch this returns torch's NCCL (same soname), otherwise the
// system one; the library itself has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <string>

#include "cwb_internal.cuh"

struct cwb_comm {
    int32_t rank, world;
    void* nccl;  // ncclComm_t, or NULL for a caller's collective
    cwb_allreduce_fn fn;
    void* user;
};

namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy && api.error_string;
        if (!api.ok) api.err = "libnccl.so.2 lacks an expected symbol";
    });
    return api;
}

std::string nccl_msg(const NcclApi& a, ncclResult_t r) {
    return a.error_string ? a.error_string(r) : "NCCL error";
}

// Keep rows [r0, r0 + nl) of the index vectors and rebuild the bin inversion (row
// ids local) for them; the pool (z, bnd, Zb, G, A^-1, lambda, global counts) stays.
int restrict_rows(cwb_ctx* c, int32_t rank, int32_t world) {
    cudaStream_t s = c->stream;
    const int64_t n = c->n, r0 = n * rank / world, r1 = n * (rank + 1) / world, nl = r1 - r0;
    if (nl < 1) return cwb_set_error(c, CWB_EINVAL, "attach: empty row block (world > n)");
    if (c->ev_plan) CWB_CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_plan, 0));  // a pre-built plan may be building
    cwb_release(c->plan, s);
    cwb_release(c->permt, s);
    c->plan = nullptr;
    c->permt = nullptr;
    c->fused_T = 0;
    c->plan_pending = false;
    const size_t K = c->K, ns = c->n_star, ib = c->idx_bytes;
    const int32_t pb = nl <= 65536 ? 2 : 4;
    void *idx = nullptr, *perm = nullptr;
    int32_t* off = nullptr;
    uint32_t* cnt = nullptr;
    bool ok = cwb_alloc(&idx, ib * K * nl + 16, s) == cudaSuccess;
    ok &= cwb_alloc(&perm, (size_t)pb * (K * nl + 8), s) == cudaSuccess;
    ok &= cwb_alloc((void**)&off, 4 * K * (ns + 1), s) == cudaSuccess;
    ok &= cwb_alloc((void**)&cnt, 4 * K * ns, s) == cudaSuccess;
    if (!ok) {
        cwb_release(idx, s); cwb_release(perm, s); cwb_release(off, s); cwb_release(cnt, s);
        return cwb_set_error(c, CWB_ENOMEM, "attach: allocation of the local row block failed");
    }
    CWB_CUDA_TRY(c, cudaMemcpy2DAsync(idx, ib * nl, (const char*)c->idx + ib * r0, ib * n, ib * nl, K,
                                      cudaMemcpyDeviceToDevice, s));
    CWB_CUDA_TRY(c, cudaMemsetAsync(perm, 0, (size_t)pb * (K * nl + 8), s));
    const int rc = cwb_launch_csr(c, idx, c->idx_bytes, nl, c->K, c->n_star, cnt, off, perm, pb, s);
    cwb_release(cnt, s);
    if (rc) {
        cwb_release(idx, s); cwb_release(perm, s); cwb_release(off, s);
        return rc;
    }
    cwb_pool_release(c, c->idx, s);
    cwb_pool_release(c, c->perm, s);
    cwb_pool_release(c, c->off, s);
    c->idx = idx;
    c->perm = perm;
    c->off = off;
    c->perm_bytes = pb;
    // the general-path workspace is sized by n: drop it
    cwb_train_ws& w = c->ws;
    void* bufs[] = {w.Rt, w.U, w.theta, w.delta, w.rr, w.zhat, w.kstar, w.part, w.narrow, w.colpart, w.acwb, w.pack,
                    w.bern, w.fold, w.lbuf};
    for (void* p : bufs) cwb_release(p, s);
    w = cwb_train_ws();
    cwb_stream_release(c, s);  // the streaming findBest plan and the chunked-H1 tables index the full rows
    cwb_release(c->h1c, s);
    c->h1c = nullptr;
    c->h1c_nch = 0;
    c->n_glob = n;
    c->row0 = r0;
    c->n = nl;
    c->rank = rank;
    c->world = world;
    c->rows = true;
    c->path = 2;
    return cwb_check_launch(c, "attach: local bin inversion");
}

}  // namespace

int cwb_rows_allreduce(cwb_ctx* c, double* buf, int64_t count, cudaStream_t s) {
    cwb_comm* m = c->comm;
    if (!m) return cwb_set_error(c, CWB_EINVAL, "row-sharded context without a communicator");
    if (m->nccl) {
        const NcclApi& a = nccl_api();
        const ncclResult_t r = a.all_reduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)m->nccl, s);
        if (r != ncclSuccess) return cwb_set_error(c, CWB_ENCCL, "ncclAllReduce: " + nccl_msg(a, r));
        return CWB_OK;
    }
    if (m->fn(buf, count, s, m->user) != 0) return cwb_set_error(c, CWB_ENCCL, "all-reduce callback failed");
    return CWB_OK;
}

extern "C" {

int cwb_comm_unique_id(void* id_out128) {
    if (!id_out128) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_comm_unique_id: NULL output");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    const NcclApi& a = nccl_api();
    if (!a.ok) return cwb_set_error(nullptr, CWB_ENCCL, "cwb_comm_unique_id: " + a.err);
    ncclUniqueId id;
    const ncclResult_t r = a.get_unique_id(&id);
    if (r != ncclSuccess) return cwb_set_error(nullptr, CWB_ENCCL, "ncclGetUniqueId: " + nccl_msg(a, r));
    memcpy(id_out128, &id, sizeof(id));
    return CWB_OK;
}

int cwb_comm_init(cwb_comm** out, const void* id128, int32_t rank, int32_t world) {
    if (!out || !id128 || world < 1 || rank < 0 || rank >= world)
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_comm_init: invalid argument");
    *out = nullptr;
    const NcclApi& a = nccl_api();
    if (!a.ok) return cwb_set_error(nullptr, CWB_ENCCL, "cwb_comm_init: " + a.err);
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = a.comm_init_rank(&comm, world, id, rank);
    if (r != ncclSuccess) return cwb_set_error(nullptr, CWB_ENCCL, "ncclCommInitRank: " + nccl_msg(a, r));
    *out = new cwb_comm{rank, world, comm, nullptr, nullptr};
    return CWB_OK;
}

int cwb_comm_init_fn(cwb_comm** out, cwb_allreduce_fn fn, void* user, int32_t rank, int32_t world) {
    if (!out || !fn || world < 1 || rank < 0 || rank >= world)
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_comm_init_fn: invalid argument");
    *out = new cwb_comm{rank, world, nullptr, fn, user};
    return CWB_OK;
}

void cwb_comm_free(cwb_comm* m) {
    if (!m) return;
    if (m->nccl) {
        const NcclApi& a = nccl_api();
        if (a.ok) a.comm_destroy((ncclComm_t)m->nccl);
    }
    delete m;
}

int cwb_attach_comm_learners(cwb_ctx* c, cwb_comm* m) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_attach_comm_learners: NULL context");
    if (c->status) return c->status;
    if (!m) return cwb_set_error(c, CWB_EINVAL, "cwb_attach_comm_learners: NULL communicator");
    if (c->rows || c->lshard) return cwb_set_error(c, CWB_EINVAL, "cwb_attach_comm_learners: context already attached");
    if (c->nb) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_attach_comm_learners: unbinned pool");
    if (m->world > c->K) return cwb_set_error(c, CWB_EINVAL, "cwb_attach_comm_learners: world > K");
    c->lk0 = (int32_t)((int64_t)c->K * m->rank / m->world);
    c->lk1 = (int32_t)((int64_t)c->K * (m->rank + 1) / m->world);
    c->lshard = true;
    c->rank = m->rank;
    c->world = m->world;
    c->comm = m;
    c->path = 2;  // per-iteration kernels
    return CWB_OK;
}

int cwb_attach_comm(cwb_ctx* c, cwb_comm* m) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_attach_comm: NULL context");
    if (c->status) return c->status;
    if (!m) return cwb_set_error(c, CWB_EINVAL, "cwb_attach_comm: NULL communicator");
    if (c->rows || c->lshard) return cwb_set_error(c, CWB_EINVAL, "cwb_attach_comm: context already attached");
    if (c->nb) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_attach_comm: unbinned pool");
    if (m->world > c->n) return cwb_set_error(c, CWB_EINVAL, "cwb_attach_comm: world > n");
    const int rc = restrict_rows(c, m->rank, m->world);
    if (rc) return rc;
    c->comm = m;
    return CWB_OK;
}

int cwb_get_rows(const cwb_ctx* c, int64_t* row_begin, int64_t* n_rows, int32_t* rank, int32_t* world) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_get_rows: NULL context");
    if (row_begin) *row_begin = c->rows ? c->row0 : 0;
    if (n_rows) *n_rows = c->n;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return CWB_OK;
}

}  // extern "C"
