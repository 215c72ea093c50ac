// smpu.cu -- host engine and C ABI of libsmpu.so (see include/smpu.h for the contract).
//
// Layout in HBM (one allocation per array, 16 B per parameter in total):
//   theta fp32[n], m fp32[n], v fp32[n]       fp32 master weights + Adam moments
//   theta_b, m_b, v_b fp32[n]                 second bank of them (fuse_final at W = 1: the speculative update)
//   w16   fp16[n]                             fp16 model weights, re-cast each update
//   acc   fp16[n]                             accumulator; buckets are views of it
//   acc32 fp32[n]                             accum_fp32 only: the sums; acc then gets rn16 of the last one
//   flag int32, stat u32, xs int64[2], DevState, Scalars, loss scale fp32   (device scalars; K0 owns them)
//   result ring: 64 smpu_step_result in mapped pinned host memory (written by K0).
//
// Streams (W > 1): K1 runs on the caller's stream; each bucket's all-reduce (the fused peer-memory kernel of
// lsa_allreduce.cuh, or NCCL) runs on a high-priority comm stream gated by that bucket's ready event (the
// paper's "background thread", becomes a stream: enqueue is already asynchronous); once the last
// micro-batch is accumulated, a decision stream exchanges 16 bytes per rank (N_r and max|A_r|: through peer
// memory in one kernel, or an NCCL all-reduce on a second communicator) and K0 EARLY decides overflow exactly
// in the common case; two K2 streams (pieces alternate) then run Adam on each all-reduce piece as soon as it
// lands, overlapping the remaining all-reduces.  smpu_step enqueues only the (normally empty) fallback.  W = 1:
// K1 -> K0 -> K2 on the caller's streams.  No host synchronisation anywhere on the update path.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "kernels.cuh"
#include "lsa_allreduce.cuh"
#include "smpu.h"

using namespace smpu;

namespace {

thread_local std::string g_err;
constexpr int kRing = 64;
constexpr int64_t kStageElems = int64_t(16) << 20;   // 32 MiB of fp16 per host-staging buffer

smpu_status set_err(smpu_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

enum PtrKind { PTR_DEVICE, PTR_HOST, PTR_FOREIGN };   // FOREIGN: device memory of another GPU

}  // namespace

struct smpu_ctx {
    smpu_config cfg{};
    int world = 1, rank = 0, dev = 0;
    int64_t n = 0;
    std::vector<int64_t> bbegin;   // bucket element offsets, size nb+1
    std::vector<int> tensor_bucket;                 // first bucket of each tensor (plan order)
    std::vector<int> tensor_bucket_last;            // last bucket of each tensor (> first only with split_tensors)
    std::vector<int> bucket_tensors;                // tensors overlapping each bucket
    std::vector<int> bucket_tensors_left;           // of the open micro-batch (smpu_tensor_ready)
    std::vector<char> tensor_seen;                  // of the open micro-batch
    int nb = 0;

    float *theta = nullptr, *m = nullptr, *v = nullptr;
    float *theta_b = nullptr, *m_b = nullptr, *v_b = nullptr;   // second bank (fuse_final, world 1)
    bool fused = false;            // fuse_final in effect: the last micro-batch runs k12_fused
    float* acc32 = nullptr;        // fp32 accumulator (smpu_config.accum_fp32, SURVEY Z1 knob), else null
    bool fused_prepped = false;    // k0_fused_prep enqueued for the open update
    uint16_t *w16 = nullptr, *acc = nullptr;
    int* flag = nullptr;
    uint32_t* stat = nullptr;      // local max fp16 magnitude bits of the last micro-batch's output (W > 1)
    int64_t* xs = nullptr;         // {N_r, M_r} -> all-reduced {N, sum_r M_r} (W > 1)
    DevState* st = nullptr;
    Scalars* sc = nullptr;
    float* scale = nullptr;
    smpu_step_result* ring_host = nullptr;
    smpu_step_result* ring_dev = nullptr;
    cudaEvent_t ring_ev[kRing] = {};
    DevCfg dcfg{};

    ncclComm_t comm = nullptr;     // gradient buckets
    ncclComm_t comm2 = nullptr;    // the 16-byte decision all-reduce, concurrent with the bucket all-reduces
    int ar_impl = 0;               // SMPU_AR_NCCL / SMPU_AR_FUSED (world > 1)
    bool acc_from_nccl = false;    // acc came from ncclMemAlloc (symmetric window)
    ncclWindow_t win = nullptr;
    ncclDevComm devcomm{};
    bool have_devcomm = false;
    int grid_ar = 0;
    bool ar_vec32 = false;                                  // 256-bit peer accesses in the fused all-reduce
    bool ar_mcast = false;                                  // all-gather by NVLS multicast stores
    int ar_unroll = 1, ar_threads = 256;                    // fused all-reduce shape (smpu_config.ar_*)
    // copy-engine all-reduce (smpu_config.ar_copy_engine): staging offset in the window of every piece, every rank's
    // window as a VA of this process (LSA peers; the copies' destinations), W - 1 copy streams and their events
    bool ce = false;
    std::vector<std::vector<size_t>> ce_off;
    char* peer_win[kMaxLsaRanks] = {};
    cudaStream_t ce_stream[kMaxLsaRanks] = {};
    cudaEvent_t ce_fork = nullptr, ce_join[kMaxLsaRanks] = {};
    smpu_group* group = nullptr;                            // virtual rank of a one-GPU group (smpu_group_init)
    bool w16_in_win = false;                                // w16 is a slice of the window allocation
    cudaStream_t step_stream = nullptr;                     // group, sharded: the stream of the deferred tail
    cudaEvent_t tail_ev = nullptr;                          // group: end of this rank's part of the update
    size_t dec_area_off = 0;
    bool sharded = false;                                   // SURVEY f2 variant (smpu_config.sharded)
    size_t w16_off = 0;                                     // w16 inside the symmetric window
    std::vector<std::vector<std::pair<int64_t, int64_t>>> shard;   // per bucket: this rank's element ranges
    cudaStream_t comm_stream = nullptr, copy_stream = nullptr, dec_stream = nullptr, k2_stream = nullptr;
    cudaStream_t k2_stream2 = nullptr;                      // second Adam stream (W > 1 pieces alternate)
    cudaEvent_t k2_join = nullptr;
    std::vector<cudaEvent_t> ready;
    // all-reduce launches of bucket b: pieces[b] = element boundaries (one piece unless smpu_config.ar_pieces
    // pipelines them), ar_done[b][i] = piece i reduced
    std::vector<std::vector<int64_t>> pieces;
    std::vector<std::vector<cudaEvent_t>> ar_done;
    cudaEvent_t comm_done = nullptr, order_ev = nullptr, dec_ev = nullptr, k2_done = nullptr;
    cudaStream_t last_stream = nullptr;
    bool have_order = false;

    uint16_t* stage[2] = {nullptr, nullptr};
    cudaEvent_t stage_free[2] = {}, stage_full[2] = {};
    int64_t stage_count = 0;

    // update-in-progress bookkeeping (host)
    int micro = 0;                 // micro-batches started in this update
    bool bucket_micro = false;     // the open micro-batch is bucket-wise
    std::vector<char> bucket_done;
    int buckets_left = 0;
    int next_issue = 0;
    int64_t local_tokens = 0;
    // CUDA graph of one whole update (smpu_graph_capture / smpu_graph_launch)
    bool capturing = false;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    bool graph_resident = false;
    bool graph_direct = false;
    const uint16_t* k2_src = nullptr;  // captured c = 1, W = 1 graphs: Adam reads the producer's buffer (R = g_1)
    int64_t* tok_dev = nullptr;        // this update's local token count, written before each replay
    int64_t* tok_host = nullptr;       // pinned ring of kRing slots feeding tok_dev
    int64_t attempts = 0;
    int64_t first_attempt = 1;         // smpu_result serves attempts >= this (reset by set_state(SCALARS))
    bool poisoned = false;

    int grid_k1 = 0, grid_k2 = 0, grid_k1s = 0;
    bool k1_oneshot = false, k2_oneshot = false;   // one unit per thread (grid cap "0 CTAs per SM")
    bool pdl = false;                              // programmatic dependent launch of K1 -> K0 -> K2 (world 1)

    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed[SMPU_N_KERNELS];
    struct TraceRec {
        int32_t kind, stream;
        cudaEvent_t b, e;
    };
    std::vector<TraceRec> trace;
    int64_t launches[SMPU_N_KERNELS] = {};
    int64_t graph_launches[SMPU_N_KERNELS] = {};   // kernels per replay of the captured update, by kind
};

// W virtual ranks on one GPU (smpu_group_init): W member ctxs, each with its own state and window, driven by one
// host thread.  The peer kernels of lsa_allreduce.cuh run over LocalPeers; a collective step is issued when the
// last member reaches it (the members' own stream events order it), so the host may interleave the ranks' calls in
// any order that a real W-process job could make.
struct smpu_group {
    int world = 0, dev = 0;
    std::vector<smpu_ctx*> m;
    cudaStream_t comm = nullptr, dec = nullptr;    // bucket all-reduces; decision exchanges
    cudaEvent_t late_ev = nullptr;
    std::vector<int> arrived;                      // per bucket: members whose last-micro-batch bucket is accumulated
    int next_issue = 0;                            // next bucket all-reduce, canonical order
    int dec_arrived = 0;                           // members whose last micro-batch is complete
    std::vector<char> stepped;                     // members that called smpu_step in the open round
    int n_stepped = 0;
    int per_rank = 1;                              // CTAs per virtual rank of the one-launch all-reduce
};

namespace {

smpu_status fail_cuda(smpu_ctx* c, cudaError_t e, const char* what, int line) {
    if (c) c->poisoned = true;
    return set_err(SMPU_ECUDA, "CUDA error %d (%s) in %s at smpu.cu:%d", (int)e, cudaGetErrorString(e), what, line);
}
smpu_status fail_nccl(smpu_ctx* c, ncclResult_t e, const char* what, int line) {
    if (c) c->poisoned = true;
    return set_err(SMPU_ENCCL, "NCCL error %d (%s) in %s at smpu.cu:%d", (int)e, ncclGetErrorString(e), what, line);
}

#define CK(x)                                                        \
    do {                                                             \
        cudaError_t e_ = (x);                                        \
        if (e_ != cudaSuccess) return fail_cuda(ctx, e_, #x, __LINE__); \
    } while (0)
#define CKL(what)                                                              \
    do {                                                                       \
        cudaError_t e_ = cudaGetLastError();                                   \
        if (e_ != cudaSuccess) return fail_cuda(ctx, e_, what, __LINE__);      \
    } while (0)
#define NK(x)                                                        \
    do {                                                             \
        ncclResult_t r_ = (x);                                       \
        if (r_ != ncclSuccess) return fail_nccl(ctx, r_, #x, __LINE__); \
    } while (0)
#define LIVE(ctx)                                                                             \
    do {                                                                                      \
        if (!(ctx)) return set_err(SMPU_EINVAL, "null ctx");                                  \
        if ((ctx)->poisoned) return set_err(SMPU_EPOISONED, "ctx poisoned by an earlier error"); \
    } while (0)

// The peer-memory kernels are templated on the world size W so that their per-rank loops unroll; dispatch a
// launch macro CALL(W) on the runtime world size.
#define SMPU_BY_WORLD(world_, CALL, what)                                 \
    switch (world_) {                                                     \
        case 2: CALL(2); break;                                           \
        case 3: CALL(3); break;                                           \
        case 4: CALL(4); break;                                           \
        case 5: CALL(5); break;                                           \
        case 6: CALL(6); break;                                           \
        case 7: CALL(7); break;                                           \
        case 8: CALL(8); break;                                           \
        default: return set_err(SMPU_EINVAL, what " supports 2..8 ranks"); \
    }

PtrKind classify(const smpu_ctx* c, const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return PTR_HOST;
    }
    if (a.type == cudaMemoryTypeManaged) return PTR_DEVICE;
    if (a.type == cudaMemoryTypeDevice) return a.device == c->dev ? PTR_DEVICE : PTR_FOREIGN;
    return PTR_HOST;
}

cudaEvent_t pool_event(smpu_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

// bracket one launch with events when timing is on
struct Timed {
    smpu_ctx* c;
    int kind;
    cudaStream_t s;
    cudaEvent_t b = nullptr;
    Timed(smpu_ctx* c_, int k, cudaStream_t s_) : c(c_), kind(k), s(s_) {
        c->launches[kind]++;
        if (c->timing && (b = pool_event(c))) cudaEventRecord(b, s);
    }
    ~Timed() {
        if (b) {
            cudaEvent_t e = pool_event(c);
            if (e) {
                cudaEventRecord(e, s);
                c->timed[kind].emplace_back(b, e);
                int sid = s == c->comm_stream ? 1 : s == c->dec_stream ? 2 :
                          (s == c->k2_stream || s == c->k2_stream2) ? 3 : 0;
                c->trace.push_back({kind, sid, b, e});
            }
        }
    }
};

// order this call's launches after the library's previous writes, whatever stream they were on
smpu_status enter_stream(smpu_ctx* ctx, cudaStream_t s) {
    if (ctx->capturing) return SMPU_OK;    // graph launches order themselves (smpu_graph_launch)
    if (ctx->have_order && s != ctx->last_stream) CK(cudaStreamWaitEvent(s, ctx->order_ev, 0));
    return SMPU_OK;
}
smpu_status leave_stream(smpu_ctx* ctx, cudaStream_t s) {
    if (ctx->capturing) return SMPU_OK;
    CK(cudaEventRecord(ctx->order_ev, s));
    ctx->last_stream = s;
    ctx->have_order = true;
    return SMPU_OK;
}

// Grid cap of a streaming kernel: 0 CTAs per SM = one-shot (one unit per thread, no cap; the default for K1
// and K2, see tools/hbm_probe.cu), else SMs x that many CTAs with a grid-stride loop.  The environment
// variable `name` overrides the default.
int grid_cap(const char* name, int sms, int default_cps) {
    const char* v = getenv(name);
    int cps = v ? atoi(v) : default_cps;
    return cps <= 0 ? 0x7fffffff : sms * cps;
}

// Launch with programmatic dependent launch (PDL) when enabled: the kernel may start its CTAs while its
// predecessor in the stream finishes (kernels call pdl_trigger / pdl_wait, kernels.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(const smpu_ctx* ctx, void (*kernel)(KArgs...), int grid, int block, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ctx->pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

int grid_for(int64_t units, int max_grid) {
    int64_t g = (units + 255) / 256;
    if (g > max_grid) g = max_grid;
    if (g < 1) g = 1;
    return (int)g;
}

smpu_status launch_k1(smpu_ctx* ctx, const uint16_t* g, int64_t lo, int64_t hi, bool first, bool detect,
                      cudaStream_t s, bool stats = false) {
    if (hi <= lo) return SMPU_OK;
    int grid = grid_for((hi - lo + 15) / 16, ctx->grid_k1);
    Timed t(ctx, first ? SMPU_K1_FIRST : SMPU_K1_ADD, s);
    if (ctx->k1_oneshot) {
        uint16_t* a = ctx->acc;
        int* f = ctx->flag;
        uint32_t* st = ctx->stat;
        cudaError_t e;
        if (first) {
            if (stats) e = launch_pdl(ctx, k1_accumulate_1<true, false, true>, grid, 256, s, a, g, lo, hi, f, st);
            else if (detect) e = launch_pdl(ctx, k1_accumulate_1<true, true, false>, grid, 256, s, a, g, lo, hi, f, st);
            else e = launch_pdl(ctx, k1_accumulate_1<true, false, false>, grid, 256, s, a, g, lo, hi, f, st);
        } else {
            if (stats) e = launch_pdl(ctx, k1_accumulate_1<false, false, true>, grid, 256, s, a, g, lo, hi, f, st);
            else if (detect) e = launch_pdl(ctx, k1_accumulate_1<false, true, false>, grid, 256, s, a, g, lo, hi, f, st);
            else e = launch_pdl(ctx, k1_accumulate_1<false, false, false>, grid, 256, s, a, g, lo, hi, f, st);
        }
        if (e != cudaSuccess) return fail_cuda(ctx, e, "k1_accumulate_1", __LINE__);
    } else if (stats) {
        if (first) k1_accumulate<true, false, true><<<grid, 256, 0, s>>>(ctx->acc, g, lo, hi, ctx->flag, ctx->stat);
        else k1_accumulate<false, false, true><<<grid, 256, 0, s>>>(ctx->acc, g, lo, hi, ctx->flag, ctx->stat);
    } else if (first) {
        if (detect) k1_accumulate<true, true><<<grid, 256, 0, s>>>(ctx->acc, g, lo, hi, ctx->flag);
        else k1_accumulate<true, false><<<grid, 256, 0, s>>>(ctx->acc, g, lo, hi, ctx->flag);
    } else {
        if (detect) k1_accumulate<false, true><<<grid, 256, 0, s>>>(ctx->acc, g, lo, hi, ctx->flag);
        else k1_accumulate<false, false><<<grid, 256, 0, s>>>(ctx->acc, g, lo, hi, ctx->flag);
    }
    CKL("k1_accumulate");
    return SMPU_OK;
}

LsaPeers lsa_peers(const smpu_ctx* ctx) { return LsaPeers{ctx->devcomm, ctx->win}; }

// rank p's window = member p's window allocation; per_rank > 0: one launch for every rank, else one for `fixed`
LocalPeers local_peers(const smpu_group* g, int per_rank, int fixed) {
    LocalPeers pe{};
    for (int p = 0; p < g->world; ++p) pe.base[p] = (char*)g->m[p]->acc;
    pe.per_rank = per_rank;
    pe.fixed = fixed;
    return pe;
}

// Adam on this rank's shard ranges of bucket b (sharded variant); one-shot grid, or a small persistent grid for
// the (normally empty) late fallback
template <class Peers>
smpu_status launch_k2_shard_with(smpu_ctx* ctx, const Peers& pe, int b, int32_t need, cudaStream_t s) {
    int launched = 0;   // the caller's Timed counts one launch; rank 0 may add its unaligned head / tail
    for (auto& rg : ctx->shard[b]) {
        if (rg.second <= rg.first) continue;
        if (launched++) ctx->launches[SMPU_K2]++;
        int grid = grid_for((rg.second - rg.first + 7) / 8, need == DEC_APPLY_LATE ? ctx->grid_k1s : 0x7fffffff);
#define SMPU_K2S(WW)                                                                                              \
    k2_adam_shard<WW, Peers><<<grid, 256, 0, s>>>(pe, ctx->w16_off, ctx->theta, ctx->m, ctx->v, ctx->acc, rg.first, \
                                                  rg.second, ctx->sc, need)
        SMPU_BY_WORLD(ctx->world, SMPU_K2S, "sharded Adam")
#undef SMPU_K2S
        CKL("k2_adam_shard");
    }
    return SMPU_OK;
}

smpu_status launch_k2_shard(smpu_ctx* ctx, int b, int32_t need, cudaStream_t s) {
    if (ctx->group) return launch_k2_shard_with(ctx, local_peers(ctx->group, 0, ctx->rank), b, need, s);
    return launch_k2_shard_with(ctx, lsa_peers(ctx), b, need, s);
}

smpu_status launch_k2(smpu_ctx* ctx, int64_t lo, int64_t hi, int32_t need, cudaStream_t s) {
    int grid = grid_for((hi - lo + 7) / 8, ctx->grid_k2);
    if (need == DEC_APPLY_LATE) {
        // the rare-path fallback: a small persistent grid, so that returning at once (the common case) costs
        // a few microseconds instead of retiring ~100k one-shot CTAs
        k2_adam<<<grid_for((hi - lo + 7) / 8, ctx->grid_k1s), 256, 0, s>>>(ctx->theta, ctx->m, ctx->v, ctx->w16,
                                                                            ctx->acc, lo, hi, ctx->sc, need);
    } else if (ctx->k2_oneshot)
    {
        const uint16_t* R = ctx->k2_src ? ctx->k2_src : ctx->acc;
        cudaError_t e = launch_pdl(ctx, k2_adam_1, grid, 256, s, ctx->theta, ctx->m, ctx->v, ctx->w16, R, lo, hi,
                                   (const Scalars*)ctx->sc, need);
        if (e != cudaSuccess) return fail_cuda(ctx, e, "k2_adam_1", __LINE__);
    }
    else
        k2_adam<<<grid, 256, 0, s>>>(ctx->theta, ctx->m, ctx->v, ctx->w16, ctx->acc, lo, hi, ctx->sc, need);
    CKL("k2_adam");
    return SMPU_OK;
}

// token count source of the decision kernels: kernel argument, or tok_dev inside a captured graph
const int64_t* tok_src(const smpu_ctx* ctx) { return ctx->capturing ? ctx->tok_dev : nullptr; }

// W = 1, fuse_final: the last micro-batch's elements [lo, hi) fused into Adam (k12_fused).  g[k] points at
// element lo of micro-gradient k; has_acc: R starts from the accumulator (else from g[0]).  The first call of
// an update first enqueues the Adam scalars (k0_fused_prep).
smpu_status launch_k12(smpu_ctx* ctx, const uint16_t* const* g, int count, int64_t lo, int64_t hi, bool has_acc,
                       cudaStream_t s) {
    if (!ctx->fused_prepped) {
        Timed t(ctx, SMPU_K0, s);
        k0_fused_prep<<<1, 32, 0, s>>>(ctx->local_tokens, tok_src(ctx), ctx->st, ctx->sc, ctx->dcfg);
        CKL("k0_fused_prep");
        ctx->fused_prepped = true;
    }
    if (hi <= lo) return SMPU_OK;
    ManyPtrs P;
    for (int k = 0; k < count; ++k) P.g[k] = g[k];
    Timed t(ctx, SMPU_K12, s);
    if (count >= 4) {     // resident micro-batches: 16-element units, four 32-B gradient loads in flight
        const int gm = grid_for((hi - lo + 15) / 16, 0x7fffffff);
        if (has_acc)
            k12_fused_many<true><<<gm, 256, 0, s>>>(ctx->acc, P, count, lo, hi, ctx->theta, ctx->m, ctx->v,
                                                    ctx->theta_b, ctx->m_b, ctx->v_b, ctx->w16, ctx->st, ctx->sc,
                                                    ctx->flag);
        else
            k12_fused_many<false><<<gm, 256, 0, s>>>(ctx->acc, P, count, lo, hi, ctx->theta, ctx->m, ctx->v,
                                                     ctx->theta_b, ctx->m_b, ctx->v_b, ctx->w16, ctx->st, ctx->sc,
                                                     ctx->flag);
        CKL("k12_fused_many");
        return SMPU_OK;
    }
    const int grid = grid_for((hi - lo + 7) / 8, 0x7fffffff);
    if (has_acc)
        k12_fused<true><<<grid, 256, 0, s>>>(ctx->acc, P, count, lo, hi, ctx->theta, ctx->m, ctx->v, ctx->theta_b,
                                             ctx->m_b, ctx->v_b, ctx->w16, ctx->st, ctx->sc, ctx->flag);
    else
        k12_fused<false><<<grid, 256, 0, s>>>(ctx->acc, P, count, lo, hi, ctx->theta, ctx->m, ctx->v, ctx->theta_b,
                                              ctx->m_b, ctx->v_b, ctx->w16, ctx->st, ctx->sc, ctx->flag);
    CKL("k12_fused");
    return SMPU_OK;
}

// host memory: double-buffered H2D staging on the copy stream, overlapped with `launch(stage, c0, c1)` on `s`
// (the staging buffer holds elements [c0, c1))
template <class Launch>
smpu_status staged(smpu_ctx* ctx, const uint16_t* src, int64_t lo, int64_t hi, cudaStream_t s, Launch launch) {
    for (int64_t c0 = lo; c0 < hi; c0 += kStageElems) {
        int64_t c1 = c0 + kStageElems < hi ? c0 + kStageElems : hi;
        int j = (int)(ctx->stage_count++ & 1);
        CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->stage_free[j], 0));
        CK(cudaMemcpyAsync(ctx->stage[j], src + (c0 - lo), (size_t)(c1 - c0) * 2, cudaMemcpyHostToDevice,
                           ctx->copy_stream));
        CK(cudaEventRecord(ctx->stage_full[j], ctx->copy_stream));
        CK(cudaStreamWaitEvent(s, ctx->stage_full[j], 0));
        smpu_status st = launch((const uint16_t*)ctx->stage[j], c0, c1);
        if (st != SMPU_OK) return st;
        CK(cudaEventRecord(ctx->stage_free[j], s));
    }
    return SMPU_OK;
}

// fp32-accumulator K1 (k1_acc32) over [lo, hi); g indexed from lo (nullptr in mode 3)
smpu_status launch_k1_32(smpu_ctx* ctx, int mode, const uint16_t* g, int64_t lo, int64_t hi, bool detect, bool stats,
                         cudaStream_t s) {
    if (hi <= lo) return SMPU_OK;
    const int grid = grid_for((hi - lo + 15) / 16, 0x7fffffff);
    Timed t(ctx, mode == 0 ? SMPU_K1_FIRST : mode == 3 ? SMPU_K1S : SMPU_K1_ADD, s);
    float* a = ctx->acc32;
    uint16_t* h = ctx->acc;
    int* f = ctx->flag;
    uint32_t* st = ctx->stat;
    switch (mode) {
        case 0: k1_acc32<0, false, false><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st); break;
        case 1: k1_acc32<1, false, false><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st); break;
        case 2:
            if (stats) k1_acc32<2, false, true><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st);
            else if (detect) k1_acc32<2, true, false><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st);
            else k1_acc32<2, false, false><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st);
            break;
        default:
            if (stats) k1_acc32<3, false, true><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st);
            else if (detect) k1_acc32<3, true, false><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st);
            else k1_acc32<3, false, false><<<grid, 256, 0, s>>>(a, h, g, lo, hi, f, st);
    }
    CKL("k1_acc32");
    return SMPU_OK;
}

// accumulate src (host or device) into acc[lo, hi); fuse: the last micro-batch at W = 1 with fuse_final, whose
// elements go straight into Adam (launch_k12) instead; last: this is the update's last micro-batch
smpu_status accumulate_range(smpu_ctx* ctx, const uint16_t* src, int64_t lo, int64_t hi, bool first, bool detect,
                             cudaStream_t s, bool stats = false, bool fuse = false, bool last = false) {
    if (ctx->acc32 && !(src && first && last)) {
        // fp32 accumulator (c = 1 with a library-read buffer takes the fp16 path below: rn16(fp32(g_1)) = g_1)
        if (!src) return last ? launch_k1_32(ctx, 3, nullptr, lo, hi, detect, stats, s) : SMPU_OK;
        const int mode = first ? 0 : last ? 2 : 1;
        const PtrKind kind = classify(ctx, src);
        if (kind == PTR_FOREIGN) return set_err(SMPU_EINVAL, "micro-gradients on another device than the ctx's");
        if (kind == PTR_DEVICE) return launch_k1_32(ctx, mode, src, lo, hi, detect, stats, s);
        return staged(ctx, src, lo, hi, s, [&](const uint16_t* g, int64_t c0, int64_t c1) {
            return launch_k1_32(ctx, mode, g, c0, c1, detect, stats, s);
        });
    }
    if (fuse) {
        if (!src) return launch_k12(ctx, nullptr, 0, lo, hi, true, s);
        const PtrKind kind = classify(ctx, src);
        if (kind == PTR_FOREIGN) return set_err(SMPU_EINVAL, "micro-gradients on another device than the ctx's");
        if (kind == PTR_DEVICE) return launch_k12(ctx, &src, 1, lo, hi, !first, s);
        return staged(ctx, src, lo, hi, s, [&](const uint16_t* g, int64_t c0, int64_t c1) {
            return launch_k12(ctx, &g, 1, c0, c1, !first, s);
        });
    }
    if (!src) {
        // accumulated in place by the producer (smpu_accumulator): only the last micro-batch's
        // overflow test / statistic remains to be done
        if ((!detect && !stats) || hi <= lo) return SMPU_OK;
        int grid = grid_for((hi - lo + 15) / 16, 0x7fffffff);
        Timed t(ctx, SMPU_K1S, s);
        if (stats) k1_scan<false, true><<<grid, 256, 0, s>>>(ctx->acc, lo, hi, ctx->flag, ctx->stat);
        else k1_scan<true, false><<<grid, 256, 0, s>>>(ctx->acc, lo, hi, ctx->flag, ctx->stat);
        CKL("k1_scan");
        return SMPU_OK;
    }
    const PtrKind kind = classify(ctx, src);
    if (kind == PTR_FOREIGN) return set_err(SMPU_EINVAL, "micro-gradients on another device than the ctx's");
    if (kind == PTR_DEVICE) return launch_k1(ctx, src, lo, hi, first, detect, s, stats);
    return staged(ctx, src, lo, hi, s, [&](const uint16_t* g, int64_t c0, int64_t c1) {
        return launch_k1(ctx, g, c0, c1, first, detect, s, stats);
    });
}

// one bucket's fused all-reduce (or reduce-scatter, sharded) with the ctx's shape; `grid` CTAs in all
template <class Peers>
smpu_status launch_ar_with(smpu_ctx* ctx, const Peers& pe, int grid, int64_t lo, int64_t hi, cudaStream_t cs) {
    const int g = grid, t = ctx->ar_threads;
#define SMPU_RS(WW) k_rs<WW, Peers><<<g, 256, 0, cs>>>(pe, lo, hi)
#define SMPU_MC(WW) k_ar32<WW, Peers, true><<<g, 256, 0, cs>>>(pe, lo, hi)
#define SMPU_U2(WW) k_ar32<WW, Peers, false, 2><<<g, t, 0, cs>>>(pe, lo, hi)
#define SMPU_V32(WW) k_ar32<WW, Peers><<<g, t, 0, cs>>>(pe, lo, hi)
#define SMPU_V16(WW) k_ar16<WW, Peers><<<g, 256, 0, cs>>>(pe, lo, hi)
    if (ctx->sharded) {
        SMPU_BY_WORLD(ctx->world, SMPU_RS, "fused reduce-scatter")
    } else if (ctx->ar_vec32 && ctx->ar_mcast) {
        if constexpr (std::is_same<Peers, LsaPeers>::value) {
            SMPU_BY_WORLD(ctx->world, SMPU_MC, "fused all-reduce")
        } else {
            return set_err(SMPU_EINVAL, "multicast all-gather needs NVLS (LSA peers)");
        }
    } else if (ctx->ar_vec32 && ctx->ar_unroll == 2) {
        SMPU_BY_WORLD(ctx->world, SMPU_U2, "fused all-reduce")
    } else if (ctx->ar_vec32) {
        SMPU_BY_WORLD(ctx->world, SMPU_V32, "fused all-reduce")
    } else {
        SMPU_BY_WORLD(ctx->world, SMPU_V16, "fused all-reduce")
    }
#undef SMPU_RS
#undef SMPU_MC
#undef SMPU_U2
#undef SMPU_V32
#undef SMPU_V16
    CKL(ctx->sharded ? "k_rs" : "k_ar");
    return SMPU_OK;
}

smpu_status launch_ar_fused(smpu_ctx* ctx, int64_t lo, int64_t hi, cudaStream_t cs) {
    return launch_ar_with(ctx, lsa_peers(ctx), ctx->grid_ar, lo, hi, cs);
}

// Copy-engine all-reduce (smpu_config.ar_copy_engine; lsa_allreduce.cuh "copy-engine variant"): shard p of
// [lo, hi) is [v0 + u_lo(p) * 16, v0 + u_hi(p) * 16) in k_ar32's 16-element units; staging slot s of a piece is at
// window offset stage_off + s * per * 32.
struct CeGeom {
    int64_t v0 = 0, units = 0, per = 0;
    CeGeom(int64_t lo, int64_t hi, int W) {
        v0 = (lo + 15) & ~(int64_t)15;
        const int64_t v1 = hi & ~(int64_t)15;
        units = v1 > v0 ? (v1 - v0) / 16 : 0;
        per = (units + W - 1) / W;
    }
    int64_t ulo(int p) const { return p * per < units ? p * per : units; }
    int64_t uhi(int p) const { return (p + 1) * per < units ? (p + 1) * per : units; }
};

// ar_copy_engine 1: every bucket on the copy engines; 2: every bucket but the last (the last one is ready only when
// the backward has ended, so nothing is left to overlap it with and k_ar32's higher in-situ bandwidth wins)
bool ce_bucket(const smpu_ctx* ctx, int b) { return ctx->ce && (ctx->cfg.ar_copy_engine == 1 || b + 1 < ctx->nb); }

// Copies issued on the ctx's W - 1 copy streams forked from / joined into `cs`: copy j goes to `dst(j)` from
// `src(j)`, `bytes(j)` bytes (skipped when 0).
template <class F>
smpu_status ce_copies(smpu_ctx* ctx, int count, cudaStream_t cs, F&& one) {
    CK(cudaEventRecord(ctx->ce_fork, cs));
    for (int j = 0; j < count; ++j) {
        cudaStream_t st = ctx->ce_stream[j % (ctx->world - 1)];
        CK(cudaStreamWaitEvent(st, ctx->ce_fork, 0));
        void* dst = nullptr;
        const void* src = nullptr;
        size_t bytes = 0;
        one(j, dst, src, bytes);
        if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
        CK(cudaEventRecord(ctx->ce_join[j % (ctx->world - 1)], st));
        CK(cudaStreamWaitEvent(cs, ctx->ce_join[j % (ctx->world - 1)], 0));
    }
    return SMPU_OK;
}

smpu_status launch_ar_ce(smpu_ctx* ctx, int64_t lo, int64_t hi, size_t stage_off, cudaStream_t cs) {
    const int W = ctx->world, r = ctx->rank;
    const CeGeom G(lo, hi, W);
    const LsaPeers pe = lsa_peers(ctx);
    uint16_t* acc = ctx->acc;
    // 1. push my contribution to shard p into p's staging slot r
    smpu_status st = ce_copies(ctx, W - 1, cs, [&](int j, void*& dst, const void*& src, size_t& bytes) {
        const int p = (r + 1 + j) % W;
        dst = ctx->peer_win[p] + stage_off + (size_t)r * G.per * 32;
        src = acc + G.v0 + G.ulo(p) * 16;
        bytes = (size_t)(G.uhi(p) - G.ulo(p)) * 32;
    });
    if (st != SMPU_OK) return st;
    // 2. every rank's pushes have landed; 3. fold my shard (+ rank 0: head / tail over peer memory)
    k_ce_barrier<LsaPeers><<<1, 32, 0, cs>>>(pe, 0);
    CKL("k_ce_barrier");
#define SMPU_CER(WW) k_ce_reduce<WW, LsaPeers><<<ctx->grid_ar, 256, 0, cs>>>(pe, lo, hi, stage_off)
    SMPU_BY_WORLD(W, SMPU_CER, "copy-engine all-reduce")
#undef SMPU_CER
    CKL("k_ce_reduce");
    // 4. all-gather R of my shard into every peer's accumulator; 5. every rank's all-gather has landed
    st = ce_copies(ctx, W - 1, cs, [&](int j, void*& dst, const void*& src, size_t& bytes) {
        const int p = (r + 1 + j) % W;
        const int64_t off = G.v0 + G.ulo(r) * 16;
        dst = ctx->peer_win[p] + (size_t)off * 2;
        src = acc + off;
        bytes = (size_t)(G.uhi(r) - G.ulo(r)) * 32;
    });
    if (st != SMPU_OK) return st;
    k_ce_barrier<LsaPeers><<<1, 32, 0, cs>>>(pe, 1);
    CKL("k_ce_barrier");
    ctx->launches[SMPU_ALLREDUCE] += 2;   // three kernels; the caller's Timed counted one
    return SMPU_OK;
}

// The same over the W windows of a virtual group, on the group's comm stream: the copies between local windows
// (issued through the issuing member's copy streams), one fold launch for every rank, stream order for barriers.
smpu_status launch_ar_ce_group(smpu_ctx* ctx, int64_t lo, int64_t hi, size_t stage_off, cudaStream_t cs) {
    smpu_group* g = ctx->group;
    const int W = g->world;
    const CeGeom G(lo, hi, W);
    char* win[kMaxLsaRanks];
    for (int p = 0; p < W; ++p) win[p] = (char*)g->m[p]->acc;
    // pushes: (r, p) for every ordered pair, rank-major
    smpu_status st = ce_copies(ctx, W * (W - 1), cs, [&](int j, void*& dst, const void*& src, size_t& bytes) {
        const int r = j / (W - 1), p = (r + 1 + j % (W - 1)) % W;
        dst = win[p] + stage_off + (size_t)r * G.per * 32;
        src = win[r] + (size_t)(G.v0 + G.ulo(p) * 16) * 2;
        bytes = (size_t)(G.uhi(p) - G.ulo(p)) * 32;
    });
    if (st != SMPU_OK) return st;
    const LocalPeers pe = local_peers(g, g->per_rank, 0);
#define SMPU_CER(WW) k_ce_reduce<WW, LocalPeers><<<g->per_rank * W, 256, 0, cs>>>(pe, lo, hi, stage_off)
    SMPU_BY_WORLD(W, SMPU_CER, "copy-engine all-reduce")
#undef SMPU_CER
    CKL("k_ce_reduce (virtual)");
    return ce_copies(ctx, W * (W - 1), cs, [&](int j, void*& dst, const void*& src, size_t& bytes) {
        const int r = j / (W - 1), p = (r + 1 + j % (W - 1)) % W;
        const size_t off = (size_t)(G.v0 + G.ulo(r) * 16) * 2;
        dst = win[p] + off;
        src = win[r] + off;
        bytes = (size_t)(G.uhi(r) - G.ulo(r)) * 32;
    });
}

smpu_status launch_k1_many(smpu_ctx* ctx, const uint16_t* const* g, int count, int64_t lo, int64_t hi, bool first,
                           bool detect, bool stats, cudaStream_t s) {
    if (hi <= lo) return SMPU_OK;
    ManyPtrs P;
    for (int k = 0; k < count; ++k) P.g[k] = g[k] + lo;
    int grid = grid_for((hi - lo + 15) / 16, 0x7fffffff);
    Timed t(ctx, SMPU_K1_MANY, s);
    uint16_t* a = ctx->acc;
    int* f = ctx->flag;
    uint32_t* st = ctx->stat;
    if (first) {
        if (stats) k1_accumulate_many<true, false, true><<<grid, 256, 0, s>>>(a, P, count, lo, hi, f, st);
        else if (detect) k1_accumulate_many<true, true, false><<<grid, 256, 0, s>>>(a, P, count, lo, hi, f, st);
        else k1_accumulate_many<true, false, false><<<grid, 256, 0, s>>>(a, P, count, lo, hi, f, st);
    } else {
        if (stats) k1_accumulate_many<false, false, true><<<grid, 256, 0, s>>>(a, P, count, lo, hi, f, st);
        else if (detect) k1_accumulate_many<false, true, false><<<grid, 256, 0, s>>>(a, P, count, lo, hi, f, st);
        else k1_accumulate_many<false, false, false><<<grid, 256, 0, s>>>(a, P, count, lo, hi, f, st);
    }
    CKL("k1_accumulate_many");
    return SMPU_OK;
}

// issue, in canonical bucket order, the all-reduces of every bucket whose final-micro K1 is enqueued
smpu_status issue_ready_buckets(smpu_ctx* ctx) {
    while (ctx->next_issue < ctx->nb && ctx->bucket_done[ctx->next_issue]) {
        int b = ctx->next_issue;
        int64_t lo = ctx->bbegin[b], hi = ctx->bbegin[b + 1];
        cudaStream_t cs = ctx->comm_stream;
        CK(cudaStreamWaitEvent(cs, ctx->ready[b], 0));
        const auto& pc = ctx->pieces[b];
        for (size_t i = 0; i + 1 < pc.size(); ++i) {
            {
                Timed t(ctx, SMPU_ALLREDUCE, cs);
                if (ce_bucket(ctx, b)) {
                    smpu_status st = launch_ar_ce(ctx, pc[i], pc[i + 1], ctx->ce_off[b][i], cs);
                    if (st != SMPU_OK) return st;
                } else if (ctx->ar_impl == SMPU_AR_FUSED) {
                    smpu_status st = launch_ar_fused(ctx, pc[i], pc[i + 1], cs);
                    if (st != SMPU_OK) return st;
                } else {
                    NK(ncclAllReduce(ctx->acc + pc[i], ctx->acc + pc[i], (size_t)(pc[i + 1] - pc[i]), ncclFloat16,
                                     ncclSum, ctx->comm, cs));
                }
            }
            CK(cudaEventRecord(ctx->ar_done[b][i], cs));
        }
        ctx->next_issue++;
    }
    if (ctx->next_issue == ctx->nb) CK(cudaEventRecord(ctx->comm_done, ctx->comm_stream));
    return SMPU_OK;
}

// Virtual group: the all-reduce of bucket b waits for every member's last-micro-batch K1 of b (their ready events)
// and is ONE launch over every rank's window (LocalPeers); it completes every member's ar_done[b].  Issued by the
// member whose call makes bucket b complete, in canonical bucket order.
smpu_status group_issue_buckets(smpu_ctx* ctx) {
    smpu_group* g = ctx->group;
    while (g->next_issue < ctx->nb && g->arrived[g->next_issue] == g->world) {
        const int b = g->next_issue;
        for (smpu_ctx* q : g->m) CK(cudaStreamWaitEvent(g->comm, q->ready[b], 0));
        const auto& pc = ctx->pieces[b];
        for (size_t i = 0; i + 1 < pc.size(); ++i) {
            smpu_status st = ce_bucket(ctx, b) ? launch_ar_ce_group(ctx, pc[i], pc[i + 1], ctx->ce_off[b][i], g->comm)
                                     : launch_ar_with(ctx, local_peers(g, g->per_rank, 0), g->per_rank * g->world,
                                                      pc[i], pc[i + 1], g->comm);
            if (st != SMPU_OK) return st;
            for (smpu_ctx* q : g->m) {
                q->launches[SMPU_ALLREDUCE]++;
                CK(cudaEventRecord(q->ar_done[b][i], g->comm));
            }
        }
        g->arrived[b] = 0;
        g->next_issue++;
    }
    if (g->next_issue == ctx->nb) {
        for (smpu_ctx* q : g->m) CK(cudaEventRecord(q->comm_done, g->comm));
        g->next_issue = 0;
    }
    return SMPU_OK;
}

// bucket b of the last micro-batch (W > 1) is accumulated on `s`: hand it to the all-reduce
smpu_status bucket_ready(smpu_ctx* ctx, int b, cudaStream_t s) {
    ctx->bucket_done[b] = 1;
    CK(cudaEventRecord(ctx->ready[b], s));
    if (ctx->group) {
        ctx->group->arrived[b]++;
        return group_issue_buckets(ctx);
    }
    return issue_ready_buckets(ctx);
}

DecArgs dec_args(const smpu_ctx* q) {
    DecArgs a{};
    a.stat = q->stat;
    a.local_tokens = q->local_tokens;
    a.tok_ptr = tok_src(q);
    a.xs = q->xs;
    a.flag = q->flag;
    a.st = q->st;
    a.sc = q->sc;
    a.loss_scale = q->scale;
    a.ring = q->ring_dev;
    return a;
}

// W > 1, once every bucket of the last micro-batch is accumulated: the exact early overflow decision
// (k0_early_x through peer memory, or k0_early after a 16-byte NCCL all-reduce on a second communicator),
// then Adam per bucket on its own stream, each bucket right behind its gradient all-reduce -- K2 overlaps the
// remaining all-reduces.
smpu_status launch_decision_lsa(smpu_ctx* ctx, cudaStream_t ds) {
    DecArgsW A{};
    A.r[ctx->rank] = dec_args(ctx);
    const LsaPeers pe = lsa_peers(ctx);
#define SMPU_DEC(WW)                                                                                            \
    k0_early_x<WW, LsaPeers, kBoth><<<1, 32, 0, ds>>>(pe, ctx->dec_area_off, A, kRing - 1, ctx->dcfg,          \
                                                      (uint32_t)ctx->grid_ar)
    SMPU_BY_WORLD(ctx->world, SMPU_DEC, "fused decision")
#undef SMPU_DEC
    CKL("k0_early_x");
    return SMPU_OK;
}

// Adam per bucket on the ctx's K2 stream, each bucket behind its all-reduce and the decision (dec_ev)
// Pieces alternate between two Adam streams: a piece whose all-reduce has landed need not wait for the previous
// piece's Adam, which is still sharing HBM with the next all-reduce (the tail's HBM is not saturated: r2n timelines).
smpu_status enqueue_adam(smpu_ctx* ctx) {
    cudaStream_t ks2[2] = {ctx->k2_stream, ctx->k2_stream2};
    for (cudaStream_t ks : ks2) CK(cudaStreamWaitEvent(ks, ctx->dec_ev, 0));
    int j = 0;
    for (int b = 0; b < ctx->nb; ++b) {
        const auto& pc = ctx->pieces[b];
        for (size_t i = 0; i + 1 < pc.size(); ++i, ++j) {   // each piece right behind its all-reduce
            cudaStream_t ks = ks2[j & 1];
            CK(cudaStreamWaitEvent(ks, ctx->ar_done[b][i], 0));
            Timed t(ctx, SMPU_K2, ks);
            smpu_status st = ctx->sharded ? launch_k2_shard(ctx, b, DEC_APPLY, ks)
                                          : launch_k2(ctx, pc[i], pc[i + 1], DEC_APPLY, ks);
            if (st != SMPU_OK) return st;
        }
    }
    CK(cudaEventRecord(ctx->k2_join, ctx->k2_stream2));
    CK(cudaStreamWaitEvent(ctx->k2_stream, ctx->k2_join, 0));
    CK(cudaEventRecord(ctx->k2_done, ctx->k2_stream));
    return SMPU_OK;
}

// Virtual group: once the last member's last micro-batch is in, the decision exchange of every rank as two launches
// (publish every rank's slot, then every rank reads and decides: the launch boundary is the barrier), then each
// member's per-bucket Adam.
smpu_status group_decision(smpu_ctx* ctx) {
    smpu_group* g = ctx->group;
    if (++g->dec_arrived < g->world) return SMPU_OK;
    g->dec_arrived = 0;
    DecArgsW A{};
    for (smpu_ctx* q : g->m) {
        for (int b = 0; b < q->nb; ++b) CK(cudaStreamWaitEvent(g->dec, q->ready[b], 0));
        A.r[q->rank] = dec_args(q);
    }
    const LocalPeers pe = local_peers(g, 1, 0);
    const int W = g->world;
#define SMPU_DEC(WW)                                                                                              \
    k0_early_x<WW, LocalPeers, kPublish><<<W, 32, 0, g->dec>>>(pe, ctx->dec_area_off, A, kRing - 1, ctx->dcfg, 0); \
    k0_early_x<WW, LocalPeers, kDecide><<<W, 32, 0, g->dec>>>(pe, ctx->dec_area_off, A, kRing - 1, ctx->dcfg, 0)
    SMPU_BY_WORLD(W, SMPU_DEC, "virtual decision")
#undef SMPU_DEC
    CKL("k0_early_x (virtual)");
    for (smpu_ctx* q : g->m) {
        q->launches[SMPU_DECISION_AR]++;
        CK(cudaEventRecord(q->dec_ev, g->dec));
    }
    for (smpu_ctx* q : g->m) {
        smpu_status st = enqueue_adam(q);
        if (st != SMPU_OK) return st;
    }
    return SMPU_OK;
}

smpu_status issue_decision(smpu_ctx* ctx) {
    if (ctx->group) return group_decision(ctx);
    cudaStream_t ds = ctx->dec_stream;
    for (int b = 0; b < ctx->nb; ++b) CK(cudaStreamWaitEvent(ds, ctx->ready[b], 0));
    if (ctx->ar_impl == SMPU_AR_FUSED) {
        Timed t(ctx, SMPU_DECISION_AR, ds);
        smpu_status st = launch_decision_lsa(ctx, ds);
        if (st != SMPU_OK) return st;
    } else {
        {
            Timed t(ctx, SMPU_K0, ds);
            k_stats_prep<<<1, 32, 0, ds>>>(ctx->stat, ctx->local_tokens, tok_src(ctx), ctx->xs);
            CKL("k_stats_prep");
        }
        {
            Timed t(ctx, SMPU_DECISION_AR, ds);
            NK(ncclAllReduce(ctx->xs, ctx->xs, 2, ncclInt64, ncclSum, ctx->comm2, ds));   // N, sum_r M_r
        }
        {
            Timed t(ctx, SMPU_K0, ds);
            k0_early<<<1, 32, 0, ds>>>(ctx->xs, ctx->st, ctx->sc, ctx->scale, ctx->ring_dev, kRing - 1, ctx->dcfg);
            CKL("k0_early");
        }
    }
    CK(cudaEventRecord(ctx->dec_ev, ds));
    return enqueue_adam(ctx);
}

// ---------------------------------------------------------------------------------------- virtual group steps
// A member may step once every member has given its c micro-batches (all collectives of the update are then
// issued); in the sharded layout its result exists only once the last member steps, so out must be NULL before.
smpu_status group_step_check(const smpu_ctx* ctx, const smpu_step_result* out) {
    const smpu_group* g = ctx->group;
    for (const smpu_ctx* q : g->m)
        if (!g->stepped[q->rank] && (q->micro != q->cfg.update_freq || q->bucket_micro))
            return set_err(SMPU_ESTATE, "virtual group: every rank gives its %d micro-batches before any rank steps "
                                        "(rank %d has %d)", q->cfg.update_freq, q->rank, q->micro);
    if (ctx->sharded && out && g->n_stepped + 1 < g->world)
        return set_err(SMPU_ESTATE, "virtual group, sharded: the update completes when the last rank steps; pass "
                                    "out = NULL and read smpu_result afterwards");
    return SMPU_OK;
}

void group_mark_stepped(smpu_ctx* ctx) {
    smpu_group* g = ctx->group;
    g->stepped[ctx->rank] = 1;
    if (++g->n_stepped == g->world) {            // the round is closed: every rank may start its next update
        std::fill(g->stepped.begin(), g->stepped.end(), 0);
        g->n_stepped = 0;
    }
}

smpu_status group_round_open_for(const smpu_ctx* ctx) {
    if (ctx->group && ctx->group->stepped[ctx->rank])
        return set_err(SMPU_ESTATE, "virtual group: rank %d stepped; the other ranks step before its next update",
                       ctx->rank);
    return SMPU_OK;
}

// Sharded layout, virtual group: this member's shard sweep is enqueued on s; the rest of the update (late flag
// exchange, late Adam, the end-of-update barrier) runs for every member once the last one steps.
smpu_status group_sharded_tail(smpu_ctx* ctx, cudaStream_t s) {
    smpu_group* g = ctx->group;
    CK(cudaEventRecord(ctx->tail_ev, s));
    ctx->step_stream = s;
    ctx->micro = 0;
    ctx->local_tokens = 0;
    std::fill(ctx->bucket_done.begin(), ctx->bucket_done.end(), 0);
    g->stepped[ctx->rank] = 1;
    if (++g->n_stepped < g->world) return SMPU_OK;
    DecArgsW A{};
    for (smpu_ctx* q : g->m) {
        CK(cudaStreamWaitEvent(g->dec, q->tail_ev, 0));
        A.r[q->rank] = dec_args(q);
    }
    const LocalPeers pe = local_peers(g, 1, 0);
    const int W = g->world;
#define SMPU_KL(WW)                                                                                               \
    k0_late_x<WW, LocalPeers, kPublish><<<W, 32, 0, g->dec>>>(pe, ctx->dec_area_off, A, kRing - 1, ctx->dcfg, 0); \
    k0_late_x<WW, LocalPeers, kDecide><<<W, 32, 0, g->dec>>>(pe, ctx->dec_area_off, A, kRing - 1, ctx->dcfg, 0)
    SMPU_BY_WORLD(W, SMPU_KL, "virtual late decision")
#undef SMPU_KL
    CKL("k0_late_x (virtual)");
    CK(cudaEventRecord(g->late_ev, g->dec));
    for (smpu_ctx* q : g->m) {
        q->launches[SMPU_K0]++;
        CK(cudaStreamWaitEvent(q->step_stream, g->late_ev, 0));
        for (int b = 0; b < q->nb; ++b) {
            q->launches[SMPU_K2]++;
            smpu_status st = launch_k2_shard(q, b, DEC_APPLY_LATE, q->step_stream);
            if (st != SMPU_OK) return st;
        }
        CK(cudaEventRecord(q->tail_ev, q->step_stream));
    }
    // end-of-update barrier: every member's next update waits for every member's w16 stores and window reads
    for (smpu_ctx* q : g->m)
        for (smpu_ctx* p : g->m) CK(cudaStreamWaitEvent(q->step_stream, p->tail_ev, 0));
    for (smpu_ctx* q : g->m) {
        q->attempts++;
        CK(cudaEventRecord(q->ring_ev[(q->attempts - 1) % kRing], q->step_stream));
        smpu_status st = leave_stream(q, q->step_stream);
        if (st != SMPU_OK) return st;
    }
    std::fill(g->stepped.begin(), g->stepped.end(), 0);
    g->n_stepped = 0;
    return SMPU_OK;
}

// split = 0: the paper's plan, whole tensors, a bucket closes once it reaches bucket_bytes (R17).
// split = 1 (smpu_config.split_tensors): fixed-size buckets of bucket_bytes rounded up to 128 elements (256 B),
// cut wherever they fall -- tensors may span buckets; the remainder is the last bucket.
smpu_status plan(const int64_t* numel, int n_tensors, int64_t bucket_bytes, std::vector<int64_t>& out,
                 bool split = false) {
    out.clear();
    out.push_back(0);
    int64_t off = 0, cur = 0;
    if (split) {
        for (int j = 0; j < n_tensors; ++j) {
            if (numel[j] <= 0) return set_err(SMPU_EINVAL, "numel[%d] = %lld must be > 0", j, (long long)numel[j]);
            off += numel[j];
        }
        const int64_t per = ((bucket_bytes / 2 + 127) / 128) * 128;
        for (int64_t b = per; b < off; b += per) out.push_back(b);
        out.push_back(off);
        return SMPU_OK;
    }
    for (int j = 0; j < n_tensors; ++j) {
        if (numel[j] <= 0) return set_err(SMPU_EINVAL, "numel[%d] = %lld must be > 0", j, (long long)numel[j]);
        off += numel[j];
        cur += numel[j] * 2;
        if (cur >= bucket_bytes) {   // close at >= threshold (reading R17)
            out.push_back(off);
            cur = 0;
        }
    }
    if (out.back() != off) out.push_back(off);
    return SMPU_OK;
}

// This rank's element ranges of bucket [lo, hi) in the sharded layout -- the split k_rs_lsa makes on the device:
// 8-element units from the first multiple of 8, ceil(units / W) per rank; rank 0 also owns the unaligned head and
// tail.  Host-only (smpu_plan_shards exports it for tests).
void shard_of_bucket(int64_t lo, int64_t hi, int world, int rank, std::vector<std::pair<int64_t, int64_t>>& out) {
    const int64_t v0 = (lo + 7) & ~(int64_t)7, v1 = hi & ~(int64_t)7;
    const int64_t units = v1 > v0 ? (v1 - v0) / 8 : 0, per = (units + world - 1) / world;
    int64_t u_lo = rank * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    out.push_back({v0 + u_lo * 8, v0 + u_hi * 8});
    if (rank == 0) {
        const int64_t head_end = v0 < hi ? v0 : hi;
        out.push_back({lo, head_end});
        out.push_back({v1 > head_end ? v1 : head_end, hi});
    }
}

smpu_status check_cfg(const smpu_config* c) {
    if (!c) return set_err(SMPU_EINVAL, "null cfg");
    if (c->update_freq < 1) return set_err(SMPU_EINVAL, "update_freq must be >= 1");
    if (c->warmup_updates < 1) return set_err(SMPU_EINVAL, "warmup_updates must be >= 1");
    if (!(c->peak_lr > 0) || !(c->beta1 >= 0 && c->beta1 < 1) || !(c->beta2 >= 0 && c->beta2 < 1) || !(c->eps > 0))
        return set_err(SMPU_EINVAL, "bad Adam / lr hyper-parameters");
    if (c->min_scale_log2 > c->init_scale_log2 || c->init_scale_log2 > c->max_scale_log2 ||
        c->min_scale_log2 < -120 || c->max_scale_log2 > 120)
        return set_err(SMPU_EINVAL, "need min_scale_log2 <= init_scale_log2 <= max_scale_log2 within +-120");
    if (c->growth_interval < 1) return set_err(SMPU_EINVAL, "growth_interval must be >= 1");
    if (c->bucket_bytes < 2) return set_err(SMPU_EINVAL, "bucket_bytes must be >= 2");
    if (c->ar_ctas < 0 || (c->ar_threads != 256 && c->ar_threads != 512) ||
        (c->ar_vec_bytes != 16 && c->ar_vec_bytes != 32) || (c->ar_unroll != 1 && c->ar_unroll != 2) ||
        (c->ar_mcast != 0 && c->ar_mcast != 1) || (c->pdl != 0 && c->pdl != 1) || c->ar_pieces < 1 ||
        c->ar_pieces > 64)
        return set_err(SMPU_EINVAL, "bad all-reduce shape: ar_ctas >= 0, ar_threads 256|512, ar_vec_bytes 16|32, "
                                    "ar_unroll 1|2, ar_mcast 0|1, pdl 0|1, ar_pieces 1..64");
    if (c->ar_mcast && c->ar_vec_bytes != 32)
        return set_err(SMPU_EINVAL, "ar_mcast needs ar_vec_bytes = 32");
    if (c->ar_copy_engine < 0 || c->ar_copy_engine > 2) return set_err(SMPU_EINVAL, "ar_copy_engine must be 0|1|2");
    if (c->ar_copy_engine && (c->sharded || c->ar_mcast || c->allreduce == SMPU_AR_NCCL))
        return set_err(SMPU_EINVAL, "ar_copy_engine runs the replicated fused all-reduce only (not with sharded, "
                                    "ar_mcast or SMPU_AR_NCCL)");
    return SMPU_OK;
}

void free_ctx(smpu_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    cudaDeviceSynchronize();
    if (c->have_devcomm) ncclDevCommDestroy(c->comm, &c->devcomm);
    if (c->win) ncclCommWindowDeregister(c->comm, c->win);
    if (c->comm2) ncclCommDestroy(c->comm2);
    if (c->comm) ncclCommDestroy(c->comm);
    cudaFree(c->theta);
    cudaFree(c->m);
    cudaFree(c->v);
    cudaFree(c->theta_b);
    cudaFree(c->acc32);
    cudaFree(c->m_b);
    cudaFree(c->v_b);
    if (!c->w16_in_win) cudaFree(c->w16);
    if (c->acc_from_nccl) ncclMemFree(c->acc);
    else cudaFree(c->acc);
    cudaFree(c->flag);
    cudaFree(c->stat);
    cudaFree(c->xs);
    cudaFree(c->st);
    cudaFree(c->sc);
    cudaFree(c->scale);
    cudaFree(c->stage[0]);
    cudaFree(c->stage[1]);
    if (c->ring_host) cudaFreeHost(c->ring_host);
    for (auto& e : c->ring_ev) if (e) cudaEventDestroy(e);
    for (auto& e : c->ready) if (e) cudaEventDestroy(e);
    for (auto& v : c->ar_done)
        for (auto& e : v) if (e) cudaEventDestroy(e);
    if (c->dec_ev) cudaEventDestroy(c->dec_ev);
    if (c->k2_done) cudaEventDestroy(c->k2_done);
    if (c->tail_ev) cudaEventDestroy(c->tail_ev);
    if (c->dec_stream) cudaStreamDestroy(c->dec_stream);
    if (c->k2_stream) cudaStreamDestroy(c->k2_stream);
    if (c->k2_stream2) cudaStreamDestroy(c->k2_stream2);
    if (c->k2_join) cudaEventDestroy(c->k2_join);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (int j = 0; j < 2; ++j) {
        if (c->stage_free[j]) cudaEventDestroy(c->stage_free[j]);
        if (c->stage_full[j]) cudaEventDestroy(c->stage_full[j]);
    }
    if (c->comm_done) cudaEventDestroy(c->comm_done);
    if (c->order_ev) cudaEventDestroy(c->order_ev);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    for (auto& x : c->ce_stream) if (x) cudaStreamDestroy(x);
    for (auto& e : c->ce_join) if (e) cudaEventDestroy(e);
    if (c->ce_fork) cudaEventDestroy(c->ce_fork);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    cudaFree(c->tok_dev);
    if (c->tok_host) cudaFreeHost(c->tok_host);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
}

void start_micro(smpu_ctx* c, int64_t ntokens) {
    c->micro++;
    c->local_tokens += ntokens;
}

bool final_micro(const smpu_ctx* c) { return c->micro == c->cfg.update_freq; }

}  // namespace

// ================================================================================================ C ABI
extern "C" {

int smpu_abi_version(void) { return SMPU_ABI_VERSION; }

const char* smpu_last_error(void) { return g_err.c_str(); }

smpu_status smpu_config_default(smpu_config* c) {
    if (!c) return set_err(SMPU_EINVAL, "null cfg");
    c->peak_lr = 5e-4;
    c->warmup_updates = 4000;
    c->beta1 = 0.9;
    c->beta2 = 0.98;
    c->eps = 1e-8;
    c->init_scale_log2 = 7;
    c->min_scale_log2 = -5;
    c->max_scale_log2 = 24;
    c->growth_interval = 2000;
    c->update_freq = 1;
    c->bucket_bytes = int64_t(150) << 20;
    c->allreduce = SMPU_AR_AUTO;
    c->sharded = 0;
    c->fuse_final = 0;
    c->accum_fp32 = 0;
    c->split_tensors = 0;
    c->ar_ctas = 0;
    c->ar_threads = 256;
    c->ar_vec_bytes = 32;
    c->ar_unroll = 1;
    c->ar_mcast = 0;
    c->pdl = 1;
    c->ar_pieces = 1;
    c->ar_copy_engine = 0;
    return SMPU_OK;
}

smpu_status smpu_unique_id(void* out, int64_t bytes) {
    smpu_ctx* ctx = nullptr;
    if (!out || bytes < (int64_t)sizeof(ncclUniqueId)) return set_err(SMPU_EINVAL, "need a >= 128-byte buffer");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof id);
    return SMPU_OK;
}

smpu_status smpu_plan_buckets(const int64_t* numel, int n_tensors, int64_t bucket_bytes, int* n_buckets,
                              int64_t* bucket_begin) {
    if (!numel || n_tensors < 1 || !n_buckets || bucket_bytes < 2) return set_err(SMPU_EINVAL, "bad arguments");
    std::vector<int64_t> b;
    smpu_status s = plan(numel, n_tensors, bucket_bytes, b);
    if (s != SMPU_OK) return s;
    *n_buckets = (int)b.size() - 1;
    if (bucket_begin) memcpy(bucket_begin, b.data(), b.size() * sizeof(int64_t));
    return SMPU_OK;
}

smpu_status smpu_plan_shards(const int64_t* bucket_begin, int n_buckets, int world, int rank, int64_t* ranges,
                             int cap, int* count) {
    if (!bucket_begin || n_buckets < 1 || world < 1 || rank < 0 || rank >= world || !count)
        return set_err(SMPU_EINVAL, "bad arguments");
    for (int b = 0; b < n_buckets; ++b)
        if (bucket_begin[b + 1] < bucket_begin[b]) return set_err(SMPU_EINVAL, "bucket_begin must not decrease");
    int k = 0;
    for (int b = 0; b < n_buckets; ++b) {
        std::vector<std::pair<int64_t, int64_t>> v;
        shard_of_bucket(bucket_begin[b], bucket_begin[b + 1], world, rank, v);
        for (auto& rg : v) {
            if (rg.second <= rg.first) continue;
            if (ranges && k < cap) {
                ranges[2 * k] = rg.first;
                ranges[2 * k + 1] = rg.second;
            }
            ++k;
        }
    }
    *count = k;
    return SMPU_OK;
}

// MIN and MAX over the ranks of v[0..k) (int64): one NCCL MAX all-reduce of [v, -v]
static ncclResult_t agree(ncclComm_t comm, cudaStream_t st, const int64_t* v, int k, int64_t* mn, int64_t* mx) {
    std::vector<int64_t> h(2 * k);
    for (int i = 0; i < k; ++i) {
        h[i] = v[i];
        h[k + i] = -v[i];
    }
    int64_t* d = nullptr;
    if (cudaMalloc(&d, 2 * k * sizeof(int64_t)) != cudaSuccess) return ncclUnhandledCudaError;
    ncclResult_t r = ncclSuccess;
    if (cudaMemcpy(d, h.data(), 2 * k * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess)
        r = ncclUnhandledCudaError;
    if (r == ncclSuccess) r = ncclAllReduce(d, d, (size_t)(2 * k), ncclInt64, ncclMax, comm, st);
    if (r == ncclSuccess && cudaStreamSynchronize(st) != cudaSuccess) r = ncclUnhandledCudaError;
    if (r == ncclSuccess && cudaMemcpy(h.data(), d, 2 * k * sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
        r = ncclUnhandledCudaError;
    cudaFree(d);
    for (int i = 0; i < k; ++i) {
        mx[i] = h[i];
        mn[i] = -h[k + i];
    }
    return r;
}

// One ctx: rank `rank` of `world` over NCCL (group == nullptr), or virtual rank `rank` of a one-GPU group.
static smpu_status create_ctx(smpu_ctx** out, const smpu_config* cfg, int world, int rank, const void* nccl_id,
                              int cuda_device, const int64_t* numel, int n_tensors, const float* init_params,
                              smpu_group* group) {
    smpu_ctx* ctx = new smpu_ctx();
    ctx->cfg = *cfg;
    ctx->world = world;
    ctx->rank = rank;
    ctx->dev = cuda_device;
    ctx->group = group;
    smpu_status s = plan(numel, n_tensors, cfg->bucket_bytes, ctx->bbegin, cfg->split_tensors != 0);
    if (s != SMPU_OK) {
        delete ctx;
        return s;
    }
    ctx->nb = (int)ctx->bbegin.size() - 1;
    {
        ctx->tensor_bucket.resize(n_tensors);
        ctx->tensor_bucket_last.resize(n_tensors);
        ctx->bucket_tensors.assign(ctx->nb, 0);
        int64_t off = 0;
        int b = 0;
        for (int j = 0; j < n_tensors; ++j) {
            while (b + 1 < ctx->nb && off >= ctx->bbegin[b + 1]) ++b;
            int e = b;
            while (e + 1 < ctx->nb && off + numel[j] > ctx->bbegin[e + 1]) ++e;
            ctx->tensor_bucket[j] = b;
            ctx->tensor_bucket_last[j] = e;
            for (int k = b; k <= e; ++k) ctx->bucket_tensors[k]++;
            off += numel[j];
        }
        ctx->bucket_tensors_left = ctx->bucket_tensors;
        ctx->tensor_seen.assign(n_tensors, 0);
    }
    ctx->n = ctx->bbegin.back();
    const int64_t n = ctx->n;

    auto bail = [&](smpu_status st) {
        std::string keep = g_err;
        free_ctx(ctx);
        g_err = keep;
        return st;
    };
#define IK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            return bail(e_ == cudaErrorMemoryAllocation                                \
                            ? set_err(SMPU_ENOMEM, "%s: out of memory", #x)            \
                            : fail_cuda(nullptr, e_, #x, __LINE__));                   \
    } while (0)
#define IN(x, what)                                                                    \
    do {                                                                               \
        ncclResult_t r_ = (x);                                                         \
        if (r_ != ncclSuccess) return bail(fail_nccl(nullptr, r_, what, __LINE__));    \
    } while (0)

    IK(cudaSetDevice(cuda_device));
    cudaDeviceProp prop;
    IK(cudaGetDeviceProperties(&prop, cuda_device));
    if (prop.major != 10 || prop.minor != 0)
        return bail(set_err(SMPU_EINVAL, "libsmpu.so is built for sm_100a (B200); device %d is sm_%d%d", cuda_device,
                            prop.major, prop.minor));
    IK(cudaMalloc(&ctx->theta, n * 4));
    IK(cudaMalloc(&ctx->m, n * 4));
    IK(cudaMalloc(&ctx->v, n * 4));
    ctx->fused = world == 1 && cfg->fuse_final != 0 && !cfg->accum_fp32;
    if (cfg->accum_fp32) IK(cudaMalloc(&ctx->acc32, n * 4));
    if (ctx->fused) {
        IK(cudaMalloc(&ctx->theta_b, n * 4));
        IK(cudaMalloc(&ctx->m_b, n * 4));
        IK(cudaMalloc(&ctx->v_b, n * 4));
    }

    // all-reduce pieces: with ar_pieces = P (replicated layout, world > 1) every bucket is cut into P pieces on
    // 256-element boundaries, each all-reduced and then updated on its own, so that Adam of piece i overlaps the
    // all-reduce of piece i + 1 and the Adam chain starts after the first piece instead of the first bucket.  Values
    // never change (elementwise).
    ctx->pieces.resize(ctx->nb);
    ctx->ar_done.resize(ctx->nb);
    for (int b = 0; b < ctx->nb; ++b) {
        const int64_t lo = ctx->bbegin[b], hi = ctx->bbegin[b + 1];
        const int split = (!cfg->sharded && world > 1) ? cfg->ar_pieces : 1;
        auto& pc = ctx->pieces[b];
        pc.push_back(lo);
        const int64_t step = (hi - lo + split - 1) / split;
        for (int i = 1; i < split; ++i) {
            const int64_t cut = (lo + i * step + 255) & ~(int64_t)255;
            if (cut > pc.back() && cut < hi) pc.push_back(cut);
        }
        pc.push_back(hi);
        ctx->ar_done[b].assign(pc.size() - 1, nullptr);
        for (auto& e : ctx->ar_done[b]) IK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const size_t acc_bytes = ((size_t)n * 2 + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
                             NCCL_WIN_REQUIRED_ALIGNMENT;
    const size_t w16_bytes = ((size_t)n * 2 + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
                             NCCL_WIN_REQUIRED_ALIGNMENT;
    // window = [acc | w16 | decision area (early + late exchange slots: 2 parities x 8 ranks x 16 B each) |
    //           copy-engine staging (ar_copy_engine: per piece, W slots of one shard each)]
    ctx->w16_off = acc_bytes;
    ctx->dec_area_off = acc_bytes + w16_bytes;
    size_t win_bytes = acc_bytes + w16_bytes + NCCL_WIN_REQUIRED_ALIGNMENT;
    ctx->ce = world > 1 && cfg->ar_copy_engine != 0;
    if (ctx->ce) {
        ctx->ce_off.resize(ctx->nb);
        for (int b = 0; b < ctx->nb; ++b) {
            const auto& pc = ctx->pieces[b];
            for (size_t i = 0; i + 1 < pc.size(); ++i) {
                const int64_t v0 = (pc[i] + 15) & ~(int64_t)15, v1 = pc[i + 1] & ~(int64_t)15;
                const int64_t units = v1 > v0 ? (v1 - v0) / 16 : 0, per = (units + world - 1) / world;
                ctx->ce_off[b].push_back(win_bytes);
                win_bytes += ((size_t)world * per * 32 + 255) & ~(size_t)255;
            }
        }
        win_bytes = (win_bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
                    NCCL_WIN_REQUIRED_ALIGNMENT;
    }
    if (cfg->sharded && world > 1 && cfg->allreduce == SMPU_AR_NCCL)
        return bail(set_err(SMPU_EINVAL, "the sharded optimizer needs the fused all-reduce"));
    if (group) {
        IK(cudaMalloc(&ctx->acc, win_bytes));            // a virtual rank's window: plain device memory
        ctx->w16_in_win = true;
    } else if (world > 1 && cfg->allreduce != SMPU_AR_NCCL && world <= kMaxLsaRanks &&
               ncclMemAlloc((void**)&ctx->acc, win_bytes) == ncclSuccess) {
        ctx->acc_from_nccl = true;
        ctx->w16_in_win = true;
    } else {
        IK(cudaMalloc(&ctx->acc, acc_bytes));
    }
    if (ctx->w16_in_win) ctx->w16 = (uint16_t*)((char*)ctx->acc + ctx->w16_off);
    else IK(cudaMalloc(&ctx->w16, n * 2));
    IK(cudaMalloc(&ctx->flag, sizeof(int)));
    IK(cudaMalloc(&ctx->stat, sizeof(uint32_t)));
    IK(cudaMalloc(&ctx->tok_dev, sizeof(int64_t)));
    IK(cudaHostAlloc(&ctx->tok_host, kRing * sizeof(int64_t), cudaHostAllocDefault));
    IK(cudaMalloc(&ctx->xs, 2 * sizeof(int64_t)));
    IK(cudaMalloc(&ctx->st, sizeof(DevState)));
    IK(cudaMalloc(&ctx->sc, sizeof(Scalars)));
    IK(cudaMalloc(&ctx->scale, sizeof(float)));
    IK(cudaMalloc(&ctx->stage[0], kStageElems * 2));
    IK(cudaMalloc(&ctx->stage[1], kStageElems * 2));
    IK(cudaHostAlloc(&ctx->ring_host, kRing * sizeof(smpu_step_result), cudaHostAllocMapped));
    IK(cudaHostGetDevicePointer((void**)&ctx->ring_dev, ctx->ring_host, 0));
    memset(ctx->ring_host, 0, kRing * sizeof(smpu_step_result));
    for (auto& e : ctx->ring_ev) IK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ready.resize(ctx->nb);
    for (auto& e : ctx->ready) IK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    IK(cudaEventCreateWithFlags(&ctx->dec_ev, cudaEventDisableTiming));
    IK(cudaEventCreateWithFlags(&ctx->k2_done, cudaEventDisableTiming));
    IK(cudaEventCreateWithFlags(&ctx->tail_ev, cudaEventDisableTiming));
    ctx->bucket_done.assign(ctx->nb, 0);
    IK(cudaEventCreateWithFlags(&ctx->comm_done, cudaEventDisableTiming));
    IK(cudaEventCreateWithFlags(&ctx->order_ev, cudaEventDisableTiming));
    int lo_prio = 0, hi_prio = 0;
    IK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    IK(cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, hi_prio));
    IK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    IK(cudaStreamCreateWithPriority(&ctx->dec_stream, cudaStreamNonBlocking, hi_prio));
    IK(cudaStreamCreateWithFlags(&ctx->k2_stream, cudaStreamNonBlocking));
    IK(cudaStreamCreateWithFlags(&ctx->k2_stream2, cudaStreamNonBlocking));
    IK(cudaEventCreateWithFlags(&ctx->k2_join, cudaEventDisableTiming));
    for (int j = 0; j < 2; ++j) {
        IK(cudaEventCreateWithFlags(&ctx->stage_free[j], cudaEventDisableTiming));
        IK(cudaEventCreateWithFlags(&ctx->stage_full[j], cudaEventDisableTiming));
        IK(cudaEventRecord(ctx->stage_free[j], ctx->copy_stream));
    }

    // K1 / K2: one-shot grids by default (grid_cap); the K1s sweep: a persistent grid of resident CTAs x SMs
    int occ = 0;
    ctx->grid_k1 = grid_cap("SMPU_K1_CTAS_PER_SM", prop.multiProcessorCount, 0);
    ctx->k1_oneshot = ctx->grid_k1 == 0x7fffffff;
    ctx->grid_k2 = grid_cap("SMPU_K2_CTAS_PER_SM", prop.multiProcessorCount, 0);
    ctx->k2_oneshot = ctx->grid_k2 == 0x7fffffff;
    ctx->pdl = world == 1 && cfg->pdl != 0;
    IK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1s_sweep, 256, 0));
    ctx->grid_k1s = prop.multiProcessorCount * (occ > 0 ? occ : 1);
    // the fused all-reduce's shape (smpu_config.ar_*): one CTA per SM with 256-bit peer accesses by default,
    // measured best at W = 2 and 4 (fewer CTAs starve NVLink, more steal issue slots and HBM from the concurrent
    // K1 / K2)
    ctx->grid_ar = cfg->ar_ctas > 0 ? cfg->ar_ctas : prop.multiProcessorCount;
    ctx->ar_vec32 = cfg->ar_vec_bytes == 32;
    ctx->ar_unroll = cfg->ar_unroll;
    ctx->ar_threads = cfg->ar_threads;

    DevCfg& d = ctx->dcfg;
    d.peak_lr = cfg->peak_lr;
    d.warmup = cfg->warmup_updates;
    d.beta1 = cfg->beta1;
    d.beta2 = cfg->beta2;
    d.eps = cfg->eps;
    d.emin = cfg->min_scale_log2;
    d.emax = cfg->max_scale_log2;
    d.growth = cfg->growth_interval;

    cudaStream_t s0 = ctx->copy_stream;
    IK(cudaMemcpyAsync(ctx->theta, init_params, n * 4, cudaMemcpyDefault, s0));
    IK(cudaMemsetAsync(ctx->m, 0, n * 4, s0));
    IK(cudaMemsetAsync(ctx->v, 0, n * 4, s0));
    if (ctx->fused) {
        IK(cudaMemsetAsync(ctx->theta_b, 0, n * 4, s0));
        IK(cudaMemsetAsync(ctx->m_b, 0, n * 4, s0));
        IK(cudaMemsetAsync(ctx->v_b, 0, n * 4, s0));
    }
    IK(cudaMemsetAsync(ctx->acc, 0, n * 2, s0));
    if (ctx->w16_in_win) IK(cudaMemsetAsync((char*)ctx->acc + ctx->dec_area_off, 0, win_bytes - ctx->dec_area_off, s0));
    if (ctx->acc32) IK(cudaMemsetAsync(ctx->acc32, 0, n * 4, s0));
    IK(cudaMemsetAsync(ctx->flag, 0, sizeof(int), s0));
    IK(cudaMemsetAsync(ctx->stat, 0, sizeof(uint32_t), s0));
    IK(cudaMemsetAsync(ctx->xs, 0, 2 * sizeof(int64_t), s0));
    IK(cudaMemsetAsync(ctx->sc, 0, sizeof(Scalars), s0));
    DevState st0{cfg->init_scale_log2, 0, 0, 0};
    IK(cudaMemcpyAsync(ctx->st, &st0, sizeof st0, cudaMemcpyHostToDevice, s0));
    float sc0 = ldexpf(1.0f, cfg->init_scale_log2);
    IK(cudaMemcpyAsync(ctx->scale, &sc0, sizeof sc0, cudaMemcpyHostToDevice, s0));
    IK(cudaStreamSynchronize(s0));

    if (group) {
        // every virtual rank was given the same theta_0 (the group init's broadcast); the peer kernels need no setup
        ctx->ar_impl = SMPU_AR_FUSED;
        ctx->sharded = cfg->sharded != 0;
    } else if (world > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof id);
        IN(ncclCommInitRank(&ctx->comm, world, id, rank), "ncclCommInitRank");
        // Every rank must agree on what shapes the collectives (plan, knobs) and on whether the fused path is
        // possible, before any collective resource is created: a difference would otherwise hang some ranks in
        // window registration or in LSA barriers the others never join.  EINVAL on every rank instead.
        static const char* kField[] = {"update_freq", "bucket_bytes", "split_tensors", "sharded", "accum_fp32",
                                       "allreduce", "ar_ctas", "ar_threads", "ar_vec_bytes", "ar_unroll", "ar_mcast",
                                       "ar_pieces", "ar_copy_engine", "n (parameter count)", "n_buckets",
                                       "symmetric-memory allocation"};
        const int64_t mine[] = {cfg->update_freq, cfg->bucket_bytes, cfg->split_tensors, cfg->sharded,
                                cfg->accum_fp32, cfg->allreduce, ctx->grid_ar, cfg->ar_threads, cfg->ar_vec_bytes,
                                cfg->ar_unroll, cfg->ar_mcast, cfg->ar_pieces, cfg->ar_copy_engine, n, ctx->nb,
                                ctx->acc_from_nccl ? 1 : 0};
        constexpr int K = sizeof(mine) / sizeof(mine[0]);
        int64_t mn[K], mx[K];
        IN(agree(ctx->comm, s0, mine, K, mn, mx), "rank agreement all-reduce");
        for (int i = 0; i < K - 1; ++i)
            if (mn[i] != mx[i])
                return bail(set_err(SMPU_EINVAL, "ranks disagree on smpu_config.%s (%lld .. %lld): every rank must "
                                                 "pass the same config and tensor list", kField[i], (long long)mn[i],
                                    (long long)mx[i]));
        const bool window_everywhere = mn[K - 1] == 1;
        // replicas start bitwise identical: rank 0's theta_0
        IN(ncclBroadcast(ctx->theta, ctx->theta, (size_t)n, ncclFloat32, 0, ctx->comm, s0), "ncclBroadcast");
        IN(ncclCommSplit(ctx->comm, 0, rank, &ctx->comm2, nullptr), "ncclCommSplit");
        ctx->ar_impl = SMPU_AR_NCCL;
        if (window_everywhere) {
            // symmetric window over the accumulator + device communicator with one LSA barrier per CTA
            IN(ncclCommWindowRegister(ctx->comm, ctx->acc, win_bytes, &ctx->win, NCCL_WIN_COLL_SYMMETRIC),
               "ncclCommWindowRegister");
            ncclDevCommRequirements reqs;
            memset(&reqs, 0, sizeof reqs);
            // one per all-reduce CTA (indices 0 / 1 also serve the copy-engine all-reduce's barrier kernels) +
            // early decision + late decision + end-of-update (sharded)
            reqs.lsaBarrierCount = ctx->grid_ar + 3;
            reqs.lsaMultimem = cfg->ar_mcast != 0;
            ncclResult_t r = ncclDevCommCreate(ctx->comm, &reqs, &ctx->devcomm);
            ctx->have_devcomm = r == ncclSuccess;
            const int64_t ok = r == ncclSuccess && ctx->devcomm.lsaSize == world && ctx->devcomm.lsaRank == rank;
            int64_t okmn, okmx;
            IN(agree(ctx->comm, s0, &ok, 1, &okmn, &okmx), "rank agreement all-reduce");
            if (okmn == 1) {
                ctx->ar_impl = SMPU_AR_FUSED;
                ctx->ar_mcast = cfg->ar_mcast != 0;
            } else if (cfg->ar_mcast) {
                return bail(set_err(SMPU_EINVAL, "ar_mcast: NVLS multicast unavailable on some rank (NCCL %d here)",
                                    (int)r));
            }
        }
        if (cfg->allreduce == SMPU_AR_FUSED && ctx->ar_impl != SMPU_AR_FUSED)
            return bail(set_err(SMPU_EINVAL, "fused all-reduce requested but unavailable on some rank (needs every "
                                             "rank an NVLink load/store peer, world <= %d)", kMaxLsaRanks));
        ctx->sharded = cfg->sharded && ctx->ar_impl == SMPU_AR_FUSED;
        if (cfg->sharded && !ctx->sharded)
            return bail(set_err(SMPU_EINVAL, "the sharded optimizer needs the fused all-reduce (unavailable)"));
        if (ctx->ce && ctx->ar_impl != SMPU_AR_FUSED)
            return bail(set_err(SMPU_EINVAL, "ar_copy_engine needs the fused all-reduce's window (unavailable)"));
        if (ctx->ce) {
            // every rank's window as a VA of this process: the copy engines' push / all-gather destinations
            unsigned long long* d = nullptr;
            unsigned long long h[kMaxLsaRanks] = {};
            IK(cudaMalloc(&d, sizeof h));
            k_peer_ptrs<LsaPeers><<<1, 32, 0, s0>>>(lsa_peers(ctx), world, d);
            IK(cudaGetLastError());
            IK(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, s0));
            IK(cudaStreamSynchronize(s0));
            IK(cudaFree(d));
            for (int p = 0; p < world; ++p) ctx->peer_win[p] = (char*)(uintptr_t)h[p];
        }
    }
    if (ctx->ce) {
        IK(cudaEventCreateWithFlags(&ctx->ce_fork, cudaEventDisableTiming));
        for (int j = 0; j + 1 < world; ++j) {
            IK(cudaStreamCreateWithPriority(&ctx->ce_stream[j], cudaStreamNonBlocking, hi_prio));
            IK(cudaEventCreateWithFlags(&ctx->ce_join[j], cudaEventDisableTiming));
        }
    }
    if (ctx->sharded) {
        // the same shard split as k_rs: 8-element units, ceil(units / W) per rank, rank 0 also owns the bucket's
        // unaligned head and tail
        ctx->shard.resize(ctx->nb);
        for (int b = 0; b < ctx->nb; ++b)
            shard_of_bucket(ctx->bbegin[b], ctx->bbegin[b + 1], world, rank, ctx->shard[b]);
    }
    kc_cast<<<grid_for(n, ctx->grid_k2), 256, 0, s0>>>(ctx->theta, ctx->w16, n);
    ctx->launches[SMPU_KCAST]++;
    IK(cudaGetLastError());
    IK(cudaStreamSynchronize(s0));
#undef IK
#undef IN
    *out = ctx;
    return SMPU_OK;
}

smpu_status smpu_init(smpu_ctx** out, const smpu_config* cfg, int world, int rank, const void* nccl_id,
                      int cuda_device, const int64_t* numel, int n_tensors, const float* init_params) {
    if (!out) return set_err(SMPU_EINVAL, "null out");
    *out = nullptr;
    smpu_status s = check_cfg(cfg);
    if (s != SMPU_OK) return s;
    if (world < 1 || rank < 0 || rank >= world) return set_err(SMPU_EINVAL, "need 0 <= rank < world");
    if (world > 1 && !nccl_id) return set_err(SMPU_EINVAL, "world > 1 needs an NCCL unique id");
    if (!numel || n_tensors < 1 || !init_params) return set_err(SMPU_EINVAL, "null tensor list / params");
    return create_ctx(out, cfg, world, rank, nccl_id, cuda_device, numel, n_tensors, init_params, nullptr);
}

smpu_status smpu_group_init(smpu_group** out, const smpu_config* cfg, int world, int cuda_device, const int64_t* numel,
                            int n_tensors, const float* init_params) {
    if (!out) return set_err(SMPU_EINVAL, "null out");
    *out = nullptr;
    smpu_status s = check_cfg(cfg);
    if (s != SMPU_OK) return s;
    if (world < 2 || world > kMaxLsaRanks) return set_err(SMPU_EINVAL, "a virtual group has 2..%d ranks", kMaxLsaRanks);
    if (cfg->allreduce == SMPU_AR_NCCL) return set_err(SMPU_EINVAL, "a virtual group runs the fused all-reduce only");
    if (cfg->ar_mcast) return set_err(SMPU_EINVAL, "a virtual group has no NVLS multicast (ar_mcast = 0)");
    if (!numel || n_tensors < 1 || !init_params) return set_err(SMPU_EINVAL, "null tensor list / params");
    smpu_group* g = new smpu_group();
    g->world = world;
    g->dev = cuda_device;
    smpu_ctx* ctx = nullptr;   // for CK: errors before any member exists poison nothing
    auto bail = [&](smpu_status st) {
        std::string keep = g_err;
        smpu_group_destroy(g);
        g_err = keep;
        return st;
    };
    if (cudaSetDevice(cuda_device) != cudaSuccess) return bail(set_err(SMPU_EINVAL, "bad device %d", cuda_device));
    int lo_prio = 0, hi_prio = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&g->comm, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&g->dec, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->late_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(fail_cuda(ctx, e, "virtual group streams", __LINE__));
    for (int r = 0; r < world; ++r) {
        smpu_ctx* m = nullptr;
        s = create_ctx(&m, cfg, world, r, nullptr, cuda_device, numel, n_tensors, init_params, g);
        if (s != SMPU_OK) return bail(s);
        g->m.push_back(m);
    }
    g->arrived.assign(g->m[0]->nb, 0);
    g->stepped.assign(world, 0);
    g->per_rank = (g->m[0]->grid_ar + world - 1) / world;
    *out = g;
    return SMPU_OK;
}

smpu_status smpu_group_member(smpu_group* g, int rank, smpu_ctx** out) {
    if (!g || !out) return set_err(SMPU_EINVAL, "null argument");
    if (rank < 0 || rank >= g->world) return set_err(SMPU_EINVAL, "rank %d out of [0, %d)", rank, g->world);
    *out = g->m[rank];
    return SMPU_OK;
}

void smpu_group_destroy(smpu_group* g) {
    if (!g) return;
    for (smpu_ctx* m : g->m) free_ctx(m);
    cudaSetDevice(g->dev);
    if (g->late_ev) cudaEventDestroy(g->late_ev);
    if (g->comm) cudaStreamDestroy(g->comm);
    if (g->dec) cudaStreamDestroy(g->dec);
    delete g;
}

smpu_status smpu_num_params(const smpu_ctx* ctx, int64_t* n) {
    if (!ctx || !n) return set_err(SMPU_EINVAL, "null argument");
    *n = ctx->n;
    return SMPU_OK;
}

smpu_status smpu_shard_ranges(const smpu_ctx* ctx, int64_t* ranges, int cap, int* count) {
    if (!ctx || !count) return set_err(SMPU_EINVAL, "null argument");
    int k = 0;
    if (!ctx->sharded) {
        if (ranges && cap > 0) {
            ranges[0] = 0;
            ranges[1] = ctx->n;
        }
        *count = 1;
        return SMPU_OK;
    }
    for (auto& v : ctx->shard)
        for (auto& rg : v) {
            if (rg.second <= rg.first) continue;
            if (ranges && k < cap) {
                ranges[2 * k] = rg.first;
                ranges[2 * k + 1] = rg.second;
            }
            ++k;
        }
    *count = k;
    return SMPU_OK;
}

smpu_status smpu_allreduce_impl(const smpu_ctx* ctx, int* impl) {
    if (!ctx || !impl) return set_err(SMPU_EINVAL, "null argument");
    *impl = ctx->world > 1 ? ctx->ar_impl : 0;
    return SMPU_OK;
}

smpu_status smpu_buckets(const smpu_ctx* ctx, int* n_buckets, int64_t* bucket_begin) {
    if (!ctx || !n_buckets) return set_err(SMPU_EINVAL, "null argument");
    *n_buckets = ctx->nb;
    if (bucket_begin) memcpy(bucket_begin, ctx->bbegin.data(), ctx->bbegin.size() * sizeof(int64_t));
    return SMPU_OK;
}

smpu_status smpu_accumulator(const smpu_ctx* ctx, void** dev_acc) {
    if (!ctx || !dev_acc) return set_err(SMPU_EINVAL, "null argument");
    *dev_acc = ctx->acc32 ? (void*)ctx->acc32 : (void*)ctx->acc;
    return SMPU_OK;
}

smpu_status smpu_weights_fp16(const smpu_ctx* ctx, const void** dev_w16) {
    if (!ctx || !dev_w16) return set_err(SMPU_EINVAL, "null argument");
    *dev_w16 = ctx->w16;
    return SMPU_OK;
}

smpu_status smpu_loss_scale(const smpu_ctx* ctx, const float** dev_scale) {
    if (!ctx || !dev_scale) return set_err(SMPU_EINVAL, "null argument");
    *dev_scale = ctx->scale;
    return SMPU_OK;
}

smpu_status smpu_micro_begin(smpu_ctx* ctx, int64_t ntokens) {
    LIVE(ctx);
    if (group_round_open_for(ctx) != SMPU_OK) return SMPU_ESTATE;
    if (ntokens < 0) return set_err(SMPU_EINVAL, "ntokens < 0");
    if (ctx->bucket_micro) return set_err(SMPU_ESTATE, "previous bucket-wise micro-batch still has %d buckets", ctx->buckets_left);
    if (ctx->micro >= ctx->cfg.update_freq)
        return set_err(SMPU_ESTATE, "already %d micro-batches this update; call smpu_step", ctx->micro);
    CK(cudaSetDevice(ctx->dev));
    start_micro(ctx, ntokens);
    ctx->bucket_micro = true;
    ctx->buckets_left = ctx->nb;
    std::fill(ctx->bucket_done.begin(), ctx->bucket_done.end(), 0);
    ctx->bucket_tensors_left = ctx->bucket_tensors;
    std::fill(ctx->tensor_seen.begin(), ctx->tensor_seen.end(), 0);
    return SMPU_OK;
}

smpu_status smpu_tensor_ready(smpu_ctx* ctx, int tensor, void* stream) {
    LIVE(ctx);
    if (!ctx->bucket_micro) return set_err(SMPU_ESTATE, "smpu_tensor_ready without smpu_micro_begin");
    if (tensor < 0 || tensor >= (int)ctx->tensor_bucket.size())
        return set_err(SMPU_EINVAL, "tensor %d out of [0, %d)", tensor, (int)ctx->tensor_bucket.size());
    if (ctx->tensor_seen[tensor]) return set_err(SMPU_ESTATE, "tensor %d already ready in this micro-batch", tensor);
    const int b0 = ctx->tensor_bucket[tensor], b1 = ctx->tensor_bucket_last[tensor];
    for (int b = b0; b <= b1; ++b)
        if (ctx->bucket_done[b]) return set_err(SMPU_ESTATE, "bucket %d of tensor %d was already given", b, tensor);
    ctx->tensor_seen[tensor] = 1;
    // "when the gradient computation for a layer finishes, we add the result to a synchronization buffer; as
    // soon as the size of the buffer reaches a predefined threshold we synchronize"
    for (int b = b0; b <= b1; ++b)
        if (--ctx->bucket_tensors_left[b] == 0) {
            smpu_status st = smpu_accumulate_bucket(ctx, b, nullptr, stream);
            if (st != SMPU_OK) return st;
        }
    return SMPU_OK;
}

smpu_status smpu_accumulate_bucket(smpu_ctx* ctx, int bucket, const void* grads, void* stream) {
    LIVE(ctx);
    if (!ctx->bucket_micro) return set_err(SMPU_ESTATE, "smpu_accumulate_bucket without smpu_micro_begin");
    if (bucket < 0 || bucket >= ctx->nb) return set_err(SMPU_EINVAL, "bucket %d out of [0, %d)", bucket, ctx->nb);
    if (ctx->bucket_done[bucket]) return set_err(SMPU_ESTATE, "bucket %d already given in this micro-batch", bucket);
    CK(cudaSetDevice(ctx->dev));
    if (grads && classify(ctx, grads) == PTR_FOREIGN)
        return set_err(SMPU_EINVAL, "bucket gradients on another device than the ctx's (%d)", ctx->dev);
    cudaStream_t s = (cudaStream_t)stream;
    smpu_status st = enter_stream(ctx, s);
    if (st != SMPU_OK) return st;
    const bool last = final_micro(ctx);
    const bool first = ctx->micro == 1;
    const bool multi = last && ctx->world > 1;
    st = accumulate_range(ctx, (const uint16_t*)grads, ctx->bbegin[bucket], ctx->bbegin[bucket + 1], first,
                          last && ctx->world == 1 && !ctx->fused, s, multi, last && ctx->fused, last);
    if (st != SMPU_OK) return st;
    if (multi) {
        st = bucket_ready(ctx, bucket, s);
        if (st != SMPU_OK) return st;
    } else {
        ctx->bucket_done[bucket] = 1;
    }
    st = leave_stream(ctx, s);
    if (st != SMPU_OK) return st;
    if (--ctx->buckets_left == 0) {
        ctx->bucket_micro = false;
        if (multi) return issue_decision(ctx);
    }
    return SMPU_OK;
}

smpu_status smpu_accumulate(smpu_ctx* ctx, const void* grads, int64_t ntokens, void* stream) {
    LIVE(ctx);
    if (group_round_open_for(ctx) != SMPU_OK) return SMPU_ESTATE;
    if (ntokens < 0) return set_err(SMPU_EINVAL, "ntokens < 0");
    if (ctx->bucket_micro) return set_err(SMPU_ESTATE, "a bucket-wise micro-batch is open");
    if (ctx->micro >= ctx->cfg.update_freq)
        return set_err(SMPU_ESTATE, "already %d micro-batches this update; call smpu_step", ctx->micro);
    CK(cudaSetDevice(ctx->dev));
    if (grads && classify(ctx, grads) == PTR_FOREIGN)
        return set_err(SMPU_EINVAL, "micro-gradients on another device than the ctx's (%d)", ctx->dev);
    cudaStream_t s = (cudaStream_t)stream;
    if (ctx->micro + 1 == ctx->cfg.update_freq && ctx->world > 1) {
        // final micro-batch of a multi-GPU update: bucket by bucket, so that bucket b's all-reduce
        // overlaps the accumulation of buckets > b
        smpu_status st = smpu_micro_begin(ctx, ntokens);
        if (st != SMPU_OK) return st;
        const uint16_t* g = (const uint16_t*)grads;
        for (int b = 0; b < ctx->nb; ++b) {
            st = smpu_accumulate_bucket(ctx, b, g ? g + ctx->bbegin[b] : nullptr, stream);
            if (st != SMPU_OK) return st;
        }
        return SMPU_OK;
    }
    smpu_status st = enter_stream(ctx, s);
    if (st != SMPU_OK) return st;
    start_micro(ctx, ntokens);
    const bool last = final_micro(ctx);
    st = accumulate_range(ctx, (const uint16_t*)grads, 0, ctx->n, ctx->micro == 1, last && !ctx->fused, s, false,
                          last && ctx->fused, last);
    if (st != SMPU_OK) return st;
    return leave_stream(ctx, s);
}

smpu_status smpu_accumulate_many(smpu_ctx* ctx, const void* const* grads, const int64_t* ntokens, int count,
                                 void* stream) {
    LIVE(ctx);
    if (!grads || !ntokens || count < 1 || count > kMaxMany) return set_err(SMPU_EINVAL, "need 1..%d buffers", kMaxMany);
    if (group_round_open_for(ctx) != SMPU_OK) return SMPU_ESTATE;
    if (ctx->bucket_micro) return set_err(SMPU_ESTATE, "a bucket-wise micro-batch is open");
    if (ctx->micro + count > ctx->cfg.update_freq)
        return set_err(SMPU_ESTATE, "%d + %d micro-batches exceed update_freq %d", ctx->micro, count,
                       ctx->cfg.update_freq);
    CK(cudaSetDevice(ctx->dev));
    const uint16_t* g[kMaxMany];
    for (int k = 0; k < count; ++k) {
        if (ntokens[k] < 0) return set_err(SMPU_EINVAL, "ntokens[%d] < 0", k);
        if (!grads[k] || classify(ctx, grads[k]) != PTR_DEVICE)
            return set_err(SMPU_EINVAL, "micro_grads[%d] must be a device buffer", k);
        g[k] = (const uint16_t*)grads[k];
    }
    if (ctx->acc32) {     // fp32 accumulator: one pass per micro-batch (the same sums as consecutive calls)
        for (int k = 0; k < count; ++k) {
            smpu_status st = smpu_accumulate(ctx, grads[k], ntokens[k], stream);
            if (st != SMPU_OK) return st;
        }
        return SMPU_OK;
    }
    cudaStream_t s = (cudaStream_t)stream;
    smpu_status st = enter_stream(ctx, s);
    if (st != SMPU_OK) return st;
    const bool first = ctx->micro == 0;
    for (int k = 0; k < count; ++k) start_micro(ctx, ntokens[k]);
    const bool last = final_micro(ctx);
    if (last && ctx->world > 1) {
        // bucket by bucket, so that bucket b's all-reduce overlaps the accumulation of buckets > b
        for (int b = 0; b < ctx->nb; ++b) {
            st = launch_k1_many(ctx, g, count, ctx->bbegin[b], ctx->bbegin[b + 1], first, false, true, s);
            if (st != SMPU_OK) return st;
            st = bucket_ready(ctx, b, s);
            if (st != SMPU_OK) return st;
        }
        st = leave_stream(ctx, s);
        if (st != SMPU_OK) return st;
        return issue_decision(ctx);
    }
    st = last && ctx->fused ? launch_k12(ctx, g, count, 0, ctx->n, !first, s)
                            : launch_k1_many(ctx, g, count, 0, ctx->n, first, last, false, s);
    if (st != SMPU_OK) return st;
    return leave_stream(ctx, s);
}

smpu_status smpu_allreduce_accumulator(smpu_ctx* ctx, void* stream) {
    LIVE(ctx);
    if (ctx->micro != 0 || ctx->bucket_micro) return set_err(SMPU_ESTATE, "smpu_allreduce_accumulator inside an update");
    if (ctx->world == 1) return SMPU_OK;
    if (ctx->sharded) return set_err(SMPU_EINVAL, "the sharded ctx reduce-scatters; no all-reduce to run");
    if (ctx->group) return set_err(SMPU_EINVAL, "virtual group members all-reduce inside updates only");
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = (cudaStream_t)stream;
    smpu_status st = enter_stream(ctx, s);
    if (st != SMPU_OK) return st;
    for (int b = 0; b < ctx->nb; ++b) {
        CK(cudaEventRecord(ctx->ready[b], s));
        ctx->bucket_done[b] = 1;
    }
    ctx->next_issue = 0;
    st = issue_ready_buckets(ctx);
    std::fill(ctx->bucket_done.begin(), ctx->bucket_done.end(), 0);
    ctx->next_issue = 0;
    if (st != SMPU_OK) return st;
    CK(cudaStreamWaitEvent(s, ctx->comm_done, 0));
    return leave_stream(ctx, s);
}

smpu_status smpu_result(smpu_ctx* ctx, int64_t attempt, smpu_step_result* out) {
    LIVE(ctx);
    if (!out) return set_err(SMPU_EINVAL, "null out");
    if (attempt < ctx->first_attempt || attempt > ctx->attempts || attempt <= ctx->attempts - kRing)
        return set_err(SMPU_EINVAL, "attempt %lld not among the last %d (issued %lld)", (long long)attempt, kRing,
                       (long long)ctx->attempts);
    int slot = (int)((attempt - 1) % kRing);
    CK(cudaEventSynchronize(ctx->ring_ev[slot]));
    memcpy(out, (const void*)&ctx->ring_host[slot], sizeof *out);
    return SMPU_OK;
}

smpu_status smpu_step(smpu_ctx* ctx, void* stream, smpu_step_result* out) {
    LIVE(ctx);
    if (ctx->micro != ctx->cfg.update_freq || ctx->bucket_micro)
        return set_err(SMPU_ESTATE, "smpu_step after %d of %d micro-batches%s", ctx->micro, ctx->cfg.update_freq,
                       ctx->bucket_micro ? " (a bucket-wise micro-batch is incomplete)" : "");
    if (ctx->group) {
        smpu_status gs = group_step_check(ctx, out);
        if (gs != SMPU_OK) return gs;
    }
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = (cudaStream_t)stream;
    smpu_status st = enter_stream(ctx, s);
    if (st != SMPU_OK) return st;
    if (ctx->world > 1 && ctx->sharded) {
        // sharded variant: sweep my shard of R, OR the flags through peer memory, Adam on my shard (all three
        // return at once when K0 EARLY decided), then one barrier so that every rank's w16 stores (and reads
        // of my accumulator) are complete before anybody's next update
        CK(cudaStreamWaitEvent(s, ctx->comm_done, 0));
        CK(cudaStreamWaitEvent(s, ctx->k2_done, 0));
        for (int b = 0; b < ctx->nb; ++b)
            for (auto& rg : ctx->shard[b]) {
                if (rg.second <= rg.first) continue;
                Timed t(ctx, SMPU_K1S, s);
                k1s_sweep<<<grid_for((rg.second - rg.first + 15) / 16, ctx->grid_k1s), 256, 0, s>>>(
                    ctx->acc, rg.first, rg.second, ctx->flag, ctx->sc);
                CKL("k1s_sweep");
            }
        if (ctx->group) return group_sharded_tail(ctx, s);
        {
            Timed t(ctx, SMPU_K0, s);
            DecArgsW A{};
            A.r[ctx->rank] = dec_args(ctx);
            const LsaPeers pe = lsa_peers(ctx);
            const uint32_t bi = (uint32_t)ctx->grid_ar + 1;
#define SMPU_KL(WW) k0_late_x<WW, LsaPeers, kBoth><<<1, 32, 0, s>>>(pe, ctx->dec_area_off, A, kRing - 1, ctx->dcfg, bi)
            SMPU_BY_WORLD(ctx->world, SMPU_KL, "sharded path")
#undef SMPU_KL
            CKL("k0_late_x");
        }
        for (int b = 0; b < ctx->nb; ++b) {
            Timed t(ctx, SMPU_K2, s);
            smpu_status st2 = launch_k2_shard(ctx, b, DEC_APPLY_LATE, s);
            if (st2 != SMPU_OK) return st2;
        }
        {
            Timed t(ctx, SMPU_K0, s);
            k_lsa_barrier<<<1, 32, 0, s>>>(lsa_peers(ctx), (uint32_t)ctx->grid_ar + 2);
            CKL("k_lsa_barrier");
        }
    } else if (ctx->world > 1) {
        // the exact early decision and the per-bucket Adam are already enqueued (issue_decision); here only
        // the fallback for the rare undecided case: sweep R, decide, Adam on everything.  All three kernels
        // return at once when K0 EARLY decided.
        CK(cudaStreamWaitEvent(s, ctx->comm_done, 0));
        CK(cudaStreamWaitEvent(s, ctx->k2_done, 0));
        {
            Timed t(ctx, SMPU_K1S, s);
            k1s_sweep<<<ctx->grid_k1s, 256, 0, s>>>(ctx->acc, 0, ctx->n, ctx->flag, ctx->sc);
            CKL("k1s_sweep");
        }
        {
            Timed t(ctx, SMPU_K0, s);
            k0_late<<<1, 32, 0, s>>>(ctx->flag, ctx->xs, ctx->st, ctx->sc, ctx->scale, ctx->ring_dev, kRing - 1,
                                     ctx->dcfg);
            CKL("k0_late");
        }
        {
            Timed t(ctx, SMPU_K2, s);
            smpu_status st2 = launch_k2(ctx, 0, ctx->n, DEC_APPLY_LATE, s);
            if (st2 != SMPU_OK) return st2;
        }
    } else if (ctx->fused) {
        // the update already ran speculatively into the other bank (k12_fused): decide, make that bank current
        // if R was finite, else re-cast w16 from the current theta
        {
            Timed t(ctx, SMPU_K0, s);
            k0_decide<<<1, 32, 0, s>>>(ctx->flag, ctx->local_tokens, tok_src(ctx), ctx->st, ctx->sc, ctx->scale,
                                       ctx->ring_dev, (int)(kRing - 1), ctx->dcfg, 1);
            CKL("k0_decide");
        }
        {
            Timed t(ctx, SMPU_KCAST, s);
            kc_restore<<<ctx->grid_k1s, 256, 0, s>>>(ctx->theta, ctx->theta_b, ctx->st, ctx->sc, ctx->w16, ctx->n);
            CKL("kc_restore");
        }
        ctx->fused_prepped = false;
    } else {
        {
            Timed t(ctx, SMPU_K0, s);
            cudaError_t e = launch_pdl(ctx, k0_decide, 1, 32, s, ctx->flag, ctx->local_tokens, tok_src(ctx), ctx->st,
                                       ctx->sc, ctx->scale, ctx->ring_dev, (int)(kRing - 1), ctx->dcfg, 0);
            if (e != cudaSuccess) return fail_cuda(ctx, e, "k0_decide", __LINE__);
            CKL("k0_decide");
        }
        {
            Timed t(ctx, SMPU_K2, s);
            smpu_status st2 = launch_k2(ctx, 0, ctx->n, DEC_APPLY, s);
            if (st2 != SMPU_OK) return st2;
        }
    }
    if (ctx->capturing) {                // smpu_graph_capture restores the host bookkeeping
        ctx->micro = 0;
        ctx->local_tokens = 0;
        ctx->next_issue = 0;
        std::fill(ctx->bucket_done.begin(), ctx->bucket_done.end(), 0);
        return SMPU_OK;
    }
    ctx->attempts++;
    CK(cudaEventRecord(ctx->ring_ev[(ctx->attempts - 1) % kRing], s));
    st = leave_stream(ctx, s);
    if (st != SMPU_OK) return st;
    ctx->micro = 0;
    ctx->local_tokens = 0;
    ctx->next_issue = 0;
    std::fill(ctx->bucket_done.begin(), ctx->bucket_done.end(), 0);
    if (ctx->group) group_mark_stepped(ctx);
    if (!out) return SMPU_OK;
    st = smpu_result(ctx, ctx->attempts, out);
    if (st != SMPU_OK) return st;
    if (out->discarded) return set_err(SMPU_ESTATE, "N = 0 tokens in this update: discarded (reading R19)");
    return SMPU_OK;
}

smpu_status smpu_graph_capture(smpu_ctx* ctx, const void* const* micro_grads, int count, int flags) {
    LIVE(ctx);
    if (!micro_grads || count != ctx->cfg.update_freq)
        return set_err(SMPU_EINVAL, "need update_freq = %d micro-gradient buffers", ctx->cfg.update_freq);
    if (ctx->micro != 0 || ctx->bucket_micro) return set_err(SMPU_ESTATE, "smpu_graph_capture inside an update");
    if (ctx->group) return set_err(SMPU_EINVAL, "graph capture of a virtual group member is not supported");
    if (ctx->world > 1 && ctx->ar_impl != SMPU_AR_FUSED)
        return set_err(SMPU_EINVAL, "graph capture at world > 1 needs the fused all-reduce (SMPU_AR_FUSED): replays "
                                    "of captured NCCL collectives on two communicators hung on B200 (2 ranks)");
    CK(cudaSetDevice(ctx->dev));
    for (int k = 0; k < count; ++k)
        if (!micro_grads[k] || classify(ctx, micro_grads[k]) != PTR_DEVICE)
            return set_err(SMPU_EINVAL, "micro_grads[%d] must be a device buffer for graph capture", k);
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    if (ctx->graph_exec) {
        CK(cudaGraphExecDestroy(ctx->graph_exec));
        ctx->graph_exec = nullptr;
    }
    ctx->graph_direct = false;
    CK(cudaDeviceSynchronize());
    const bool timing = ctx->timing;
    ctx->timing = false;
    ctx->capturing = true;
    // the launch counters tick while the update is captured: the difference is one replay's kernels
    int64_t before[SMPU_N_KERNELS];
    memcpy(before, ctx->launches, sizeof before);
    cudaGraph_t graph = nullptr;
    smpu_status st = SMPU_OK;
    cudaError_t e = cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
        if (ctx->cfg.update_freq == 1 && ctx->world == 1 && ctx->k2_oneshot && !ctx->fused &&
            ((uintptr_t)micro_grads[0] & 31) == 0) {
            // c = 1, W = 1: R = g_1.  The buffer is fixed and read at replay, so nothing needs copying: test it
            // for overflow in place (2 B/elem) and let Adam read it directly -- 30 instead of 32 B/elem.  Only for
            // a 32-byte aligned buffer (k1_scan / k2_adam_1 take its vectors as they do the library's own arrays);
            // any other buffer is accumulated as usual.
            // (The accumulator, smpu_get_state(ACCUM), is then left untouched by these replays.)
            Timed t(ctx, SMPU_K1S, ctx->cap_stream);
            k1_scan<true, false><<<grid_for((ctx->n + 15) / 16, 0x7fffffff), 256, 0, ctx->cap_stream>>>(
                (const uint16_t*)micro_grads[0], 0, ctx->n, ctx->flag, ctx->stat);
            cudaError_t el = cudaGetLastError();
            if (el != cudaSuccess) st = fail_cuda(ctx, el, "k1_scan", __LINE__);
            start_micro(ctx, 0);
            ctx->k2_src = (const uint16_t*)micro_grads[0];
            ctx->graph_direct = true;
        } else if (flags & SMPU_GRAPH_RESIDENT) {
            std::vector<int64_t> zeros(count, 0);
            st = smpu_accumulate_many(ctx, micro_grads, zeros.data(), count, ctx->cap_stream);
        } else {
            for (int k = 0; k < count && st == SMPU_OK; ++k)
                st = smpu_accumulate(ctx, micro_grads[k], 0, ctx->cap_stream);
        }
        if (st == SMPU_OK) st = smpu_step(ctx, ctx->cap_stream, nullptr);
        ctx->k2_src = nullptr;
        cudaError_t e2 = cudaStreamEndCapture(ctx->cap_stream, &graph);
        if (e == cudaSuccess) e = e2;
    }
    ctx->capturing = false;
    ctx->timing = timing;
    ctx->fused_prepped = false;
    for (int k = 0; k < SMPU_N_KERNELS; ++k) {
        ctx->graph_launches[k] = ctx->launches[k] - before[k];
        ctx->launches[k] = before[k];
    }
    ctx->micro = 0;
    ctx->bucket_micro = false;
    ctx->local_tokens = 0;
    ctx->next_issue = 0;
    std::fill(ctx->bucket_done.begin(), ctx->bucket_done.end(), 0);
    if (st != SMPU_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (e != cudaSuccess) return fail_cuda(ctx, e, "stream capture of the update", __LINE__);
    ctx->graph_resident = (flags & SMPU_GRAPH_RESIDENT) != 0 && !ctx->graph_direct;
    e = cudaGraphInstantiate(&ctx->graph_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail_cuda(ctx, e, "cudaGraphInstantiate", __LINE__);
    return SMPU_OK;
}

smpu_status smpu_graph_launch(smpu_ctx* ctx, const int64_t* ntokens, int count, void* stream) {
    LIVE(ctx);
    if (!ctx->graph_exec) return set_err(SMPU_ESTATE, "no captured update graph (smpu_graph_capture)");
    if (!ntokens || count != ctx->cfg.update_freq) return set_err(SMPU_EINVAL, "need update_freq token counts");
    if (ctx->micro != 0 || ctx->bucket_micro) return set_err(SMPU_ESTATE, "smpu_graph_launch inside an update");
    int64_t N = 0;
    for (int k = 0; k < count; ++k) {
        if (ntokens[k] < 0) return set_err(SMPU_EINVAL, "ntokens[%d] < 0", k);
        N += ntokens[k];
    }
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = (cudaStream_t)stream;
    smpu_status st = enter_stream(ctx, s);
    if (st != SMPU_OK) return st;
    const int slot = (int)(ctx->attempts % kRing);
    if (ctx->attempts >= kRing) CK(cudaEventSynchronize(ctx->ring_ev[slot]));   // slot's previous copy has run
    ctx->tok_host[slot] = N;
    CK(cudaMemcpyAsync(ctx->tok_dev, &ctx->tok_host[slot], sizeof(int64_t), cudaMemcpyHostToDevice, s));
    for (int k = 0; k < SMPU_N_KERNELS; ++k) ctx->launches[k] += ctx->graph_launches[k];
    CK(cudaGraphLaunch(ctx->graph_exec, s));
    ctx->attempts++;
    CK(cudaEventRecord(ctx->ring_ev[(ctx->attempts - 1) % kRing], s));
    return leave_stream(ctx, s);
}

// the ctx's device is current and its work complete (the bank of a fused ctx is read from the device)
static smpu_status state_array(smpu_ctx* ctx, int which, void** p, int64_t* bytes) {
    int64_t bank = 0;
    if (ctx->fused && which >= SMPU_STATE_MASTER && which <= SMPU_STATE_V)
        CK(cudaMemcpy(&bank, &ctx->st->bank, sizeof bank, cudaMemcpyDeviceToHost));
    switch (which) {
        case SMPU_STATE_MASTER: *p = bank ? ctx->theta_b : ctx->theta; *bytes = ctx->n * 4; break;
        case SMPU_STATE_M: *p = bank ? ctx->m_b : ctx->m; *bytes = ctx->n * 4; break;
        case SMPU_STATE_V: *p = bank ? ctx->v_b : ctx->v; *bytes = ctx->n * 4; break;
        case SMPU_STATE_W16: *p = ctx->w16; *bytes = ctx->n * 2; break;
        case SMPU_STATE_ACCUM: *p = ctx->acc; *bytes = ctx->n * 2; break;
        case SMPU_STATE_SCALARS: *p = ctx->st; *bytes = 4 * sizeof(int64_t); break;
        default: return set_err(SMPU_EINVAL, "unknown state selector %d", which);
    }
    return SMPU_OK;
}

smpu_status smpu_get_state(smpu_ctx* ctx, int which, void* dst, int64_t bytes) {
    LIVE(ctx);
    if (!dst) return set_err(SMPU_EINVAL, "null dst");
    CK(cudaSetDevice(ctx->dev));
    CK(cudaDeviceSynchronize());
    void* p;
    int64_t nb;
    smpu_status s = state_array(ctx, which, &p, &nb);
    if (s != SMPU_OK) return s;
    if (bytes != nb) return set_err(SMPU_EINVAL, "state %d is %lld bytes, got %lld", which, (long long)nb, (long long)bytes);
    CK(cudaMemcpy(dst, p, (size_t)nb, cudaMemcpyDefault));
    return SMPU_OK;
}

smpu_status smpu_set_state(smpu_ctx* ctx, int which, const void* src, int64_t bytes) {
    LIVE(ctx);
    if (!src) return set_err(SMPU_EINVAL, "null src");
    if (ctx->micro != 0 || ctx->bucket_micro) return set_err(SMPU_ESTATE, "smpu_set_state in the middle of an update");
    CK(cudaSetDevice(ctx->dev));
    CK(cudaDeviceSynchronize());
    void* p;
    int64_t nb;
    smpu_status s = state_array(ctx, which, &p, &nb);
    if (s != SMPU_OK) return s;
    if (bytes != nb) return set_err(SMPU_EINVAL, "state %d is %lld bytes, got %lld", which, (long long)nb, (long long)bytes);
    if (which == SMPU_STATE_SCALARS) {
        int64_t v[4];
        memcpy(v, src, sizeof v);
        if (v[0] < ctx->cfg.min_scale_log2 || v[0] > ctx->cfg.max_scale_log2 || v[1] < 0 || v[2] < 0 || v[3] < 0)
            return set_err(SMPU_EINVAL, "scalar state out of range");
        CK(cudaMemcpy(p, src, (size_t)nb, cudaMemcpyHostToDevice));
        float sc = ldexpf(1.0f, (int)v[0]);
        CK(cudaMemcpy(ctx->scale, &sc, sizeof sc, cudaMemcpyHostToDevice));
        ctx->attempts = v[3];
        ctx->first_attempt = v[3] + 1;     // the ring holds no result of a restored attempt
        return SMPU_OK;
    }
    CK(cudaMemcpy(p, src, (size_t)nb, cudaMemcpyDefault));
    return SMPU_OK;
}

smpu_status smpu_get_master(smpu_ctx* ctx, float* dst, int64_t n) {
    LIVE(ctx);
    if (n != ctx->n) return set_err(SMPU_EINVAL, "n = %lld, ctx has %lld", (long long)n, (long long)ctx->n);
    return smpu_get_state(ctx, SMPU_STATE_MASTER, dst, n * 4);
}

smpu_status smpu_set_timing(smpu_ctx* ctx, int enable) {
    LIVE(ctx);
    ctx->timing = enable != 0;
    return SMPU_OK;
}

smpu_status smpu_kernel_stats(smpu_ctx* ctx, int64_t* launches, double* total_ms, int reset) {
    LIVE(ctx);
    if (!launches) return set_err(SMPU_EINVAL, "null launches");
    CK(cudaSetDevice(ctx->dev));
    CK(cudaDeviceSynchronize());
    for (int k = 0; k < SMPU_N_KERNELS; ++k) {
        launches[k] = ctx->launches[k];
        if (total_ms) {
            double tot = 0;
            for (auto& pr : ctx->timed[k]) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
                tot += ms;
            }
            total_ms[k] = tot;
        }
    }
    if (reset) {
        for (int k = 0; k < SMPU_N_KERNELS; ++k) {
            ctx->launches[k] = 0;
            ctx->timed[k].clear();
        }
        ctx->trace.clear();
        ctx->ev_used = 0;
    }
    return SMPU_OK;
}

smpu_status smpu_kernel_trace(smpu_ctx* ctx, int32_t* kind, int32_t* stream, double* start_ms, double* end_ms,
                              int64_t cap, int64_t* count) {
    LIVE(ctx);
    if (!count || cap < 0) return set_err(SMPU_EINVAL, "null count / negative cap");
    CK(cudaSetDevice(ctx->dev));
    CK(cudaDeviceSynchronize());
    *count = (int64_t)ctx->trace.size();
    if (ctx->trace.empty()) return SMPU_OK;
    cudaEvent_t origin = ctx->trace[0].b;
    for (int64_t i = 0; i < cap && i < (int64_t)ctx->trace.size(); ++i) {
        const auto& r = ctx->trace[i];
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, origin, r.b));
        CK(cudaEventElapsedTime(&b, origin, r.e));
        if (kind) kind[i] = r.kind;
        if (stream) stream[i] = r.stream;
        if (start_ms) start_ms[i] = a;
        if (end_ms) end_ms[i] = b;
    }
    return SMPU_OK;
}

void smpu_destroy(smpu_ctx* ctx) {
    if (ctx && ctx->group) return;   // a group member: smpu_group_destroy frees it
    free_ctx(ctx);
}

}  // extern "C"
