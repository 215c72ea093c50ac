/*
 * smpu.h -- Synchronous Mixed-Precision large-batch Update step: C ABI of libsmpu.so.
 *
 * The data-parallel hot path of Ott et al., "Scaling Neural Machine Translation"
 * (arXiv 1806.00187), built B200-native (sm_100a).  One update step is
 *
 *   c x accumulate(micro_grads, ntokens)   fp16 gradient accumulation over `update_freq`
 *                                          sub-batches ("cumul", PAPER.md 4.2 P:178, Table 1)
 *   bucketed fp16 all-reduce, overlapped   "as soon as the size of the buffer reaches a predefined
 *                                          threshold we synchronize" (PAPER.md 4.3 P:209-212, 150MB fn)
 *   step()                                 overflow test, dynamic loss scaler, unscale and
 *                                          normalise by the global target-token count,
 *                                          fp32-master Adam 0.9/0.98/1e-8 with the
 *                                          inverse-sqrt warmup LR, fp16 re-cast.
 *
 * Conventions for every call
 *  - Pointers marked "device" are CUDA device pointers of the ctx's device; "host or device" pointers
 *    are classified with cudaPointerGetAttributes (pinned or pageable host memory is accepted).  Device
 *    memory of another GPU is refused with SMPU_EINVAL.
 *  - `stream` arguments are cudaStream_t values passed as void*; NULL means the legacy default stream.
 *    Reads of caller buffers are stream-ordered on that stream: the caller may reuse a buffer after
 *    later work on the same stream.  Different calls may use different streams; the library orders its
 *    own state across them with events.
 *  - Every call returns smpu_status.  SMPU_EINVAL / SMPU_ESTATE leave the ctx unchanged (except where
 *    stated).  SMPU_ECUDA / SMPU_ENCCL poison the ctx: every later call returns SMPU_EPOISONED.
 *    smpu_last_error() gives a thread-local message for the last failing call.
 *  - Non-finite gradients are NOT errors: they are the overflow signal the method reacts to.
 *  - A ctx is not thread-safe.  All ranks of a world must make the same sequence of calls (NCCL).
 *  - Arrays are packed in gradient-READY order (reverse forward order): tensor j occupies
 *    elements [sum_{i<j} numel_i, sum_{i<=j} numel_i) of every per-parameter vector.  No padding.
 */
#ifndef SMPU_H
#define SMPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMPU_ABI_VERSION 4
#define SMPU_NCCL_ID_BYTES 128

typedef struct smpu_ctx smpu_ctx;
typedef struct smpu_group smpu_group;   /* W virtual ranks on one GPU (smpu_group_init) */

typedef enum {
    SMPU_OK = 0,
    SMPU_EINVAL = 1,     /* null / misaligned / out-of-range argument                                  */
    SMPU_ESTATE = 2,     /* call-order violation (see smpu_step); also N = 0 at step (update discarded)   */
    SMPU_ECUDA = 3,      /* CUDA runtime error: ctx poisoned                                            */
    SMPU_ENCCL = 4,      /* NCCL error: ctx poisoned                                                    */
    SMPU_ENOMEM = 5,     /* device or pinned-host allocation failed (init only)                         */
    SMPU_EPOISONED = 6   /* an earlier call poisoned this ctx                                           */
} smpu_status;

typedef struct {
    double peak_lr;            /* 5e-4; 1e-3 = "2x lr"                                  */
    int64_t warmup_updates;    /* 4000                                                          */
    double beta1, beta2, eps;  /* 0.9, 0.98, 1e-8                                               */
    int32_t init_scale_log2;   /* 7: initial loss scale 2^7 (paper silent; reading R8)         */
    int32_t min_scale_log2;    /* -5 (R8): halving stops here                                            */
    int32_t max_scale_log2;    /* 24 (R8): growth stops here                                             */
    int64_t growth_interval;   /* 2000 clean updates before the scale doubles                   */
    int32_t update_freq;       /* c >= 1 micro-batches per update ("cumul")                      */
    int64_t bucket_bytes;      /* 150 MiB of fp16 gradient per all-reduce bucket (P:212 footnote, R22)  */
    int32_t allreduce;         /* world > 1 bucket all-reduce: SMPU_AR_AUTO (fused when every rank is an
                                  NVLink load/store peer, else NCCL), SMPU_AR_NCCL, SMPU_AR_FUSED          */
    int32_t sharded;           /* 0: the paper's replicated optimizer (every rank updates all of theta).
                                  1: sharded variant (world > 1, fused all-reduce): reduce-scatter,
                                  Adam on this rank's shard only, all-gather of w16.  theta/m/v are then valid
                                  only on smpu_shard_ranges; per element the arithmetic is unchanged.        */
    int32_t fuse_final;        /* world == 1 (ignored above).  0 (default): accumulate, decide, then Adam -- w16 changes
                                  only inside smpu_step (SURVEY 8(b)'s contract).  1 (opt-in): fuse the last
                                  micro-batch's accumulation into Adam -- one pass of 30 B/element instead of K1's
                                  6 + Adam's 28 (28 instead of 4 + 28 at c = 1).  The overflow decision needs all of R,
                                  so the update is computed speculatively into a second copy of theta/m/v (+12 B per
                                  parameter) that becomes current only if R was finite; w16 is then rewritten by the
                                  last micro-batch's accumulate call and re-cast on a skip.  Same arithmetic per
                                  element, bitwise (tested); R itself is never stored (SMPU_STATE_ACCUM).          */
    int32_t accum_fp32;        /* 0 (default, the north star's fp16 accumulation, reading Z1).  1: SURVEY Z1's knob --
                                  an fp32 accumulator (+4 B per parameter): A32 = fp32(g_1), A32 = fl32(A32 + g_k),
                                  and the last micro-batch writes the rank's fp16 gradient rn16(A32) into the fp16
                                  accumulator, from where everything is unchanged (fp16 all-reduce, overflow test,
                                  Adam).  K1 moves 10 instead of 6 B per element.  fuse_final is then ignored and
                                  accumulate_many runs one pass per micro-batch.                                    */
    int32_t split_tensors;     /* 0 (default): the paper's plan, whole tensors per bucket (R17).  1: fixed
                                  buckets of bucket_bytes (rounded up to 128 elements) cut wherever they fall, so a
                                  tensor may span buckets (smpu_tensor_ready then counts it in each).  Buckets
                                  change timing, never values.                                        */
    /* Shape of the fused all-reduce (world > 1, SMPU_AR_FUSED).  They decide the number of NCCL LSA barriers and
       whether the device communicator needs NVLS multicast -- collective resources -- so every rank must pass the
       same values: smpu_init compares them (and the fields above) across ranks and returns SMPU_EINVAL on EVERY rank
       when they differ, instead of hanging.  They never change results (the sum order is fixed), only speed.      */
    int32_t ar_ctas;           /* CTAs per rank of each bucket all-reduce; 0 (default) = one per SM                 */
    int32_t ar_threads;        /* threads per CTA: 256 (default) or 512                                             */
    int32_t ar_vec_bytes;      /* bytes per peer load / store: 32 (default, 256-bit) or 16                           */
    int32_t ar_unroll;         /* 32-byte units in flight per thread: 1 (default) or 2                               */
    int32_t ar_mcast;          /* 1: all-gather by NVLS multicast stores (multimem.st; EINVAL on every rank if some
                                  rank has no NVLS); 0 (default): unicast peer stores                                 */
    int32_t pdl;               /* world == 1: programmatic dependent launch of the K1 -> K0 -> K2 chain, 1 (default)
                                  or 0.  Per rank; no effect at world > 1.                                           */
    int32_t ar_pieces;         /* world > 1, replicated layout: all-reduce every bucket as this many consecutive
                                  pieces, Adam of each piece right behind its all-reduce, so that the Adam chain
                                  starts after the first piece rather than the first whole bucket and the two
                                  pipeline.  1 (default) = one launch per bucket; 1..64.  Collective: compared across
                                  ranks like the ar_* fields.                                                        */
    int32_t ar_copy_engine;    /* world > 1, fused all-reduce, replicated layout: 0 (default) = SM peer loads / stores
                                  (k_ar32); 1 = the NVLink traffic moved by the copy engines (one cudaMemcpyAsync per
                                  peer for the reduce-scatter push and the all-gather, an SM kernel only for the local
                                  ascending-rank fold), so a bucket in flight holds no SM while a backward or K1 runs;
                                  2 = the copy engines for every bucket but the last, which is ready only once the
                                  backward has ended and goes through the SM kernel (higher bandwidth).  Same bits.  The window grows by ~2 B per parameter of staging.  EINVAL with sharded,
                                  ar_mcast or SMPU_AR_NCCL.  Collective: compared across ranks.                       */
} smpu_config;

/* bucket all-reduce implementations (smpu_config.allreduce, smpu_allreduce_impl) */
enum {
    SMPU_AR_AUTO = 0,
    SMPU_AR_NCCL = 1,   /* ncclAllReduce(fp16, sum) per bucket: NCCL's order (R3: not bitwise-pinned for W > 2)  */
    SMPU_AR_FUSED = 2   /* deterministic reduce-scatter + all-gather kernel over NVLink peer memory (NCCL device
                           API symmetric window): ascending-rank fp16 sum, bitwise the oracle's for any W      */
};

typedef struct {
    int32_t overflow;          /* 1 iff the reduced fp16 gradient held a non-finite element     */
    int32_t applied;           /* 1 iff theta/m/v/w16 were updated (== !overflow unless discarded)       */
    int32_t scale_log2_used;   /* e of the scale 2^e the micro-gradients of this update carried         */
    int32_t scale_log2_next;   /* e after the scaler step: multiply the next losses by 2^this            */
    float lr;                  /* fp32 lr(t) applied; on a skip, lr(t+1) (reading R15)                   */
    int32_t discarded;         /* 1 iff global N was 0: nothing changed, the update is dropped (R19)     */
    int64_t num_updates;       /* t after this call: applied updates only (reading R7)                   */
    int64_t ntokens_total;     /* N: non-pad target tokens over all ranks and micro-batches       */
    int64_t clean_streak;      /* consecutive clean updates since the last scale change                   */
    int64_t attempt;           /* 1-based index of this update attempt (applied or not)                  */
} smpu_step_result;

/* which-selectors of smpu_get_state / smpu_set_state (checkpoint / resume, test access) */
enum {
    SMPU_STATE_MASTER = 0,     /* fp32[n] master weights theta                                           */
    SMPU_STATE_M = 1,          /* fp32[n] Adam first moment                                               */
    SMPU_STATE_V = 2,          /* fp32[n] Adam second moment                                              */
    SMPU_STATE_W16 = 3,        /* fp16[n] model weights (the re-cast copy)                                */
    SMPU_STATE_ACCUM = 4,      /* fp16[n] gradient accumulator: after step, the reduced gradient R (sharded: on
                                  this rank's shard ranges); with fuse_final = 1 at world 1 the sum of the
                                  first c - 1 micro-batches instead (untouched at c = 1), because R is then
                                  consumed without being stored                                           */
    SMPU_STATE_SCALARS = 5     /* int64[4] = {e, clean_streak, num_updates, attempts}                     */
};

/* kernel ids of smpu_kernel_stats */
enum { SMPU_K1_FIRST = 0, SMPU_K1_ADD = 1, SMPU_K1S = 2, SMPU_K0 = 3, SMPU_K2 = 4, SMPU_KCAST = 5,
       SMPU_ALLREDUCE = 6, SMPU_DECISION_AR = 7, SMPU_K1_MANY = 8, SMPU_K12 = 9 /* fused last micro + Adam */,
       SMPU_N_KERNELS = 10 };

/* flags of smpu_graph_capture */
enum { SMPU_GRAPH_STREAMING = 0, SMPU_GRAPH_RESIDENT = 1 };

int smpu_abi_version(void);

/* Fill *cfg with the paper's defaults (values in the comments of smpu_config). */
smpu_status smpu_config_default(smpu_config* cfg);

/* NCCL unique id for world > 1: call on rank 0 only, distribute the SMPU_NCCL_ID_BYTES bytes to every
 * rank out of band (the harness uses torch.distributed), pass to smpu_init.  `out` host, >= 128 B. */
smpu_status smpu_unique_id(void* out, int64_t bytes);

/* Host-only bucket plan (reading R17): walk the tensors in ready order, add whole tensors to
 * the current bucket and close it as soon as its fp16 bytes reach bucket_bytes; the remainder is the
 * last bucket.  bucket_begin (host, capacity n_tensors+1 entries, or NULL to query the count) receives
 * the element offset of each bucket plus the total n at [*n_buckets].  Needs no GPU. */
smpu_status smpu_plan_buckets(const int64_t* numel, int n_tensors, int64_t bucket_bytes, int* n_buckets,
                              int64_t* bucket_begin);

/* Host-only shard plan of the sharded layout: the element ranges whose theta/m/v rank `rank` of
 * `world` updates, for the buckets bucket_begin[0..n_buckets] (as smpu_plan_buckets / smpu_buckets give them):
 * per bucket, 8-element units from its first multiple of 8, ceil(units / world) consecutive units per rank, and
 * the bucket's unaligned head and tail to rank 0 -- the split the device reduce-scatter makes.  Same output
 * convention as smpu_shard_ranges (ranges host, capacity 2*cap; NULL to query).  Needs no GPU. */
smpu_status smpu_plan_shards(const int64_t* bucket_begin, int n_buckets, int world, int rank, int64_t* ranges,
                             int cap, int* count);

/* Create a ctx on CUDA device `cuda_device`.
 *   cfg          host; copied.
 *   world, rank  0 <= rank < world.  world > 1 needs nccl_id (host, 128 B, identical on every rank) and
 *                every rank calling smpu_init concurrently (collective).
 *   numel        host int64[n_tensors] > 0, gradient-ready order; copied.
 *   init_params  host or device fp32[n]: theta_0; copied.  Rank 0's copy is broadcast so all replicas
 *                start bitwise identical (P:55-57 synchronous data parallelism).
 * Allocates theta, m, v (fp32), w16, accumulator (fp16) on the device: 16 B per parameter (+12 for the
 * second theta/m/v of fuse_final at world 1). */
smpu_status smpu_init(smpu_ctx** out, const smpu_config* cfg, int world, int rank, const void* nccl_id,
                      int cuda_device, const int64_t* numel, int n_tensors, const float* init_params);

/* A VIRTUAL world: `world` (2..8) data-parallel ranks held on ONE GPU, for running and checking the world > 1 path
 * (bucketed all-reduce, exact early / late overflow decision, sharded optimizer)
 * without W GPUs.  Each member is a full ctx -- its own theta/m/v/w16/accumulator and scaler state, packed as for
 * smpu_init -- whose "window" is a plain device allocation; the peer kernels are the very kernels of the NCCL path
 * (lsa_allreduce.cuh), instantiated over local windows instead of NVLink peers: one launch covers every rank and
 * kernel boundaries replace the LSA barriers.  Sums are in ascending rank order, as with SMPU_AR_FUSED.
 *   cfg          host; copied.  allreduce must not be SMPU_AR_NCCL and ar_mcast must be 0 (EINVAL).
 *   numel, init_params   as smpu_init; every member starts from the same theta_0.
 * Members (smpu_group_member) take the smpu_* calls of a rank, driven from one host thread in any interleaving a
 * W-process job could produce, with two rules: every member gives its c micro-batches before any member calls
 * smpu_step (ESTATE otherwise), and a member that stepped starts its next update only after every member stepped
 * (ESTATE).  A collective step runs when the last member reaches it.  Sharded (cfg->sharded): the update of every
 * member completes when the last one steps, so smpu_step(out != NULL) is ESTATE before that -- pass NULL and read
 * smpu_result.  Not available on members: smpu_graph_capture, smpu_allreduce_accumulator (EINVAL).
 * smpu_destroy on a member is a no-op; smpu_group_destroy frees the group and its members. */
smpu_status smpu_group_init(smpu_group** out, const smpu_config* cfg, int world, int cuda_device, const int64_t* numel,
                            int n_tensors, const float* init_params);
smpu_status smpu_group_member(smpu_group* group, int rank, smpu_ctx** member);
void smpu_group_destroy(smpu_group* group);

smpu_status smpu_num_params(const smpu_ctx* ctx, int64_t* n);

/* Element ranges [ranges[2i], ranges[2i+1]) whose theta/m/v this rank updates (every element when not
 * sharded).  `ranges` host, capacity 2*cap int64 (NULL to query); *count receives the number of ranges. */
smpu_status smpu_shard_ranges(const smpu_ctx* ctx, int64_t* ranges, int cap, int* count);

/* Which bucket all-reduce this ctx runs (SMPU_AR_NCCL or SMPU_AR_FUSED; 0 at world == 1). */
smpu_status smpu_allreduce_impl(const smpu_ctx* ctx, int* impl);

/* Bucket boundaries chosen at init (same as smpu_plan_buckets with cfg->bucket_bytes unless split_tensors). */
smpu_status smpu_buckets(const smpu_ctx* ctx, int* n_buckets, int64_t* bucket_begin /* or NULL */);

/* Device fp16[n] weights (library-owned, valid until smpu_destroy).  Rewritten only by smpu_step, in stream order
 * on the stream passed to it.  Exception, opt-in: with fuse_final = 1 at world 1 they are already
 * rewritten by the last micro-batch's accumulate call (or each bucket's, in stream order on its stream: a bucket is
 * handed over once its gradients are done, so the backward no longer reads those weights); a skipped update
 * restores them in smpu_step.  Read them for the next forward after smpu_step. */
smpu_status smpu_weights_fp16(const smpu_ctx* ctx, const void** dev_w16);

/* Device fp32 scalar holding the current loss scale 2^e ("we scale the loss right after the forward
 * pass").  Updated in stream order by smpu_step; a producer multiplies its loss by it without a
 * host round trip. */
smpu_status smpu_loss_scale(const smpu_ctx* ctx, const float** dev_scale);

/* The fp16[n] accumulator itself (fp32[n] with accum_fp32; device, library-owned, valid until smpu_destroy),
 * for producers that add their weight gradients in place -- e.g. a cuBLAS dW GEMM with beta = 0 for the first
 * micro-batch of an update and beta = 1 after it -- and then declare the micro-batch with
 * micro_grads = NULL below.
 * The result is the producer's: cuBLAS's fp16 epilogue was measured to compute rn16(rn16(dW) + A), the same
 * two roundings as K1 (reading R1; tests/test_gpu_parity.py), but a GEMM that rounds once would differ. */
smpu_status smpu_accumulator(const smpu_ctx* ctx, void** dev_acc);

/* One whole micro-batch.  micro_grads: host or device fp16[n] (bit patterns), packed; device buffers
 * should be 32-byte aligned for the vector path (any 2-byte alignment is correct).  Gradients are those
 * of the SCALED token-SUM loss of the micro-batch (reading R11).  ntokens >= 0: its non-pad target
 * tokens.  Micro-batch 1 of an update copies, 2..c add in fp16 round-to-nearest-even (R1, R2).
 * On the last micro-batch with world > 1 each bucket's all-reduce starts as soon as that bucket is
 * accumulated.  ESTATE if c micro-batches were already given or a bucket-wise micro-batch is open. */
smpu_status smpu_accumulate(smpu_ctx* ctx, const void* micro_grads, int64_t ntokens, void* stream);

/* `count` whole micro-batches at once, for producers that keep several micro-batch gradients resident
 * (B200's 180 GB holds all 16 of Transformer-big, 6.7 GB): equivalent, bit for bit, to `count` consecutive
 * smpu_accumulate calls (same additions in the same order), in one pass that reads each gradient once
 * and the accumulator once -- 2 count + 2 (+4) bytes per element instead of 6 count (-2).  micro_grads[k]:
 * DEVICE fp16[n]; ntokens[k] >= 0; 1 <= count <= 32 and count <= micro-batches left in the update. */
smpu_status smpu_accumulate_many(smpu_ctx* ctx, const void* const* micro_grads, const int64_t* ntokens, int count,
                                 void* stream);

/* micro_grads == NULL (here and in smpu_accumulate_bucket): the producer already accumulated this micro-batch
 * (or bucket) into smpu_accumulator in place, stream-ordered before this call on `stream`; the library only
 * counts it and, on the last micro-batch, runs the overflow test / statistic and the bucket all-reduces. */

/* Per-tensor ready hook for in-place producers ("when the gradient computation for a layer
 * finishes, we add the result to a synchronization buffer"): after smpu_micro_begin, call it once per tensor
 * (gradient-ready index, as given to smpu_init) when that tensor's gradient is in smpu_accumulator; when the
 * last tensor of a bucket is in, the bucket is handed over exactly as smpu_accumulate_bucket(b, NULL).
 * ESTATE on a repeated tensor or a bucket already given whole. */
smpu_status smpu_tensor_ready(smpu_ctx* ctx, int tensor, void* stream);

/* Bucket-wise micro-batch, for overlap with a still-running backward: micro_begin, then
 * exactly one accumulate_bucket per bucket in any order (buckets are all-reduced in canonical bucket
 * order on every rank).  bucket_grads: host or device fp16 of bucket b only
 * (bucket_begin[b+1]-bucket_begin[b] elements).  ESTATE on a repeated bucket or a missing micro_begin. */
smpu_status smpu_micro_begin(smpu_ctx* ctx, int64_t ntokens);
smpu_status smpu_accumulate_bucket(smpu_ctx* ctx, int bucket, const void* bucket_grads, void* stream);

/* Finish the update: overflow decision, scaler, LR, fused unscale/normalise/Adam/re-cast, all on the
 * device in stream order on `stream` (no host synchronisation).  ESTATE unless exactly c micro-batches
 * (every bucket of the last one) were given.  out != NULL: wait for the update and fill *out
 * (returns ESTATE if N was 0: the update was discarded).  out == NULL: asynchronous; fetch the result
 * later with smpu_result. */
smpu_status smpu_step(smpu_ctx* ctx, void* stream, smpu_step_result* out);

/* CUDA-graph form of a whole update, for producers with fixed gradient buffers (CUDA graphs instead of a
 * tracing compiler): smpu_graph_capture records update_freq x smpu_accumulate over micro_grads[0..c) (DEVICE
 * buffers; their addresses are frozen, their contents are read at replay time) followed by smpu_step into a
 * graph owned by the ctx (replacing any earlier one); flags = SMPU_GRAPH_RESIDENT records one
 * smpu_accumulate_many over all c buffers instead (the producer keeps the c gradients until the replay).
 * It enqueues nothing.  With fuse_final = 0, update_freq = 1 and world = 1 the graph tests the buffer for
 * overflow in place and Adam reads it directly (the accumulator is then not written by the replays).  At
 * world > 1 it needs the fused all-reduce (EINVAL with SMPU_AR_NCCL).  smpu_graph_launch replays it on
 * `stream` with this update's token counts ntokens[0..c) (host): identical arithmetic and decisions to the
 * call-by-call path, one launch instead of c + 2 (or, at world > 1, the bucket all-reduces, decision and
 * per-bucket Adam as well); asynchronous, results via smpu_result.  Both ESTATE inside an update.  Launch
 * counts in smpu_kernel_stats are incremented per replay; per-kernel event timing does not see inside it. */
smpu_status smpu_graph_capture(smpu_ctx* ctx, const void* const* micro_grads, int count, int flags);
smpu_status smpu_graph_launch(smpu_ctx* ctx, const int64_t* ntokens, int count, void* stream);

/* The bucketed all-reduce alone (a collective primitive and a benchmark handle): sums the fp16 accumulator over
 * all ranks in place, bucket by bucket in canonical order, with this ctx's implementation (fused deterministic
 * or NCCL), stream-ordered on `stream`.  Collective; between updates only (ESTATE inside one); no-op at
 * world == 1; EINVAL on a sharded ctx. */
smpu_status smpu_allreduce_accumulator(smpu_ctx* ctx, void* stream);

/* Result of update attempt `attempt` (1-based; one of the last 64).  Waits for it. */
smpu_status smpu_result(smpu_ctx* ctx, int64_t attempt, smpu_step_result* out);

/* Copy theta (fp32[n]) to dst (host or device); synchronises the ctx's work first. */
smpu_status smpu_get_master(smpu_ctx* ctx, float* dst, int64_t n);

/* Read / write one state array (see SMPU_STATE_*); `bytes` must equal its size.  Synchronising.
 * Writing MASTER does not touch W16 (write both to resume).  Refused (ESTATE) mid-update. */
smpu_status smpu_get_state(smpu_ctx* ctx, int which, void* dst, int64_t bytes);
smpu_status smpu_set_state(smpu_ctx* ctx, int which, const void* src, int64_t bytes);

/* Per-kernel instrumentation (bench): enable=1 records CUDA events around every library launch on the
 * stream it is launched on.  smpu_kernel_stats returns, per kernel id, the launch count since init and
 * (when timing was on) the summed device time in ms; it synchronises. */
smpu_status smpu_set_timing(smpu_ctx* ctx, int enable);
smpu_status smpu_kernel_stats(smpu_ctx* ctx, int64_t* launches /* [SMPU_N_KERNELS] */,
                              double* total_ms /* [SMPU_N_KERNELS] or NULL */, int reset);

/* Ordered launch trace of the launches timed since the last smpu_kernel_stats reset (timing enabled): record
 * i has kernel id kind[i], stream[i] (0 = the caller's, 1 = bucket all-reduce, 2 = decision, 3 = per-bucket
 * Adam) and start/end in ms relative to the first record (CUDA events on the launching stream).  Arrays hold
 * `cap` records (any may be NULL); *count receives the total.  Synchronising.  The paper's Fig. 3 (overlap of
 * backward and synchronisation) is this trace with the producer's own events beside it. */
smpu_status smpu_kernel_trace(smpu_ctx* ctx, int32_t* kind, int32_t* stream, double* start_ms, double* end_ms,
                              int64_t cap, int64_t* count);

const char* smpu_last_error(void);
void smpu_destroy(smpu_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SMPU_H */
