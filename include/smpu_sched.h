/*
 * smpu_sched.h -- C ABI of libsmpu_sched.so: the straggler / batching side of Ott et al. 2018,
 * host-only (no GPU), native C++.  PAPER.md section 5 "Analysis of Stragglers":
 *
 *   token-budget sub-batches   "each sub-batch has at most N tokens (e.g., N = 3.5k tokens), with padding
 *                              added as required"
 *   timing table               "we build a table to estimate the processing time for a sub-batch based on the
 *                              number of sentences and maximum source and target sentence lengths"
 *   time-balanced sub-batches  "we construct each worker's sub-batches by tuning the number of sentences until
 *                              the estimated processing time reaches our target", target e.g. the 90th
 *                              percentile
 *   idle-time simulation       "Slower workers, or stragglers, cause other workers to wait"; gradient
 *                              accumulation reduces the variance between workers (Fig. 2)
 *
 * Conventions: every pointer is host memory owned by the caller; arrays are written, never retained.  Return
 * 0 on success, 1 on invalid arguments (nothing written), 2 if an output array is too small (*count tells the
 * size needed).  Deterministic: ties in the length sort break by sentence id.
 */
#ifndef SMPU_SCHED_H
#define SMPU_SCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Token-budget sub-batches (SPEC S:265-272 reading of the padded area): sentences sorted by
 * (max(src, tgt), tgt, src, id), then grouped greedily so that
 * num_sentences x max(max_src_len, max_tgt_len) <= max_tokens.  order[n] receives the sentence ids in batch
 * order; batch_begin[*n_batches + 1] the offsets of each sub-batch in `order` (capacity cap_batches + 1). */
int smpu_sched_token_budget(const int32_t* src_len, const int32_t* tgt_len, int64_t n, int64_t max_tokens,
                            int64_t* order, int64_t* batch_begin, int64_t cap_batches, int64_t* n_batches);

/* Least-squares fit of the timing model t = a * S * Ls + b * S * Lt + c (S sentences, Ls / Lt max lengths) to
 * m measured sub-batches; coef[3] = {a, b, c}.  A negative coefficient is clamped to 0 and the others refit
 * (monotone estimates). */
int smpu_sched_fit_timing(const int32_t* sentences, const int32_t* max_src, const int32_t* max_tgt,
                          const double* seconds, int64_t m, double* coef);

/* Estimated seconds of each sub-batch of a batching (order / batch_begin as above) under coef. */
int smpu_sched_estimate(const int32_t* src_len, const int32_t* tgt_len, const int64_t* order,
                        const int64_t* batch_begin, int64_t n_batches, const double* coef, double* seconds);

/* Time-balanced sub-batches: over the same length-sorted order, add the next sentence while the
 * current sub-batch's estimate is below target_seconds and the grown one stays within 1.1 x target (the last
 * sentence may overshoot by at most 10%; the paper is silent).  A sentence alone above the target
 * stays a singleton. */
int smpu_sched_time_balanced(const int32_t* src_len, const int32_t* tgt_len, int64_t n, const double* coef,
                             double target_seconds, int64_t* order, int64_t* batch_begin, int64_t cap_batches,
                             int64_t* n_batches);

/* Synchronous data-parallel idle time: sub-batch k of update step s on worker w is
 * (s * W + w) * c + j, j < c (round robin); a worker's compute = the sum of its c sub-batch times; every step
 * waits for the slowest worker.  Uses the first floor(n / (W c)) * W c sub-batches.  Outputs: *wall = sum of
 * per-step maxima, *idle_fraction = sum(idle) / sum(compute + idle), *steps. */
int smpu_sched_simulate(const double* batch_seconds, int64_t n_batches, int workers, int update_freq,
                        double* wall, double* idle_fraction, int64_t* steps);

/* The paper's overlap of the bucketed all-reduce with the backward ("we add the result to a
 * synchronization buffer.  As soon as the size of the buffer reaches a predefined threshold we synchronize the
 * buffered gradients in a background thread"), as SPEC's analytic schedule: layers arrive in backward
 * (reverse) order, layer i ready at the sum of backward_seconds[0..i]; the buffer is flushed once it holds
 * >= threshold_bytes (threshold 0: every layer) and whatever is left at the end of the backward; flushes run FIFO on
 * one channel, a flush of b bytes costing latency + b / bytes_per_second x 2 (W-1) / W (W = workers;
 * W = 1 costs nothing).  Per flush k: the last layer in it, ready time, start and end on the channel (arrays of
 * cap_buckets, may be NULL).  *total_overlap = the later of the backward's end and the last flush's end;
 * *total_serial = the backward + one flush of all bytes after it.  Returns 2 if more than cap_buckets flushes
 * (*n_buckets then tells how many). */
int smpu_sched_overlap_schedule(const double* layer_bytes, const double* backward_seconds, int64_t n_layers,
                                double threshold_bytes, double latency_seconds, double bytes_per_second, int workers,
                                int64_t* bucket_last_layer, double* bucket_ready, double* bucket_start,
                                double* bucket_end, int64_t cap_buckets, int64_t* n_buckets, double* total_overlap,
                                double* total_serial);

#ifdef __cplusplus
}
#endif
#endif /* SMPU_SCHED_H */
