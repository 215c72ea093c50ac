// sched.cpp -- host-side straggler / batching component (include/smpu_sched.h, PAPER.md 5).
#include "smpu_sched.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

std::vector<int64_t> length_sorted(const int32_t* src, const int32_t* tgt, int64_t n) {
    std::vector<int64_t> ids(n);
    std::iota(ids.begin(), ids.end(), 0);
    std::stable_sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) {
        int32_t ka = std::max(src[a], tgt[a]), kb = std::max(src[b], tgt[b]);
        if (ka != kb) return ka < kb;
        if (tgt[a] != tgt[b]) return tgt[a] < tgt[b];
        if (src[a] != src[b]) return src[a] < src[b];
        return a < b;
    });
    return ids;
}

double estimate(const double* coef, int64_t s, int32_t ls, int32_t lt) {
    return coef[0] * (double)s * ls + coef[1] * (double)s * lt + coef[2];
}

// `accept(s, ls, lt)`: may the sub-batch grow to s sentences with these max lengths?  With coef != nullptr the
// current sub-batch must also still be below `target` (time-balanced batching).
template <class Accept>
int group(const int32_t* src, const int32_t* tgt, int64_t n, Accept accept, int64_t* order, int64_t* batch_begin,
          int64_t cap, int64_t* n_batches, const double* coef = nullptr, double target = 0) {
    std::vector<int64_t> ids = length_sorted(src, tgt, n);
    std::vector<int64_t> begins{0};
    int64_t cnt = 0;
    int32_t ms = 0, mt = 0;
    for (int64_t k = 0; k < n; ++k) {
        int64_t id = ids[k];
        int32_t ns = std::max(ms, src[id]), nt = std::max(mt, tgt[id]);
        const bool below = !coef || estimate(coef, cnt, ms, mt) < target;
        if (cnt > 0 && (!below || !accept(cnt + 1, ns, nt))) {   // close the current sub-batch
            begins.push_back(k);
            cnt = 0;
            ns = src[id];
            nt = tgt[id];
        }
        ms = ns;
        mt = nt;
        ++cnt;
    }
    if (n > 0) begins.push_back(n);
    *n_batches = (int64_t)begins.size() - 1;
    if (*n_batches > cap) return 2;
    std::memcpy(order, ids.data(), sizeof(int64_t) * (size_t)n);
    std::memcpy(batch_begin, begins.data(), sizeof(int64_t) * begins.size());
    return 0;
}

// solve the k x k normal equations (k <= 3) by Gaussian elimination with partial pivoting
bool solve(std::vector<double> A, std::vector<double> b, int k, double* x) {
    for (int c = 0; c < k; ++c) {
        int p = c;
        for (int r = c + 1; r < k; ++r)
            if (std::fabs(A[r * k + c]) > std::fabs(A[p * k + c])) p = r;
        if (std::fabs(A[p * k + c]) < 1e-300) return false;
        for (int j = 0; j < k; ++j) std::swap(A[c * k + j], A[p * k + j]);
        std::swap(b[c], b[p]);
        for (int r = c + 1; r < k; ++r) {
            double f = A[r * k + c] / A[c * k + c];
            for (int j = c; j < k; ++j) A[r * k + j] -= f * A[c * k + j];
            b[r] -= f * b[c];
        }
    }
    for (int c = k - 1; c >= 0; --c) {
        double s = b[c];
        for (int j = c + 1; j < k; ++j) s -= A[c * k + j] * x[j];
        x[c] = s / A[c * k + c];
    }
    return true;
}

}  // namespace

extern "C" {

int smpu_sched_token_budget(const int32_t* src_len, const int32_t* tgt_len, int64_t n, int64_t max_tokens,
                            int64_t* order, int64_t* batch_begin, int64_t cap_batches, int64_t* n_batches) {
    if (n < 0 || !n_batches || (n > 0 && (!src_len || !tgt_len || !order || !batch_begin)) || max_tokens < 1)
        return 1;
    for (int64_t i = 0; i < n; ++i)
        if (src_len[i] < 1 || tgt_len[i] < 1 || std::max(src_len[i], tgt_len[i]) > max_tokens) return 1;
    return group(src_len, tgt_len, n,
                 [&](int64_t s, int32_t ls, int32_t lt) { return s * (int64_t)std::max(ls, lt) <= max_tokens; },
                 order, batch_begin, cap_batches, n_batches);
}

int smpu_sched_fit_timing(const int32_t* sentences, const int32_t* max_src, const int32_t* max_tgt,
                          const double* seconds, int64_t m, double* coef) {
    if (m < 1 || !sentences || !max_src || !max_tgt || !seconds || !coef) return 1;
    bool active[3] = {true, true, true};
    for (int round = 0; round < 3; ++round) {
        int idx[3], k = 0;
        for (int j = 0; j < 3; ++j)
            if (active[j]) idx[k++] = j;
        std::vector<double> A(k * k, 0.0), b(k, 0.0);
        for (int64_t i = 0; i < m; ++i) {
            double f[3] = {(double)sentences[i] * max_src[i], (double)sentences[i] * max_tgt[i], 1.0};
            for (int r = 0; r < k; ++r) {
                b[r] += f[idx[r]] * seconds[i];
                for (int c = 0; c < k; ++c) A[r * k + c] += f[idx[r]] * f[idx[c]];
            }
        }
        double x[3] = {0, 0, 0};
        if (!solve(A, b, k, x)) {
            // degenerate design (e.g. one measurement): fall back to the mean as the constant
            double mean = 0;
            for (int64_t i = 0; i < m; ++i) mean += seconds[i];
            coef[0] = coef[1] = 0;
            coef[2] = mean / (double)m;
            return 0;
        }
        double full[3] = {0, 0, 0};
        bool neg = false;
        for (int r = 0; r < k; ++r) {
            full[idx[r]] = x[r];
            if (x[r] < 0 && idx[r] < 2) {
                active[idx[r]] = false;
                neg = true;
            }
        }
        if (!neg) {
            std::memcpy(coef, full, sizeof full);
            return 0;
        }
    }
    return 1;
}

int smpu_sched_estimate(const int32_t* src_len, const int32_t* tgt_len, const int64_t* order,
                        const int64_t* batch_begin, int64_t n_batches, const double* coef, double* seconds) {
    if (n_batches < 0 || (n_batches > 0 && (!src_len || !tgt_len || !order || !batch_begin || !coef || !seconds)))
        return 1;
    for (int64_t b = 0; b < n_batches; ++b) {
        int32_t ms = 0, mt = 0;
        for (int64_t k = batch_begin[b]; k < batch_begin[b + 1]; ++k) {
            ms = std::max(ms, src_len[order[k]]);
            mt = std::max(mt, tgt_len[order[k]]);
        }
        seconds[b] = estimate(coef, batch_begin[b + 1] - batch_begin[b], ms, mt);
    }
    return 0;
}

int smpu_sched_time_balanced(const int32_t* src_len, const int32_t* tgt_len, int64_t n, const double* coef,
                             double target_seconds, int64_t* order, int64_t* batch_begin, int64_t cap_batches,
                             int64_t* n_batches) {
    if (n < 0 || !n_batches || !coef || !(target_seconds > 0) ||
        (n > 0 && (!src_len || !tgt_len || !order || !batch_begin)))
        return 1;
    for (int64_t i = 0; i < n; ++i)
        if (src_len[i] < 1 || tgt_len[i] < 1) return 1;
    // grow while the sub-batch is still below the target, allowing the last sentence to overshoot it by at
    // most 10% (the paper is silent on the boundary)
    return group(src_len, tgt_len, n,
                 [&](int64_t s, int32_t ls, int32_t lt) { return estimate(coef, s, ls, lt) <= 1.1 * target_seconds; },
                 order, batch_begin, cap_batches, n_batches, coef, target_seconds);
}

int smpu_sched_simulate(const double* batch_seconds, int64_t n_batches, int workers, int update_freq,
                        double* wall, double* idle_fraction, int64_t* steps) {
    if (workers < 1 || update_freq < 1 || n_batches < 0 || !wall || !idle_fraction || !steps ||
        (n_batches > 0 && !batch_seconds))
        return 1;
    const int64_t per_step = (int64_t)workers * update_freq;
    const int64_t S = n_batches / per_step;
    double w = 0, busy = 0, idle = 0;
    std::vector<double> comp(workers);
    for (int64_t s = 0; s < S; ++s) {
        double mx = 0;
        for (int r = 0; r < workers; ++r) {
            double t = 0;
            for (int j = 0; j < update_freq; ++j) t += batch_seconds[(s * workers + r) * update_freq + j];
            comp[r] = t;
            mx = std::max(mx, t);
        }
        for (int r = 0; r < workers; ++r) {
            busy += comp[r];
            idle += mx - comp[r];
        }
        w += mx;
    }
    *wall = w;
    *steps = S;
    *idle_fraction = busy + idle > 0 ? idle / (busy + idle) : 0.0;
    return 0;
}

int smpu_sched_overlap_schedule(const double* layer_bytes, const double* backward_seconds, int64_t n_layers,
                                double threshold_bytes, double latency_seconds, double bytes_per_second, int workers,
                                int64_t* bucket_last_layer, double* bucket_ready, double* bucket_start,
                                double* bucket_end, int64_t cap_buckets, int64_t* n_buckets, double* total_overlap,
                                double* total_serial) {
    if (n_layers < 0 || (n_layers > 0 && (!layer_bytes || !backward_seconds)) || !(threshold_bytes >= 0) ||
        !(latency_seconds >= 0) || !(bytes_per_second > 0) || workers < 1 || !n_buckets || !total_overlap ||
        !total_serial || cap_buckets < 0)
        return 1;
    for (int64_t i = 0; i < n_layers; ++i)
        if (!(layer_bytes[i] >= 0) || !(backward_seconds[i] >= 0)) return 1;
    // ring all-reduce cost of b bytes over `workers`; a flush of nothing costs nothing
    const double ring = workers > 1 ? 2.0 * (workers - 1) / workers : 0.0;
    auto cost = [&](double b) { return b > 0 ? latency_seconds + b / bytes_per_second * ring : 0.0; };
    int64_t nb = 0;
    double t = 0, buffered = 0, channel_free = 0, total_bytes = 0, backward = 0;
    bool pending = false;
    auto flush = [&](int64_t last_layer) {
        const double start = std::max(t, channel_free), end = start + cost(buffered);
        if (nb < cap_buckets) {
            if (bucket_last_layer) bucket_last_layer[nb] = last_layer;
            if (bucket_ready) bucket_ready[nb] = t;
            if (bucket_start) bucket_start[nb] = start;
            if (bucket_end) bucket_end[nb] = end;
        }
        channel_free = end;
        buffered = 0;
        pending = false;
        ++nb;
    };
    for (int64_t i = 0; i < n_layers; ++i) {
        t += backward_seconds[i];            // layer i's gradient is ready
        backward += backward_seconds[i];
        buffered += layer_bytes[i];
        total_bytes += layer_bytes[i];
        pending = true;
        if (buffered >= threshold_bytes) flush(i);   // threshold 0: every layer
    }
    if (pending) flush(n_layers - 1);        // the rest at the end of the backward
    *n_buckets = nb;
    *total_overlap = std::max(backward, channel_free);
    *total_serial = backward + cost(total_bytes);
    return nb > cap_buckets ? 2 : 0;
}

}  // extern "C"
