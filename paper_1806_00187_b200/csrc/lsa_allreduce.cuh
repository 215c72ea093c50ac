// lsa_allreduce.cuh -- deterministic fused bucket all-reduce over NVLink peer memory.
//
// The accumulator is one NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister), so every rank's
// accumulator is load/store-accessible from every GPU of the NVLink domain ("LSA" peers, NCCL device API).
// For bucket [lo, hi) rank r owns shard r (1/W of the bucket).  After a cross-GPU barrier (the last K1 of the
// bucket has finished on every rank), rank r reads A_0 .. A_{W-1} of its shard from all ranks, sums them in
// ascending rank order with a round-to-nearest-even fp16 add after each term -- the oracle's order, reading
// R3, so R is bitwise the oracle's for ANY values, not only exactly-summable ones -- and stores R into the
// shard of every rank's accumulator (the all-gather).  A second barrier publishes the stores.
//
// Bus bytes per rank are those of a ring all-reduce, 2 (W-1)/W x 2 B per element (reads of peer shards in,
// peer stores out); HBM: the local shard read once, every element of the local accumulator written once.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "kernels.cuh"

namespace smpu {

constexpr int kMaxLsaRanks = 8;

__device__ __forceinline__ V4 ld128_peer(const void* p) {
    V4 r;
    asm volatile("ld.global.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ void st128_peer(void* p, const V4& v) {
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
                 "r"(v.w[3])
                 : "memory");
}

__device__ __forceinline__ V8 ld256_peer(const void* p) {
    V8 r;
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                   "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ void st256_peer(void* p, const V8& v) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
                 "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

// one CTA-wide barrier across the same CTA index of every rank (acquire + release at system scope)
__device__ __forceinline__ void lsa_sync(const ncclDevComm& dc) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

template <int W>
__global__ void __launch_bounds__(256) k_ar_lsa(ncclDevComm dc, ncclWindow_t win, int64_t lo, int64_t hi) {
    lsa_sync(dc);   // every rank's last K1 of this bucket is complete and visible
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)ncclGetLsaPointer(win, 0, p);
    const int me = dc.lsaRank;
    // shard boundaries on 8-element (16 B) units inside the bucket; shard `me` = [s_lo, s_hi)
    const int64_t v0 = (lo + 7) & ~(int64_t)7, v1 = hi & ~(int64_t)7;
    const int64_t units = v1 > v0 ? (v1 - v0) / 8 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t u = u_lo + tid;
    for (; u + nthr < u_hi; u += 2 * nthr) {
        const int64_t i0 = v0 + u * 8, i1 = v0 + (u + nthr) * 8;
        V4 a[W], b[W];
#pragma unroll
        for (int p = 0; p < W; ++p) {
            a[p] = ld128_peer(base[p] + i0);
            b[p] = ld128_peer(base[p] + i1);
        }
#pragma unroll
        for (int p = 1; p < W; ++p)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                a[0].w[j] = hadd2_rn(a[0].w[j], a[p].w[j]);
                b[0].w[j] = hadd2_rn(b[0].w[j], b[p].w[j]);
            }
#pragma unroll
        for (int p = 0; p < W; ++p) {
            st128_peer(base[p] + i0, a[0]);
            st128_peer(base[p] + i1, b[0]);
        }
    }
    if (u < u_hi) {
        const int64_t i0 = v0 + u * 8;
        V4 a[W];
#pragma unroll
        for (int p = 0; p < W; ++p) a[p] = ld128_peer(base[p] + i0);
#pragma unroll
        for (int p = 1; p < W; ++p)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[0].w[j] = hadd2_rn(a[0].w[j], a[p].w[j]);
#pragma unroll
        for (int p = 0; p < W; ++p) st128_peer(base[p] + i0, a[0]);
    }
    // unaligned head [lo, v0) and tail [v1, hi) of the bucket: rank 0 does them element by element
    if (me == 0) {
        auto elem = [&](int64_t i) {
            uint32_t x = base[0][i];
#pragma unroll
            for (int p = 1; p < W; ++p) x = hadd2_rn(x, (uint32_t)base[p][i]) & 0xFFFFu;
#pragma unroll
            for (int p = 0; p < W; ++p) base[p][i] = (uint16_t)x;
        };
        const int64_t head_end = v0 < hi ? v0 : hi;
        for (int64_t i = lo + tid; i < head_end; i += nthr) elem(i);
        for (int64_t i = (v1 > head_end ? v1 : head_end) + tid; i < hi; i += nthr) elem(i);
    }
    lsa_sync(dc);   // every shard of every rank has been written
}

// Multicast store of 32 bytes through NVSwitch (NVLS): one store reaches the same offset of every rank's window.
// (multimem.st moves at most 128 bits: two stores)
__device__ __forceinline__ void st256_multicast(void* mc, const V8& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.w[0]), "r"(v.w[1]),
                 "r"(v.w[2]), "r"(v.w[3])
                 : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"((char*)mc + 16), "r"(v.w[4]),
                 "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

// Variant with 32-byte units (256-bit peer loads/stores), one unit per thread per iteration: fewer, wider NVLink
// transactions.  Shards are split on 16-element units; head/tail on rank 0 as above.
// MC: the all-gather is one multicast store per unit instead of W peer stores (same bits: the sum is computed
// once, by the shard's owner, in ascending rank order, as before).
template <int W, bool MC = false, int U = 1>
__global__ void __launch_bounds__(512) k_ar_lsa32(ncclDevComm dc, ncclWindow_t win, int64_t lo, int64_t hi) {
    lsa_sync(dc);
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)ncclGetLsaPointer(win, 0, p);
    uint16_t* mc = MC ? (uint16_t*)ncclGetLsaMultimemPointer(win, 0, dc) : nullptr;
    const int me = dc.lsaRank;
    const int64_t v0 = (lo + 15) & ~(int64_t)15, v1 = hi & ~(int64_t)15;
    const int64_t units = v1 > v0 ? (v1 - v0) / 16 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = u_lo + tid; u < u_hi; u += U * nthr) {
        V8 a[U][W];
#pragma unroll
        for (int q = 0; q < U; ++q)
            if (u + q * nthr < u_hi) {
#pragma unroll
                for (int p = 0; p < W; ++p) a[q][p] = ld256_peer(base[p] + v0 + (u + q * nthr) * 16);
            }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            if (u + q * nthr >= u_hi) break;
            const int64_t i0 = v0 + (u + q * nthr) * 16;
#pragma unroll
            for (int p = 1; p < W; ++p)
#pragma unroll
                for (int j = 0; j < 8; ++j) a[q][0].w[j] = hadd2_rn(a[q][0].w[j], a[q][p].w[j]);
            if (MC) {
                st256_multicast(mc + i0, a[q][0]);
            } else {
#pragma unroll
                for (int p = 0; p < W; ++p) st256_peer(base[p] + i0, a[q][0]);
            }
        }
    }
    if (me == 0) {
        auto elem = [&](int64_t i) {
            uint32_t x = base[0][i];
#pragma unroll
            for (int p = 1; p < W; ++p) x = hadd2_rn(x, (uint32_t)base[p][i]) & 0xFFFFu;
#pragma unroll
            for (int p = 0; p < W; ++p) base[p][i] = (uint16_t)x;
        };
        const int64_t head_end = v0 < hi ? v0 : hi;
        for (int64_t i = lo + tid; i < head_end; i += nthr) elem(i);
        for (int64_t i = (v1 > head_end ? v1 : head_end) + tid; i < hi; i += nthr) elem(i);
    }
    lsa_sync(dc);
}

// The early overflow decision of K0 EARLY with the 16-byte exchange done in peer memory instead of an NCCL
// all-reduce (one kernel instead of prep + NCCL + K0, ~10 us instead of ~130 us): every rank stores
// {N_r, M_r} into slot r of every rank's decision area (double-buffered by update parity, so a fast peer's
// next update cannot overwrite slots not yet read), one LSA barrier, then each rank sums the W slots in rank
// order -- identical inputs and order on every rank, hence identical decisions -- and decides.
template <int W>
__global__ void k0_early_lsa(ncclDevComm dc, ncclWindow_t win, size_t area_off, uint32_t* stat,
                             int64_t local_tokens, const int64_t* tok_ptr, int64_t* xs, DevState* st, Scalars* sc,
                             float* loss_scale, smpu_step_result* ring, int ring_mask, DevCfg cfg,
                             uint32_t barrier_index) {
    const int me = dc.lsaRank;
    if (tok_ptr) local_tokens = *tok_ptr;
    const int parity = (int)(((volatile const DevState*)st)->attempts & 1);   // same on every rank; graph-safe
    const size_t slot_off = area_off + ((size_t)parity * W + me) * 16;
    if (threadIdx.x == 0) {
        int64_t mine[2] = {local_tokens, mag_units(*stat)};
        *stat = 0;                                     // re-armed for the next update
#pragma unroll
        for (int p = 0; p < W; ++p) {
            int64_t* dst = (int64_t*)ncclGetLsaPointer(win, slot_off, p);
            dst[0] = mine[0];
            dst[1] = mine[1];
        }
    }
    {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), barrier_index);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
    if (threadIdx.x == 0) {
        const int64_t* area = (const int64_t*)ncclGetLocalPointer(win, area_off + (size_t)parity * W * 16);
        int64_t N = 0, M = 0;
        for (int p = 0; p < W; ++p) {
            N += ((volatile const int64_t*)area)[2 * p];
            M += ((volatile const int64_t*)area)[2 * p + 1];
        }
        xs[0] = N;
        xs[1] = M;
        if (M >= kNonFinite) decide(1, N, st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY);
        else if (M <= (int64_t(1) << 39)) decide(0, N, st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY);
        else sc->state = DEC_UNDECIDED;
    }
}

}  // namespace smpu

namespace smpu {

// ============================================================================ sharded optimizer
// An adjacent variant of the paper's replicated update, opt-in (smpu_config.sharded): the bucket all-reduce
// becomes a reduce-scatter (R of my shard only, same ascending-rank order), Adam runs on my shard only and
// all-gathers the fp16 weights by storing w16 of the shard into every rank's window.  Per element the
// arithmetic is exactly the replicated path's, so theta/m/v of a shard and the full w16 are bitwise those of
// the replicated update; HBM per rank for the optimizer drops from 28 to ~28/W + 2 bytes per element.

// Reduce-scatter of one bucket: like k_ar_lsa, but R is stored into my own window only.  No closing barrier:
// the end-of-update barrier (k_lsa_barrier) orders every rank's reads of my accumulator before anybody's next
// update overwrites it.
template <int W>
__global__ void __launch_bounds__(256) k_rs_lsa(ncclDevComm dc, ncclWindow_t win, int64_t lo, int64_t hi) {
    lsa_sync(dc);
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)ncclGetLsaPointer(win, 0, p);
    const int me = dc.lsaRank;
    const int64_t v0 = (lo + 7) & ~(int64_t)7, v1 = hi & ~(int64_t)7;
    const int64_t units = v1 > v0 ? (v1 - v0) / 8 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = u_lo + tid; u < u_hi; u += nthr) {
        const int64_t i0 = v0 + u * 8;
        V4 a[W];
#pragma unroll
        for (int p = 0; p < W; ++p) a[p] = ld128_peer(base[p] + i0);
#pragma unroll
        for (int p = 1; p < W; ++p)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[0].w[j] = hadd2_rn(a[0].w[j], a[p].w[j]);
        st128_peer(base[me] + i0, a[0]);
    }
    if (me == 0) {
        auto elem = [&](int64_t i) {
            uint32_t x = base[0][i];
#pragma unroll
            for (int p = 1; p < W; ++p) x = hadd2_rn(x, (uint32_t)base[p][i]) & 0xFFFFu;
            base[0][i] = (uint16_t)x;
        };
        const int64_t head_end = v0 < hi ? v0 : hi;
        for (int64_t i = lo + tid; i < head_end; i += nthr) elem(i);
        for (int64_t i = (v1 > head_end ? v1 : head_end) + tid; i < hi; i += nthr) elem(i);
    }
}

// Adam on [lo, hi) of my shard (one-shot), w16 stored into every rank's window at window offset w16_off.
template <int W>
__global__ void __launch_bounds__(256, 4) k2_adam_shard(ncclWindow_t win, size_t w16_off, float* __restrict__ theta,
                                                        float* __restrict__ m, float* __restrict__ v,
                                                        const uint16_t* __restrict__ R, int64_t lo, int64_t hi,
                                                        const Scalars* __restrict__ scp, int32_t need) {
    if (decision_of(scp) != need) return;
    const Scalars s = *scp;
    uint16_t* wb[W];
#pragma unroll
    for (int p = 0; p < W; ++p) wb[p] = (uint16_t*)ncclGetLsaPointer(win, w16_off, p);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 7) & ~(int64_t)7;
    if (vbeg > hi) vbeg = hi;
    const int64_t nvec = (hi - vbeg) / 8, vend = vbeg + nvec * 8;
    for (int64_t u = tid; u < nvec; u += nthr) {
        const int64_t i0 = vbeg + u * 8;
        V4 r0 = ld128_ro(R + i0);
        V8 t0 = ld256(theta + i0), m0 = ld256(m + i0), v0 = ld256(v + i0);
        V4 w0;
        adam_unit(r0, t0, m0, v0, w0, s);
        st256(theta + i0, t0);
        st256(m + i0, m0);
        st256(v + i0, v0);
#pragma unroll
        for (int p = 0; p < W; ++p) st128_peer(wb[p] + i0, w0);
    }
    auto elem = [&](int64_t i) {
        float th = theta[i], mm = m[i], vv = v[i];
        adam_elem(__half2float(__ushort_as_half(R[i])), th, mm, vv, s);
        theta[i] = th;
        m[i] = mm;
        v[i] = vv;
        uint16_t w = __half_as_ushort(__float2half_rn(th));
#pragma unroll
        for (int p = 0; p < W; ++p) wb[p][i] = w;
    };
    for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
    for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
}

// One cross-rank barrier (acquire + release, system scope) at barrier index `idx`.
__global__ void k_lsa_barrier(ncclDevComm dc, uint32_t idx) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), idx);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// Late decision of the sharded path (only when K0 EARLY was undecided, identically on every rank): each rank
// swept its own shard of R; the flags are OR-ed through peer memory, then decided as K0 LATE.
template <int W>
__global__ void k0_late_lsa(ncclDevComm dc, ncclWindow_t win, size_t area_off, int* flag, const int64_t* xs,
                            DevState* st, Scalars* sc, float* loss_scale, smpu_step_result* ring, int ring_mask,
                            DevCfg cfg, uint32_t barrier_index) {
    if (decision_of(sc) != DEC_UNDECIDED) {
        if (threadIdx.x == 0) *(volatile int*)flag = 0;
        return;
    }
    const int me = dc.lsaRank;
    const int parity = (int)(((volatile const DevState*)st)->attempts & 1);
    area_off += 2 * kMaxLsaRanks * 16;                 // slots of their own: the early exchange may still be read
    const size_t slot_off = area_off + ((size_t)parity * W + me) * 16;
    if (threadIdx.x == 0) {
        const int64_t mine = *(volatile int*)flag != 0;
        for (int p = 0; p < W; ++p) *(int64_t*)ncclGetLsaPointer(win, slot_off, p) = mine;
    }
    {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), barrier_index);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
    if (threadIdx.x == 0) {
        const int64_t* area = (const int64_t*)ncclGetLocalPointer(win, area_off + (size_t)parity * W * 16);
        int64_t any = 0;
        for (int p = 0; p < W; ++p) any |= ((volatile const int64_t*)area)[2 * p];
        decide(any != 0, xs[0], st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY_LATE);
        *(volatile int*)flag = 0;
    }
}

}  // namespace smpu
