// lsa_allreduce.cuh -- deterministic fused bucket all-reduce over peer memory, the exact early
// overflow decision exchange, and the sharded optimizer's peer kernels (f2).
//
// Every kernel here is written once, templated on the world size W and on a PEERS policy that says where rank p's
// window lives and how ranks meet:
//
//   LsaPeers    W processes, one GPU each (the product at world > 1).  The accumulator is one NCCL symmetric window
//               (ncclMemAlloc + ncclCommWindowRegister), so every rank's accumulator is load/store-accessible from
//               every GPU of the NVLink domain ("LSA" peers, NCCL device API); ranks meet at NCCL LSA barriers
//               inside the kernel.  One launch per rank.
//   LocalPeers  W virtual ranks held as W windows (plain cudaMalloc) on ONE GPU (smpu_group_init): the same kernel
//               bodies, with rank p's window at base[p].  A single launch covers every rank -- CTAs
//               [r*per_rank, (r+1)*per_rank) act for rank r -- and the ranks meet at kernel boundaries instead of
//               barriers (a phase that needs every rank's stores is a second launch).  This lets the W > 1
//               arithmetic, at any W up to 8, run and be checked against the oracle on a one-GPU box.
//
// All-reduce of bucket [lo, hi): rank r owns shard r (1/W of the bucket).  After every rank's last K1 of the bucket
// has finished, rank r reads A_0 .. A_{W-1} of its shard from all windows, sums them in ascending rank order with a
// round-to-nearest-even fp16 add after each term -- the oracle's order, reading R3, so R is bitwise the oracle's for
// ANY values, not only exactly-summable ones -- and stores R into the shard of every window (the all-gather).
// Shards are disjoint, so one launch over all virtual ranks is race-free.
//
// Bus bytes per rank are those of a ring all-reduce, 2 (W-1)/W x 2 B per element (reads of peer shards in, peer
// stores out); HBM: the local shard read once, every element of the local accumulator written once.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "kernels.cuh"

namespace smpu {

constexpr int kMaxLsaRanks = 8;

// ------------------------------------------------------------------------------------------------ peer policies
struct LsaPeers {
    ncclDevComm dc;
    ncclWindow_t win;
    __device__ __forceinline__ int rank() const { return dc.lsaRank; }
    __device__ __forceinline__ int cta() const { return (int)blockIdx.x; }
    __device__ __forceinline__ int ctas() const { return (int)gridDim.x; }
    __device__ __forceinline__ char* at(int p, size_t off) const { return (char*)ncclGetLsaPointer(win, off, p); }
    __device__ __forceinline__ char* multicast(size_t off) const {
        return (char*)ncclGetLsaMultimemPointer(win, off, dc);
    }
    // one CTA-wide barrier across barrier `idx` of every rank (acquire + release at system scope)
    __device__ __forceinline__ void sync(uint32_t idx) const {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), idx);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
};

struct LocalPeers {
    char* base[kMaxLsaRanks];   // window of virtual rank p
    int per_rank;               // > 0: one launch for every rank, per_rank CTAs each; 0: a launch for rank `fixed`
    int fixed;
    __device__ __forceinline__ int rank() const { return per_rank ? (int)blockIdx.x / per_rank : fixed; }
    __device__ __forceinline__ int cta() const { return per_rank ? (int)blockIdx.x % per_rank : (int)blockIdx.x; }
    __device__ __forceinline__ int ctas() const { return per_rank ? per_rank : (int)gridDim.x; }
    __device__ __forceinline__ char* at(int p, size_t off) const { return base[p] + off; }
    __device__ __forceinline__ void sync(uint32_t) const {}   // the launch boundary is the barrier
};

// ------------------------------------------------------------------------------------------------ peer accesses
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

// Unaligned head [lo, v0) and tail [v1, hi) of a bucket: rank 0 sums them element by element, same order, and
// stores R into every window (ALL_GATHER) or its own only (reduce-scatter).
template <int W, bool ALL_GATHER>
__device__ __forceinline__ void head_tail(uint16_t* const* base, int64_t lo, int64_t hi, int64_t v0, int64_t v1,
                                          int64_t tid, int64_t nthr) {
    auto elem = [&](int64_t i) {
        uint32_t x = base[0][i];
#pragma unroll
        for (int p = 1; p < W; ++p) x = hadd2_rn(x, (uint32_t)base[p][i]) & 0xFFFFu;
        if (ALL_GATHER) {
#pragma unroll
            for (int p = 0; p < W; ++p) base[p][i] = (uint16_t)x;
        } else {
            base[0][i] = (uint16_t)x;
        }
    };
    const int64_t head_end = v0 < hi ? v0 : hi;
    for (int64_t i = lo + tid; i < head_end; i += nthr) elem(i);
    for (int64_t i = (v1 > head_end ? v1 : head_end) + tid; i < hi; i += nthr) elem(i);
}

// 16-byte units (smpu_config.ar_vec_bytes = 16), two per thread in flight.
template <int W, class Peers>
__global__ void __launch_bounds__(256) k_ar16(Peers pe, int64_t lo, int64_t hi) {
    pe.sync(pe.cta());   // every rank's last K1 of this bucket is complete and visible
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)pe.at(p, 0);
    const int me = pe.rank();
    // shard boundaries on 8-element (16 B) units inside the bucket; shard `me` = [s_lo, s_hi)
    const int64_t v0 = (lo + 7) & ~(int64_t)7, v1 = hi & ~(int64_t)7;
    const int64_t units = v1 > v0 ? (v1 - v0) / 8 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const int64_t tid = (int64_t)pe.cta() * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)pe.ctas() * blockDim.x;
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
    if (me == 0) head_tail<W, true>(base, lo, hi, v0, v1, tid, nthr);
    pe.sync(pe.cta());   // every shard of every rank has been written
}

// 32-byte units (256-bit peer loads/stores, the default), U units per thread per iteration: fewer, wider NVLink
// transactions.  Shards are split on 16-element units; head/tail on rank 0 as above.
// MC (LsaPeers only): the all-gather is one multicast store per unit instead of W peer stores (same bits: the sum is
// computed once, by the shard's owner, in ascending rank order, as before).
template <int W, class Peers, bool MC = false, int U = 1>
__global__ void __launch_bounds__(512) k_ar32(Peers pe, int64_t lo, int64_t hi) {
    pe.sync(pe.cta());
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)pe.at(p, 0);
    uint16_t* mc = nullptr;
    if constexpr (MC) mc = (uint16_t*)pe.multicast(0);
    const int me = pe.rank();
    const int64_t v0 = (lo + 15) & ~(int64_t)15, v1 = hi & ~(int64_t)15;
    const int64_t units = v1 > v0 ? (v1 - v0) / 16 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const int64_t tid = (int64_t)pe.cta() * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)pe.ctas() * blockDim.x;
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
            if constexpr (MC) {
                st256_multicast(mc + i0, a[q][0]);
            } else {
#pragma unroll
                for (int p = 0; p < W; ++p) st256_peer(base[p] + i0, a[q][0]);
            }
        }
    }
    if (me == 0) head_tail<W, true>(base, lo, hi, v0, v1, tid, nthr);
    pe.sync(pe.cta());
}

// ------------------------------------------------------------------- copy-engine variant (smpu_config.ar_copy_engine)
// The same reduce-scatter + all-gather with the NVLink traffic moved by the copy engines instead of SM loads and
// stores, so the bucket all-reduce holds no SM while the data crosses the fabric (a running backward or K1 keeps
// every SM).  Shards as in k_ar32 (16-element units, ceil(units / W) per rank).  Per bucket, on rank r:
//   1. push: one cudaMemcpyAsync per peer p of r's contribution to shard p into p's staging slot r (window offset
//      stage_off + r * per * 32 B), issued from r's copy streams (NVLink writes);
//   2. k_ce_barrier: every rank's pushes of this bucket have completed (a stream runs the barrier kernel only after
//      its copies are done);
//   3. k_ce_reduce: R of shard r = the ascending-rank fold of the W contributions (slot s, or r's own accumulator
//      for s = r) with an rn16 add after each term -- the order of k_ar32 and of the oracle (reading R3) -- stored
//      into r's accumulator; rank 0 also does the unaligned head / tail over peer memory as k_ar32 does;
//   4. all-gather: one cudaMemcpyAsync per peer of R's shard r into p's accumulator;
//   5. k_ce_barrier: every rank's all-gather has landed before anything reads the accumulator.
// Bits are identical to k_ar32's (same fold, same order).  LocalPeers (virtual ranks): the same copies between the
// local windows, one k_ce_reduce launch for every rank, and stream order instead of the two barriers.
template <class Peers>
__global__ void k_ce_barrier(Peers pe, uint32_t idx) {
    pe.sync(idx);
}

template <class Peers>
__global__ void k_peer_ptrs(Peers pe, int W, unsigned long long* out) {
    if ((int)threadIdx.x < W) out[threadIdx.x] = (unsigned long long)(uintptr_t)pe.at((int)threadIdx.x, 0);
}

template <int W, class Peers>
__global__ void __launch_bounds__(256) k_ce_reduce(Peers pe, int64_t lo, int64_t hi, size_t stage_off) {
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)pe.at(p, 0);
    const int me = pe.rank();
    const int64_t v0 = (lo + 15) & ~(int64_t)15, v1 = hi & ~(int64_t)15;
    const int64_t units = v1 > v0 ? (v1 - v0) / 16 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const uint16_t* stage = (const uint16_t*)pe.at(me, stage_off);   // slot s at stage + s * per * 16
    uint16_t* acc = base[me];
    const int64_t tid = (int64_t)pe.cta() * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)pe.ctas() * blockDim.x;
    for (int64_t u = u_lo + tid; u < u_hi; u += nthr) {
        const int64_t i0 = v0 + u * 16, j0 = (u - u_lo) * 16;
        V8 a[W];
#pragma unroll
        for (int s = 0; s < W; ++s) a[s] = s == me ? ld256(acc + i0) : ld256_ro(stage + s * per * 16 + j0);
#pragma unroll
        for (int s = 1; s < W; ++s)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[0].w[j] = hadd2_rn(a[0].w[j], a[s].w[j]);
        st256(acc + i0, a[0]);
    }
    if (me == 0) head_tail<W, true>(base, lo, hi, v0, v1, tid, nthr);
}

// --------------------------------------------------------------------------------------- decision exchange
// Per-rank arguments of the decision kernels.  An LsaPeers launch fills r[its rank]; a LocalPeers launch fills
// every virtual rank's (the kernel indexes r[pe.rank()]).
struct DecArgs {
    uint32_t* stat;            // max fp16 magnitude bits of this rank's last-micro-batch output (K1 STATS)
    int64_t local_tokens;      // N_r (host value), unless tok_ptr (graph replays) holds it
    const int64_t* tok_ptr;
    int64_t* xs;               // {N, sum_r M_r} after the exchange
    int* flag;                 // K1s sweep flag (late decision)
    DevState* st;
    Scalars* sc;
    float* loss_scale;
    smpu_step_result* ring;
};
struct DecArgsW {
    DecArgs r[kMaxLsaRanks];
};

// PHASE bits: 1 = publish this rank's slot into every window, 2 = read my window's slots and decide; LsaPeers runs
// both (3) around an LSA barrier, LocalPeers runs phase 1 for every rank, then phase 2 for every rank.
constexpr int kPublish = 1, kDecide = 2, kBoth = 3;

// The early overflow decision (K0 EARLY) with the 16-byte exchange done in peer memory instead of an NCCL
// all-reduce (one kernel instead of prep + NCCL + K0, ~10 us instead of ~130 us): every rank stores
// {N_r, M_r} into slot r of every rank's decision area (double-buffered by update parity, so a fast peer's
// next update cannot overwrite slots not yet read), one barrier, then each rank sums the W slots in rank
// order -- identical inputs and order on every rank, hence identical decisions -- and decides (k0_early's rule).
template <int W, class Peers, int PHASE>
__global__ void k0_early_x(Peers pe, size_t area_off, DecArgsW A, int ring_mask, DevCfg cfg, uint32_t barrier_index) {
    const int me = pe.rank();
    const DecArgs& a = A.r[me];
    const int parity = (int)(((volatile const DevState*)a.st)->attempts & 1);   // same on every rank; graph-safe
    if ((PHASE & kPublish) && threadIdx.x == 0) {
        const int64_t tokens = a.tok_ptr ? *a.tok_ptr : a.local_tokens;
        const int64_t mine[2] = {tokens, mag_units(*a.stat)};
        *a.stat = 0;                                   // re-armed for the next update
        const size_t slot_off = area_off + ((size_t)parity * W + me) * 16;
#pragma unroll
        for (int p = 0; p < W; ++p) {
            int64_t* dst = (int64_t*)pe.at(p, slot_off);
            dst[0] = mine[0];
            dst[1] = mine[1];
        }
    }
    if (PHASE == kBoth) pe.sync(barrier_index);       // the whole CTA takes the barrier
    if ((PHASE & kDecide) && threadIdx.x == 0) {
        const int64_t* area = (const int64_t*)pe.at(me, area_off + (size_t)parity * W * 16);
        int64_t N = 0, M = 0;
        for (int p = 0; p < W; ++p) {
            N += ((volatile const int64_t*)area)[2 * p];
            M += ((volatile const int64_t*)area)[2 * p + 1];
        }
        a.xs[0] = N;
        a.xs[1] = M;
        if (M >= kNonFinite) decide(1, N, a.st, a.sc, a.loss_scale, a.ring, ring_mask, cfg, DEC_APPLY);
        else if (M <= (int64_t(1) << 39)) decide(0, N, a.st, a.sc, a.loss_scale, a.ring, ring_mask, cfg, DEC_APPLY);
        else a.sc->state = DEC_UNDECIDED;
    }
}

// Late decision of the sharded path (only when K0 EARLY was undecided, identically on every rank): each rank
// swept its own shard of R; the flags are OR-ed through peer memory, then decided as K0 LATE.
template <int W, class Peers, int PHASE>
__global__ void k0_late_x(Peers pe, size_t area_off, DecArgsW A, int ring_mask, DevCfg cfg, uint32_t barrier_index) {
    const int me = pe.rank();
    const DecArgs& a = A.r[me];
    // read by every thread before anybody decides: uniform over the CTA, and the same on every rank
    if (decision_of(a.sc) != DEC_UNDECIDED) {          // decided early: nobody takes the barrier
        if ((PHASE & kDecide) && threadIdx.x == 0) *(volatile int*)a.flag = 0;
        return;
    }
    const int parity = (int)(((volatile const DevState*)a.st)->attempts & 1);
    area_off += 2 * kMaxLsaRanks * 16;                 // slots of their own: the early exchange may still be read
    if ((PHASE & kPublish) && threadIdx.x == 0) {
        const int64_t mine = *(volatile int*)a.flag != 0;
        const size_t slot_off = area_off + ((size_t)parity * W + me) * 16;
        for (int p = 0; p < W; ++p) *(int64_t*)pe.at(p, slot_off) = mine;
    }
    if (PHASE == kBoth) pe.sync(barrier_index);
    if ((PHASE & kDecide) && threadIdx.x == 0) {
        const int64_t* area = (const int64_t*)pe.at(me, area_off + (size_t)parity * W * 16);
        int64_t any = 0;
        for (int p = 0; p < W; ++p) any |= ((volatile const int64_t*)area)[2 * p];
        decide(any != 0, a.xs[0], a.st, a.sc, a.loss_scale, a.ring, ring_mask, cfg, DEC_APPLY_LATE);
        *(volatile int*)a.flag = 0;
    }
}

// ============================================================================ sharded optimizer
// An adjacent variant of the paper's replicated update, opt-in (smpu_config.sharded): the bucket all-reduce
// becomes a reduce-scatter (R of my shard only, same ascending-rank order), Adam runs on my shard only and
// all-gathers the fp16 weights by storing w16 of the shard into every rank's window.  Per element the
// arithmetic is exactly the replicated path's, so theta/m/v of a shard and the full w16 are bitwise those of
// the replicated update; HBM per rank for the optimizer drops from 28 to ~28/W + 2 bytes per element.

// Reduce-scatter of one bucket: like k_ar16, but R is stored into my own window only.  No closing barrier:
// the end-of-update barrier orders every rank's reads of my accumulator before anybody's next update overwrites it.
template <int W, class Peers>
__global__ void __launch_bounds__(256) k_rs(Peers pe, int64_t lo, int64_t hi) {
    pe.sync(pe.cta());
    uint16_t* base[W];
#pragma unroll
    for (int p = 0; p < W; ++p) base[p] = (uint16_t*)pe.at(p, 0);
    const int me = pe.rank();
    const int64_t v0 = (lo + 7) & ~(int64_t)7, v1 = hi & ~(int64_t)7;
    const int64_t units = v1 > v0 ? (v1 - v0) / 8 : 0;
    const int64_t per = (units + W - 1) / W;
    int64_t u_lo = me * per, u_hi = u_lo + per;
    if (u_lo > units) u_lo = units;
    if (u_hi > units) u_hi = units;
    const int64_t tid = (int64_t)pe.cta() * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)pe.ctas() * blockDim.x;
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
    if (me == 0) head_tail<W, false>(base, lo, hi, v0, v1, tid, nthr);
}

// Adam on [lo, hi) of my shard (one-shot), w16 stored into every rank's window at window offset w16_off.
template <int W, class Peers>
__global__ void __launch_bounds__(256, 4) k2_adam_shard(Peers pe, size_t w16_off, float* __restrict__ theta,
                                                        float* __restrict__ m, float* __restrict__ v,
                                                        const uint16_t* __restrict__ R, int64_t lo, int64_t hi,
                                                        const Scalars* __restrict__ scp, int32_t need) {
    if (decision_of(scp) != need) return;
    const Scalars s = *scp;
    uint16_t* wb[W];
#pragma unroll
    for (int p = 0; p < W; ++p) wb[p] = (uint16_t*)pe.at(p, w16_off);
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

// One cross-rank barrier (acquire + release, system scope) at barrier index `idx` (LsaPeers only: virtual ranks
// meet through stream events instead).
__global__ void k_lsa_barrier(LsaPeers pe, uint32_t idx) { pe.sync(idx); }

}  // namespace smpu
