// snp_device.cuh -- device layouts and sm_100a kernels of the SNP step engine.
//
// One simulation step of the reference (engine.py:441-458: sv_calc ->
// step_{sparse,ell,compressed} -> update_delays -> halting test) is executed
// as ONE fused, neuron-parallel kernel per step (`step_kernel`) plus, for the
// push formats, the paper's scatter kernels:
//
//   step_kernel (k):   finish step k-1 for neuron j
//                        C_k = Ĉ_{k-1} + [open_{k-1}(j)] * recv_{k-1}(j)
//                        D_k = fired_{k-1} ? d : max(D_{k-1} - 1, 0)
//                        (engine.py:263/307/352 + update_delays :358-366)
//                      NegativeSpikes guard on C_k (engine.py:264)
//                      select step k's rule (sv_calc, engine.py:192-236)
//                        Ĉ_k = C_k - c[r]  (COMPRESSED consumes at selection)
//                        publish P_k(j) = p[r] (pull) / chosen (push)
//                      last CTA: halting decision (engine.py:443-450)
//   push_kernel (k):   ELL (Alg. 4) / COMPRESSED-push (Alg. 5) scatter into
//                      recv with 64-bit RED.ADD (engine.py:290-300, :338-345)
//   dense_kernel (k):  S_k . M_Π over the fired rows (engine.py:257-262)
//
// recv(j) is either gathered from the in-adjacency (`pull`: sum of P_{k-1}
// over in-neighbours, atomic-free) or read from the `recv` array written by
// the push/dense kernels.  Deliveries to closed neurons are dropped at the
// destination (the open gate above), which is exactly the reference's
// per-target `delays[tgt] == 0` filter.
//
// All spike counts are int64 like the reference; thresholds / amounts /
// delays are stored as int32 (range-checked at engine creation).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace snp {

constexpr int kBlock = 256;
constexpr uint32_t kLightRules = 32;   // thread-per-neuron selection (32-bit mask)
constexpr uint32_t kLightIn = 256;     // thread-per-neuron gather
constexpr uint32_t kLightOut = 64;     // thread-per-rule scatter
constexpr uint32_t kExactBit = 0x80000000u;
#ifndef SNP_STEP_MIN_BLOCKS
#define SNP_STEP_MIN_BLOCKS 4
#endif
constexpr int kStepMinBlocks = SNP_STEP_MIN_BLOCKS;  // 4 caps the step kernel at 64 registers
constexpr int kGatherBatch = 4;        // uint4 index loads in flight per gather round

enum PMode { P_BIT = 0, P_U8 = 1, P_U16 = 2, P_U32 = 3 };

// tiled pull layout
#ifndef SNP_TILE_THREADS
#define SNP_TILE_THREADS 992  // 31 consumer warps + 1 producer warp = 1024 threads
#endif
constexpr int kTileThreads = SNP_TILE_THREADS;  // consumer threads per CTA (multiple of 32)
static_assert(kTileThreads % 32 == 0 && kTileThreads + 32 <= 1024, "CTA must fit 1024 threads");
constexpr int kSegEdges = 256;            // one warp pass: 8 consecutive words per lane
#ifndef SNP_SRC_BITS
#define SNP_SRC_BITS 15
#endif
constexpr uint32_t kSrcBits = SNP_SRC_BITS;  // source offset within a segment
constexpr uint32_t kDstBits = 32 - kSrcBits; // destination slot within a tile
constexpr uint32_t kSrcSpan = 1u << kSrcBits;
constexpr uint32_t kSrcMask = kSrcSpan - 1u;
static_assert(kDstBits + kSrcBits == 32, "segment words are 32 bits");
constexpr uint32_t kDummyEdge = 0xffffffffu;  // CSR / legacy padding marker
constexpr int kMaxTile = (1 << kDstBits) - 32;
enum RecvKind { RECV_PULL = 0, RECV_ARRAY = 1 };
enum Rec { REC_CONFIGS = 1, REC_DELAYS = 2, REC_SPIKING = 4 };
enum Halt { RUNNING = 0, HALT_STEP_LIMIT = 1, HALT_NO_APPLICABLE = 2, HALT_NEGATIVE = 3, HALT_EXCHANGE = 4, HALT_FAULT = 5 };
enum Stat { ST_STEPS = 0, ST_SCANNED, ST_FIRED, ST_SENDING, ST_EDGES, ST_ROWS, ST_OPEN, ST_COUNT };

// Run-control block in device memory.  Written by the last CTA of each
// step kernel, read by every CTA of the next kernel; the host reads it after
// each device loop segment.
struct Ctrl {
    long long step;          // k of the next step kernel
    long long max_steps;     // SimOptions.max_steps
    long long stop_at;       // segment end: kernels with step >= stop_at idle
    long long trace_base;    // step of trace row 0
    unsigned long long seed;
    long long neg_index;
    long long neg_value;
    unsigned long long stats[8];
    int policy;
    int record;
    int stats_on;
    int halted;
    int reason;
    int fired_any;
    int closed_any;
    int neg_any;
    unsigned int blocks_done;
    int push_armed;          // a scatter for step (step-1) is pending
    unsigned int list_count[2];   // dense fired-rule list, by step parity
    unsigned int heavy_count[2];  // push heavy queue, by step parity
    unsigned long long epoch;     // peer exchange: run number (snp_begin), high half of step flags
    int fault;                    // sticky internal error (binned push: a bin region overflowed)
};

struct StageDesc;

struct DevSys {
    long long q;
    long long m;
    const uint32_t* roff;     // [q+1] rule offsets
    const void* rw;           // [m] rule words (compact uint2 / wide uint4), hot path
    const uint32_t* rw4;      // [m] tiny rule words (tiled, when every rule fits) or null
    const int4* rrec;         // [m] {consumed, produced, delay, 0}, cold paths
    const uint32_t* outdeg;   // [q] out-degree (traffic counters only)
    const uint32_t* ioff;     // pull: [q+1] in-adjacency offsets (4-aligned)
    const uint32_t* isrc;     // pull: sources, padded with the sentinel q
    const uint32_t* soff;     // push COMPRESSED: [q+1] out-adjacency
    const uint32_t* sdst;
    const int2* ell;          // ELL: [m][ell_ld] (target, amount) pairs
    const uint32_t* ell_len;  // ELL: live pairs per rule column
    long long ell_ld;
    const int* dense;         // SPARSE: [m][dense_ld]
    long long dense_ld;
    const uint32_t* heavy;    // CTA-per-neuron list
    int n_heavy;
    // FirstApplicable guard index of the heavy-rule neurons (by heavy index):
    // exactly-thresholds with their lowest rule, at-least thresholds with the
    // prefix-minimum rule, each sorted by threshold
    const uint32_t* hx_eoff;
    const uint2* hx_e;
    const uint32_t* hx_aoff;
    const uint2* hx_a;
    // dense FirstApplicable table per heavy neuron (null / empty range = none):
    // hx_lut[hx_loff[h] + min(C, len - 1)] = local rule index or ~0
    const uint32_t* hx_loff;
    const uint32_t* hx_lut;
    const uint16_t* hx_lcnt;  // same indexing: number of applicable rules (saturated at 65535)
    int light_ctas;           // CTAs striding over light tiles
    int heavy_ctas;           // CTAs striding over the heavy list
    long long light_tiles;    // ceil(q / 256)
    int z;                    // max out-degree
    int ell_rows;             // z + 1
    long long p_common;       // P_BIT: the single produced amount
    // tiled pull (default COMPRESSED kernel)
    const uint32_t* seg_words;  // [nseg * kSegEdges] dst slot << kSrcBits | (src - seg_base)
    const uint32_t* seg_base;   // [nseg] first source of each segment, rounded down to 32
    const StageDesc* stages;    // TMA stage descriptors, tile-major (build_tiles)
    const uint32_t* tstage;     // [n_tiles + 1] stage range of each tile
    const uint32_t* stage_bases;  // segment bases per phase-1 stage (16-byte aligned runs)
    const uint32_t* tseg;       // [n_tiles + 1] segment range of each tile
    const uint32_t* theavy;     // [n_tiles + 1] range of s.heavy inside each tile
    int tile;                   // destinations per tile (multiple of 32)
    int ring;                   // TMA ring stages (<= kMaxRing)
    int rpn;                    // tiled: rules per neuron when every neuron has the same count (<= 32), else 0
    int pf;                     // tiled: ring stages prefetched into L2 ahead of the TMA copies (0 = off)
    int dbg;                    // timing experiments (SNPB200_DEBUG_SKIP): 1 skip phase-1 math, 2 skip phase 2
    long long n_tiles;
    // row partition (sharded.py): local neuron j is global neuron gbase + j and
    // publishes its P element (bit / u8 / u16 / u32) at exchange-space
    // position xbase + j; rank r's chunk is x_stride words, the last 4 of
    // which carry its step flags
    long long gbase;
    long long xbase;
    long long x_stride;         // words per rank chunk (0 = not sharded)
    int world;
    int rank;
    // two-pass receive (variant TILED2, large source ranges): pass 1 turns
    // each source window's P bits into one bit per in-edge (tp_bits, grouped
    // 32 per word in tile order); the tiled kernel's phase 1 then streams
    // 16-bit destination slots + those bits instead of segments + P windows
    int tp;                       // 1 = two-pass layout
    int tp_wlog;                  // log2 source-window size
    long long tp_nw;              // source windows
    const uint16_t* tp_slots;     // [groups * 32] destination slots, tile order (padding = T)
    uint32_t* tp_bits;            // [groups] per-step edge bits, tile order
    const uint16_t* tp_off;       // [groups * 32] source offsets in the window, window order
    const uint32_t* tp_gword;     // [groups] window-order group -> tile-order group
    const uint32_t* tp_wgroup;    // [tp_nw + 1] window -> first window-order group
    const uint4* tp_items;        // pass-1 work items {window, first group, end group, 0}
    long long tp_nitems;
    // peer exchange (NVLink P2P): every rank's exchange block (3 slots of
    // p_words words, then `world` 64-bit step flags), mapped into this process
    const unsigned long long* peers;
    long long p_words;
    int p2p;
    // binned push (ell_bin_step_kernel): destination tiles of bin_T, each with
    // a bin region [bin_off[t], bin_off[t] + bin_cap[t]) per step parity
    int bin_T;
    int bin_ntiles;
    unsigned long long bin_magic;  // ceil(2^64 / bin_T): floor(x / bin_T) = umul64hi(x, bin_magic) for x < 2^31
    int bin_amount;                // UNIT entries: the common amount of every delivery
    const uint32_t* bin_off;       // [ntiles + 1] main region starts (entries, multiples of 8)
    const uint32_t* bin_ooff;      // [ntiles + 1] overflow region starts (same buffer, after the main regions)
    int bin_cpc;                   // ELL: 16-byte chunks per column (ell_ld / 2) when <= 16, else 0
};

struct DevState {
    long long* cfg;           // Ĉ (C after this step's consumption)
    int* ds;                  // delay state, see decode_ds
    int* chosen;              // [q] chosen rule (push/dense formats, phase API)
    uint32_t* P[3];           // pull exchange vectors (triple buffered)
    long long* recv;          // push/dense accumulation
    void* rbuf[2];            // fused push (push_step_kernel): receive buffers by step parity, int32 or int64
    void* bins[2];            // binned push: bin entries by step parity (u16 slots or u32 slot|amount)
    uint32_t* bin_fill[2];    // binned push: [2 * ntiles] entries written into each tile's main / overflow region, by step parity
    uint32_t* list[2];        // fired rules (dense) / heavy queue (push), by parity
    Ctrl* ctrl;
    long long* tr_cfg;        // [tr_rows][q]
    int* tr_dly;
    int* tr_chosen;
    long long tr_rows;
};

// ---------------------------------------------------------------------------
// helpers

// Kernel-parameter arrays indexed with a runtime value are spilled to the
// stack; select through branches instead.
__device__ __forceinline__ uint32_t* pick3(uint32_t* const (&a)[3], long long i) {
    return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}
__device__ __forceinline__ uint32_t* pick2(uint32_t* const (&a)[2], long long i) {
    return (i & 1) ? a[1] : a[0];
}

// selection.py:37-45 -- SplitMix64-style finaliser, wrapping uint64.
__device__ __forceinline__ unsigned long long mix64(unsigned long long seed, long long step,
                                                    long long neuron) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(step + 1) +
                           0xBF58476D1CE4E5B9ull * (unsigned long long)(neuron + 1);
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

// Delay state word: ds < 0  -> fired last step with delay d = -ds-1 (open then)
//                   ds >= 0 -> did not fire; ds is that step's delay counter.
__device__ __forceinline__ bool ds_open(int ds) { return ds <= 0; }
__device__ __forceinline__ int ds_next(int ds) { return ds < 0 ? -ds - 1 : (ds > 0 ? ds - 1 : 0); }

// regex guard (model.py:58-61)
__device__ __forceinline__ bool guard_ok(uint32_t w, long long count) {
    long long t = (long long)(w & ~kExactBit);
    return (w & kExactBit) ? count == t : count >= t;
}

// position of the (k+1)-th set bit of mask (k < popc(mask))
__device__ __forceinline__ int nth_set_bit(uint32_t mask, uint32_t k) {
#pragma unroll 1
    for (uint32_t i = 0; i < k; ++i) mask &= mask - 1;
    return __ffs(mask) - 1;
}

__device__ __forceinline__ void red_add_i64(long long* addr, long long v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(v));
}

template <int PM>
__device__ __forceinline__ long long p_lookup(const uint32_t* __restrict__ P, uint32_t s) {
    if constexpr (PM == P_BIT) {
        return (__ldg(P + (s >> 5)) >> (s & 31)) & 1u;
    } else if constexpr (PM == P_U8) {
        return __ldg(reinterpret_cast<const uint8_t*>(P) + s);
    } else if constexpr (PM == P_U16) {
        return __ldg(reinterpret_cast<const uint16_t*>(P) + s);
    } else {
        return __ldg(P + s);
    }
}

// Thread-serial gather over a 4-aligned, sentinel-padded in-list.
template <int PM>
__device__ __forceinline__ long long gather_thread(const uint32_t* __restrict__ isrc,
                                                   const uint32_t* __restrict__ P,
                                                   uint32_t e0, uint32_t e1) {
    long long acc = 0;
    const uint4* p4 = reinterpret_cast<const uint4*>(isrc + e0);
    const uint32_t n4 = (e1 - e0) >> 2;
#pragma unroll 4
    for (uint32_t i = 0; i < n4; ++i) {
        uint4 v = __ldg(p4 + i);
        acc += p_lookup<PM>(P, v.x) + p_lookup<PM>(P, v.y) + p_lookup<PM>(P, v.z) +
               p_lookup<PM>(P, v.w);
    }
    return acc;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct BlockStats {
    unsigned long long v[ST_COUNT];
};

// Block-wide reduction of per-thread stats into Ctrl (one atomic per counter).
__device__ __forceinline__ void flush_stats(Ctrl* ctl, unsigned int (&loc)[ST_COUNT]) {
    __shared__ unsigned long long sh[ST_COUNT];
    if (threadIdx.x < ST_COUNT) sh[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ST_COUNT; ++i) {
        unsigned long long v = loc[i];  // per-thread counts fit 32 bits; sums may not
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sh[i], v);
    }
    __syncthreads();
    if (threadIdx.x < ST_COUNT && sh[threadIdx.x]) atomicAdd(&ctl->stats[threadIdx.x], sh[threadIdx.x]);
}

// ---- peer exchange (row partition over NVLink P2P, sharded.py)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Step flag value of run `epoch` after step k: monotonic across runs.
__device__ __forceinline__ unsigned long long step_tag(unsigned long long epoch, long long k) {
    return (epoch << 32) | (unsigned long long)(k + 1);
}
__device__ __forceinline__ uint32_t* peer_slot(const DevSys& s, int r, long long slot) {
    return reinterpret_cast<uint32_t*>(s.peers[r]) + slot * s.p_words;
}
__device__ __forceinline__ unsigned long long* peer_flags(const DevSys& s, int r) {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<uint32_t*>(s.peers[r]) + 3 * s.p_words);
}
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

// Wait until every rank has published step `kdone` (its P chunk and header
// are in this rank's slot kdone % 3).  Returns false on timeout.
static __device__ __noinline__ bool wait_peers(const DevSys& s, unsigned long long epoch, long long kdone) {
    const unsigned long long want = step_tag(epoch, kdone);
    const unsigned long long* fl = peer_flags(s, s.rank);
    const unsigned long long t0 = globaltimer_ns();
    for (int r = 0; r < s.world; ++r) {
        while (ld_acquire_sys(fl + r) < want) {
            if (globaltimer_ns() - t0 > kPeerTimeoutNs) return false;
            __nanosleep(100);
        }
    }
    return true;
}

// Last CTA of a peer-exchange step: this rank's header words (already in its
// own slot) go to every peer, then the step flag (release) to every rank.
static __device__ __noinline__ void publish_peers(const DevSys& s, long long k, unsigned long long epoch, const uint32_t* hdr) {
    const long long slot = k % 3;
    const long long hw = (long long)s.rank * s.x_stride + s.x_stride - 4;
    for (int r = 0; r < s.world; ++r) {
        if (r == s.rank) continue;
        volatile uint32_t* d = peer_slot(s, r, slot) + hw;
        d[0] = hdr[0];
        d[1] = hdr[1];
        d[2] = hdr[2];
        d[3] = hdr[3];
    }
    __threadfence_system();
    for (int r = 0; r < s.world; ++r) st_release_sys(peer_flags(s, r) + s.rank, step_tag(epoch, k));
}

// Last-CTA-done: halting decision for step k (engine.py:443-450) and reset
// of the per-step flags.  Called by thread 0 of every CTA.
__device__ __forceinline__ void finish_step(Ctrl* ctl, long long k, bool sel, bool bf, bool bc,
                                            bool bn, long long neg_idx, long long neg_val,
                                            uint32_t* xhdr = nullptr, const DevSys* p2p = nullptr) {
    if (bf) atomicOr(&ctl->fired_any, 1);
    if (bc) atomicOr(&ctl->closed_any, 1);
    if (bn) {
        atomicOr(&ctl->neg_any, 1);
        long long prev = atomicMin(&ctl->neg_index, neg_idx);
        if (neg_idx < prev) ctl->neg_value = neg_val;  // best effort (diagnostics only)
    }
    if (p2p) __threadfence_system();  // this CTA's peer stores before the flag
    else __threadfence();
    unsigned int done = atomicAdd(&ctl->blocks_done, 1u);
    if (done != gridDim.x - 1) return;
    __threadfence();
    volatile Ctrl* v = ctl;
    const int fired = v->fired_any, closed = v->closed_any, neg = v->neg_any;
    v->fired_any = 0;
    v->closed_any = 0;
    v->blocks_done = 0;
    // counters used by the NEXT step (parity (k+1)&1) start from zero
    v->list_count[(k + 1) & 1] = 0;
    v->heavy_count[(k + 1) & 1] = 0;
    int armed = 0;
    if (xhdr) {
        // row partition: publish this rank's flags with its P chunk; every
        // rank takes the same decision at the start of the next step kernel
        volatile uint32_t* h = xhdr;
        h[0] = (uint32_t)fired;
        h[1] = (uint32_t)closed;
        h[2] = (uint32_t)neg;
        h[3] = 0u;
        if (p2p) publish_peers(*p2p, k, v->epoch, xhdr);
        // a step kernel without selection (k == max_steps) still finished
        // step k-1 and may have seen a negative count on any rank: the next
        // kernel decides NegativeSpikes vs STEP_LIMIT from every rank's
        // header (tiled_step_kernel's partition check), as for any step
        v->step = k + 1;
        if (sel && v->stats_on) v->stats[ST_STEPS] += 1;
        v->push_armed = 0;
        __threadfence();
        return;
    }
    if (v->fault) {
        v->halted = 1;
        v->reason = HALT_FAULT;
    } else if (neg) {
        v->halted = 1;
        v->reason = HALT_NEGATIVE;
    } else if (!sel) {
        v->halted = 1;
        v->reason = HALT_STEP_LIMIT;
    } else if (!fired && !closed) {
        v->halted = 1;
        v->reason = HALT_NO_APPLICABLE;
    } else {
        v->step = k + 1;
        armed = 1;
        if (v->stats_on) v->stats[ST_STEPS] += 1;
    }
    v->push_armed = armed;
    __threadfence();
}

// ---------------------------------------------------------------------------
// Rule words.  Compact: uint2 {guard, c | p << 16 | d << 24} when every rule
// has c < 2^16, p < 2^8, d < 2^8 (one 8-byte word carries everything the
// step needs, so selection and consumption read one sector per neuron);
// otherwise wide: uint4 {guard, c, p, d}.
// Tiny: one 32-bit word per rule for the tiled kernel's staged selection:
// threshold[9:0] | exact[10] | consumed[20:11] | produced[24:21] | delay[31:25]
// (host-checked ranges); the compact / wide words stay the general store.
enum RuleWords { RW_COMPACT = 0, RW_WIDE = 1, RW_TINY = 2 };
__host__ __device__ constexpr uint32_t tiny_word(uint32_t guard, uint32_t c, uint32_t p, uint32_t d) {
    return (guard & 0x3ffu) | ((guard & kExactBit) ? 0x400u : 0u) | (c << 11) | (p << 21) | (d << 25);
}

template <bool WIDE>
__device__ __forceinline__ uint4 load_rule(const void* __restrict__ rw, uint32_t r) {
    if constexpr (WIDE) {
        return __ldg(reinterpret_cast<const uint4*>(rw) + r);
    } else {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(rw) + r);
        return make_uint4(w.x, w.y & 0xffffu, (w.y >> 16) & 0xffu, w.y >> 24);
    }
}
template <bool WIDE>
struct RuleRaw {
    using T = uint2;
};
template <>
struct RuleRaw<true> {
    using T = uint4;
};
template <bool WIDE>
__device__ __forceinline__ typename RuleRaw<WIDE>::T load_raw(const void* __restrict__ rw, uint32_t r) {
    return __ldg(reinterpret_cast<const typename RuleRaw<WIDE>::T*>(rw) + r);
}
template <bool WIDE>
__device__ __forceinline__ uint4 unpack_rule(typename RuleRaw<WIDE>::T w) {
    if constexpr (WIDE) {
        return w;
    } else {
        return make_uint4(w.x, w.y & 0xffffu, (w.y >> 16) & 0xffu, w.y >> 24);
    }
}
__device__ __forceinline__ uint32_t rule_guard_word(const void* __restrict__ rw, bool wide, uint32_t r) {
    return wide ? __ldg(reinterpret_cast<const uint4*>(rw) + r).x : __ldg(reinterpret_cast<const uint2*>(rw) + r).x;
}

// Gather over a 4-aligned, sentinel-padded in-list with batched independent
// loads: kGatherBatch uint4 index loads in flight, then their P lookups.
template <int PM>
__device__ __forceinline__ long long gather_batched(const uint32_t* __restrict__ isrc,
                                                    const uint32_t* __restrict__ P, uint32_t e0,
                                                    uint32_t e1) {
    const uint4* p4 = reinterpret_cast<const uint4*>(isrc + e0);
    const uint32_t n4 = (e1 - e0) >> 2;
    long long acc = 0;
    for (uint32_t b = 0; b < n4; b += kGatherBatch) {
        uint4 v[kGatherBatch];
#pragma unroll
        for (int i = 0; i < kGatherBatch; ++i)
            if (b + i < n4) v[i] = __ldg(p4 + b + i);
#pragma unroll
        for (int i = 0; i < kGatherBatch; ++i)
            if (b + i < n4)
                acc += p_lookup<PM>(P, v[i].x) + p_lookup<PM>(P, v[i].y) + p_lookup<PM>(P, v[i].z) +
                       p_lookup<PM>(P, v[i].w);
    }
    return acc;
}

// Per-step constants shared by the step kernels.
struct StepCtx {
    long long k;
    long long slot;
    long long q;
    unsigned long long seed;
    uint32_t* Pcur;
    int policy;
    int record;
    bool sel;
    bool stats_on;
};

// Light-neuron tail of a step: C_k / D_k are final; records the trace rows,
// applies the NegativeSpikes guard, selects among <= 32 rules (the first
// four words w0..w3 were preloaded by the caller), commits Ĉ_k / delay state
// / chosen and publishes non-bit P.  Returns the produced amount (0 if none).
template <int KIND, int PM, bool CONSUME, bool FLIST, bool WIDE>
__device__ __forceinline__ long long light_commit(const DevSys& s, const DevState& st, Ctrl* ctl, const StepCtx& cx,
                                                  long long j, uint32_t r0, uint32_t nr,
                                                  typename RuleRaw<WIDE>::T w0, typename RuleRaw<WIDE>::T w1,
                                                  typename RuleRaw<WIDE>::T w2, typename RuleRaw<WIDE>::T w3,
                                                  long long C, int D, bool can_sel, unsigned int (&stat)[ST_COUNT],
                                                  bool& t_fired, bool& t_closed, bool& t_neg, long long& neg_idx,
                                                  long long& neg_val, int& r) {
    long long pval = 0;
    if (C < 0) {
        t_neg = true;
        neg_idx = j + s.gbase;
        neg_val = C;
    }
    if (cx.record & REC_CONFIGS) st.tr_cfg[cx.slot * cx.q + j] = C;
    if (cx.record & REC_DELAYS) st.tr_dly[cx.slot * cx.q + j] = D;
    t_closed |= D != 0;
    uint4 wr = make_uint4(0, 0, 0, 0);
    if (can_sel) {
        uint32_t mask = (nr > 0 && guard_ok(w0.x, C) ? 1u : 0u) |
                        (nr > 1 && guard_ok(w1.x, C) ? 2u : 0u) |
                        (nr > 2 && guard_ok(w2.x, C) ? 4u : 0u) |
                        (nr > 3 && guard_ok(w3.x, C) ? 8u : 0u);
        for (uint32_t t = 4; t < nr; ++t)
            mask |= (uint32_t)guard_ok(rule_guard_word(s.rw, WIDE, r0 + t), C) << t;
        stat[ST_OPEN] += 1;
        if (mask) {
            int idx;
            if (cx.policy == 0) {
                idx = __ffs(mask) - 1;
                stat[ST_SCANNED] += idx + 1;
            } else {
                idx = nth_set_bit(mask, (uint32_t)(mix64(cx.seed, cx.k, j + s.gbase) % (uint32_t)__popc(mask)));
                stat[ST_SCANNED] += nr;
            }
            r = (int)(r0 + idx);
            wr = unpack_rule<WIDE>(idx == 0 ? w0 : idx == 1 ? w1 : idx == 2 ? w2 : idx == 3 ? w3
                                                                          : load_raw<WIDE>(s.rw, r));
        } else {
            stat[ST_SCANNED] += nr;
        }
    }
    int nds = D;
    long long Cn = C;
    if (r >= 0) {
        if (CONSUME) Cn -= (long long)wr.y;
        pval = (long long)wr.z;
        nds = -((int)wr.w + 1);
        t_fired = true;
        stat[ST_FIRED] += 1;
        if (pval > 0) {
            stat[ST_SENDING] += 1;
            if (cx.stats_on) {
                const uint32_t od = __ldg(s.outdeg + j);
                stat[ST_ROWS] += od + (od < (uint32_t)s.z ? 1u : 0u);
            }
        }
        if (FLIST) {
            unsigned int pos = atomicAdd(&ctl->list_count[cx.k & 1], 1u);
            pick2(st.list, cx.k)[pos] = (uint32_t)r;
        }
    }
    st.cfg[j] = Cn;
    st.ds[j] = nds;
    if (cx.sel) {
        if (KIND == RECV_ARRAY) st.chosen[j] = r;
        if (cx.record & REC_SPIKING) st.tr_chosen[cx.slot * cx.q + j] = r;
        if (KIND == RECV_PULL && PM != P_BIT) {
            if (PM == P_U8) reinterpret_cast<uint8_t*>(cx.Pcur)[j + s.xbase] = (uint8_t)pval;
            else if (PM == P_U16) reinterpret_cast<uint16_t*>(cx.Pcur)[j + s.xbase] = (uint16_t)pval;
            else cx.Pcur[j + s.xbase] = (uint32_t)pval;
        }
    }
    return pval;
}

// x mod c for c in 1..4 (choose_index, selection.py:66-71) without a 64-bit
// division: 2^32 = 1 (mod 3), so x mod 3 = (hi mod 3 + lo mod 3) mod 3.
__device__ __forceinline__ uint32_t mod_upto4(unsigned long long x, uint32_t c) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    if (c == 3) return (hi % 3u + lo % 3u) % 3u;
    return lo & (c - 1u);  // c = 1, 2, 4
}

// FirstApplicable over a heavy-rule neuron through its guard index: the
// lowest rule whose guard holds for count C (local index), or -1.
__device__ __forceinline__ int heavy_first_applicable(const DevSys& s, int h, long long C) {
    if (C < 0) return -1;
    const uint32_t cc = (C >> 31) != 0 ? 0x80000000u : (uint32_t)C;
    uint32_t best = 0xffffffffu;
    {   // exactly: threshold == cc
        uint32_t lo = __ldg(s.hx_eoff + h), hi = __ldg(s.hx_eoff + h + 1);
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&s.hx_e[mid].x) < cc) lo = mid + 1;
            else hi = mid;
        }
        if (lo < __ldg(s.hx_eoff + h + 1)) {
            const uint2 v = __ldg(&s.hx_e[lo]);
            if (v.x == cc) best = v.y;
        }
    }
    {   // at least: the last threshold <= cc carries the prefix minimum
        const uint32_t a0 = __ldg(s.hx_aoff + h);
        uint32_t lo = a0, hi = __ldg(s.hx_aoff + h + 1);
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&s.hx_a[mid].x) <= cc) lo = mid + 1;
            else hi = mid;
        }
        if (lo > a0) best = min(best, __ldg(&s.hx_a[lo - 1].y));
    }
    return best == 0xffffffffu ? -1 : (int)best;
}

// Warp-cooperative 32-ary search over sorted guard keys [lo, hi): the number
// of keys with x < v (UPPER = false) or x <= v (UPPER = true).  Each round
// the 32 lanes probe 32 evenly spaced keys with one load, so a 4096-key
// index takes 3 dependent loads instead of 12.  All lanes return the result.
template <bool UPPER>
__device__ __forceinline__ uint32_t warp_bound(const uint2* __restrict__ keys, uint32_t lo, uint32_t hi, uint32_t v,
                                               int lane) {
    uint32_t len = hi - lo;
    while (len > 32) {
        const uint32_t step = (len + 31u) >> 5;
        const uint32_t idx = lo + (uint32_t)(lane + 1) * step - 1u;
        bool below = false;
        if (idx < lo + len) {
            const uint32_t x = __ldg(&keys[idx].x);
            below = UPPER ? x <= v : x < v;
        }
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, below));
        const uint32_t nlo = lo + c * step;
        const uint32_t nhi = min(lo + len, lo + (c + 1u) * step - 1u);
        lo = nlo;
        len = nhi - nlo;
    }
    bool below = false;
    if ((uint32_t)lane < len) {
        const uint32_t x = __ldg(&keys[lo + lane].x);
        below = UPPER ? x <= v : x < v;
    }
    return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// FirstApplicable from the dense table alone (one thread): local rule index,
// -1 (none applicable), or -2 (this neuron has no table).
__device__ __forceinline__ int heavy_first_table(const DevSys& s, int h, long long C) {
    if (C < 0) return -1;
    if (!s.hx_loff) return -2;
    const uint32_t l0 = __ldg(s.hx_loff + h), l1 = __ldg(s.hx_loff + h + 1);
    if (l1 == l0) return -2;
    const uint32_t c = C >= (long long)(l1 - l0 - 1) ? l1 - l0 - 1 : (uint32_t)C;
    const uint32_t v = __ldg(s.hx_lut + l0 + c);
    return v == 0xffffffffu ? -1 : (int)v;
}

// heavy_first_applicable, one warp (all lanes get the answer).
__device__ __forceinline__ int heavy_first_applicable_warp(const DevSys& s, int h, long long C, int lane) {
    if (C < 0) return -1;
    if (s.hx_loff) {
        const uint32_t l0 = __ldg(s.hx_loff + h), l1 = __ldg(s.hx_loff + h + 1);
        if (l1 > l0) {
            const uint32_t c = C >= (long long)(l1 - l0 - 1) ? l1 - l0 - 1 : (uint32_t)C;
            const uint32_t v = __ldg(s.hx_lut + l0 + c);
            return v == 0xffffffffu ? -1 : (int)v;
        }
    }
    const uint32_t cc = (C >> 31) != 0 ? 0x80000000u : (uint32_t)C;
    uint32_t best = 0xffffffffu;
    {   // exactly: the first threshold >= cc, if it equals cc
        const uint32_t e0 = __ldg(s.hx_eoff + h), e1 = __ldg(s.hx_eoff + h + 1);
        const uint32_t i = warp_bound<false>(s.hx_e, e0, e1, cc, lane);
        if (i < e1) {
            const uint2 v = __ldg(&s.hx_e[i]);
            if (v.x == cc) best = v.y;
        }
    }
    {   // at least: the last threshold <= cc carries the prefix minimum
        const uint32_t a0 = __ldg(s.hx_aoff + h), a1 = __ldg(s.hx_aoff + h + 1);
        const uint32_t i = warp_bound<true>(s.hx_a, a0, a1, cc, lane);
        if (i > a0) best = min(best, __ldg(&s.hx_a[i - 1].y));
    }
    return best == 0xffffffffu ? -1 : (int)best;
}

// SeededRandom through the dense table: when at most one rule is applicable
// for count C the choice is forced (mix64 % 1 = 0, choose_index), so no scan
// is needed.  Returns the local rule index, -1 (none applicable) or -2 (no
// table, or several applicable: scan).
__device__ __forceinline__ int heavy_seeded_table(const DevSys& s, int h, long long C) {
    if (C < 0) return -1;
    if (!s.hx_loff) return -2;
    const uint32_t l0 = __ldg(s.hx_loff + h), l1 = __ldg(s.hx_loff + h + 1);
    if (l1 == l0) return -2;
    const uint32_t c = C >= (long long)(l1 - l0 - 1) ? l1 - l0 - 1 : (uint32_t)C;
    const uint32_t n = __ldg(s.hx_lcnt + l0 + c);
    if (n == 0) return -1;
    if (n > 1) return -2;
    return (int)__ldg(s.hx_lut + l0 + c);
}

// SeededRandom over a heavy-rule neuron, one warp: count the applicable
// rules, then take the (mix64 % count)-th in index order (choose_index,
// selection.py:66-71).  Returns the global rule id or -1 (all lanes).
template <bool WIDE>
__device__ __forceinline__ int heavy_seeded_warp(const DevSys& s, uint32_t r0, uint32_t r1, long long C,
                                                 unsigned long long seed, long long k, long long jg, int lane) {
    uint32_t cnt = 0;
#pragma unroll 4
    for (uint32_t t = r0 + lane; t < r1; t += 32) cnt += guard_ok(rule_guard_word(s.rw, WIDE, t), C) ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (cnt == 0) return -1;
    uint32_t want = (uint32_t)(mix64(seed, k, jg) % cnt);
    for (uint32_t base = r0; base < r1; base += 32) {
        const uint32_t t = base + lane;
        const bool ok = t < r1 && guard_ok(rule_guard_word(s.rw, WIDE, t), C);
        const uint32_t b = __ballot_sync(0xffffffffu, ok);
        const uint32_t c = __popc(b);
        if (want < c) return (int)(base + nth_set_bit(b, want));
        want -= c;
    }
    return -1;  // not reached
}

// Lean light-neuron tail (no recording, no counters) for <= 4 compact rule
// words already in shared memory: the same decisions as light_commit, computed
// branch-free on a 32-bit saturated count (thresholds are < 2^31).  A negative
// count selects nothing, as in light_commit (no guard matches C < 0).
template <int PM, bool TINY>
__device__ __forceinline__ long long lean_commit4(const DevSys& s, const DevState& st, Ctrl* ctl, const StepCtx& cx,
                                                  long long j, uint32_t nr, const void* rpv, long long C, int D,
                                                  bool can_sel, bool& t_fired, bool& t_closed, bool& t_neg) {
    if (__builtin_expect(C < 0, 0)) {
        // NegativeSpikes (engine.py:48-54): rare, reported straight to Ctrl
        t_neg = true;
        const long long jg = j + s.gbase;
        if (jg < atomicMin(&ctl->neg_index, jg)) ctl->neg_value = C;
    }
    t_closed |= D != 0;
    // Guard of a rule with threshold t: count in [t, t] (exactly) or [t, inf)
    // (at least).  With the count saturated to cc <= 2^31 and t < 2^31 that is
    // one unsigned compare: (cc - t) <= lim, lim = 0 (exactly) or 2^31.
    const uint32_t cc = (C >> 31) != 0 ? 0x80000000u : (uint32_t)C;
    uint32_t w[4], y[4];
    uint32_t mask = 0;
    if (TINY) {
        const uint32_t* rp = reinterpret_cast<const uint32_t*>(rpv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w[k] = rp[k];
            const uint32_t lim = ~(w[k] << 21) & 0x80000000u;  // exact bit 10 -> 31
            mask |= (cc - (w[k] & 0x3ffu)) <= lim ? (1u << k) : 0u;
        }
    } else {
        const uint2* rp = reinterpret_cast<const uint2*>(rpv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint2 v = rp[k];
            w[k] = v.x;
            y[k] = v.y;
            mask |= (cc - (v.x & ~kExactBit)) <= (~v.x & kExactBit) ? (1u << k) : 0u;
        }
    }
    mask &= (can_sel && C >= 0) ? (1u << nr) - 1u : 0u;
    int idx;
    if (cx.policy == 0) {
        idx = __ffs(mask) - 1;
    } else {
        idx = mask ? nth_set_bit(mask, mod_upto4(mix64(cx.seed, cx.k, j + s.gbase), (uint32_t)__popc(mask))) : 0;
    }
    uint32_t c, p, d;
    if (TINY) {
        const uint32_t ws = idx <= 0 ? w[0] : (idx == 1 ? w[1] : (idx == 2 ? w[2] : w[3]));
        c = (ws >> 11) & 0x3ffu, p = (ws >> 21) & 0xfu, d = ws >> 25;
    } else {
        const uint32_t ys = idx <= 0 ? y[0] : (idx == 1 ? y[1] : (idx == 2 ? y[2] : y[3]));
        c = ys & 0xffffu, p = (ys >> 16) & 0xffu, d = ys >> 24;
    }
    const bool fired = mask != 0;
    t_fired |= fired;
    st.cfg[j] = fired ? C - (long long)c : C;
    st.ds[j] = fired ? -(int)(d + 1u) : D;
    p = fired ? p : 0u;
    if (PM != P_BIT && cx.sel) {
        if (PM == P_U8) reinterpret_cast<uint8_t*>(cx.Pcur)[j + s.xbase] = (uint8_t)p;
        else if (PM == P_U16) reinterpret_cast<uint16_t*>(cx.Pcur)[j + s.xbase] = (uint16_t)p;
        else cx.Pcur[j + s.xbase] = p;
    }
    return (long long)p;
}

// ---------------------------------------------------------------------------
// The fused step kernel.
//
// Light CTAs (blockIdx < light_ctas) stride over 256-neuron tiles, thread ->
// neuron (light neurons: <= 32 rules and, for pull, in-degree <= 256).  Heavy
// CTAs stride over s.heavy, one neuron at a time (e.g. the sorter's detectors
// with n rules and n in-neighbours): block-strided gather + block-wide ballot
// scan.  The grid is sized to the resident capacity of the 148 SMs, so the
// per-CTA end-of-step reductions are few.

template <int KIND, int PM, bool CONSUME, bool FLIST, bool WIDE>
__global__ void __launch_bounds__(kBlock, kStepMinBlocks) step_kernel(const __grid_constant__ DevSys s, DevState st) {
    Ctrl* ctl = st.ctrl;
    const volatile Ctrl* vc = ctl;
    const int halted = vc->halted;
    const long long k = vc->step;
    if (halted || k >= vc->stop_at) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->push_armed = 0;
        return;
    }
    const bool sel = k < vc->max_steps;
    const int policy = vc->policy;
    const unsigned long long seed = vc->seed;
    const int record = vc->record;
    const bool stats_on = vc->stats_on != 0;
    const long long slot = k - vc->trace_base;
    const uint32_t* __restrict__ Pprev = pick3(st.P, (k + 2) % 3);
    uint32_t* Pcur = pick3(st.P, k % 3);
    uint32_t* Pzero = pick3(st.P, (k + 1) % 3);
    const long long q = s.q;
    const StepCtx cx{k, slot, q, seed, Pcur, policy, record, sel, stats_on};

    unsigned int stat[ST_COUNT];
#pragma unroll
    for (int i = 0; i < ST_COUNT; ++i) stat[i] = 0;
    bool t_fired = false, t_closed = false, t_neg = false;
    long long neg_idx = 0x7fffffffffffffffll, neg_val = 0;

    if (blockIdx.x < (unsigned)s.light_ctas) {
        // ------------------------------------------------------------ light
        for (long long tile = blockIdx.x; tile < s.light_tiles; tile += s.light_ctas) {
            const long long j = tile * kBlock + threadIdx.x;
            const bool active = j < q;
            uint32_t r0 = 0, r1 = 0, e0 = 0, e1 = 0;
            long long Cprev = 0;
            int dsv = 0;
            if (active) {
                r0 = __ldg(s.roff + j);
                r1 = __ldg(s.roff + j + 1);
                if (KIND == RECV_PULL) {
                    e0 = __ldg(s.ioff + j);
                    e1 = __ldg(s.ioff + j + 1);
                }
                Cprev = st.cfg[j];
                dsv = st.ds[j];
            }
            const uint32_t nr = r1 - r0;
            const bool heavy = active && (nr > kLightRules || (KIND == RECV_PULL && (e1 - e0) > kLightIn));
            const bool mine = active && !heavy;
            int r = -1;
            long long pval = 0;
            if (mine) {
                const bool open_prev = ds_open(dsv);
                const int D = ds_next(dsv);
                const bool can_sel = sel && D == 0;
                // rule words of the first 4 rules, issued with the gather
                using Raw = typename RuleRaw<WIDE>::T;
                Raw w0{}, w1{}, w2{}, w3{};
                if (can_sel) {
                    if (nr > 0) w0 = load_raw<WIDE>(s.rw, r0);
                    if (nr > 1) w1 = load_raw<WIDE>(s.rw, r0 + 1);
                    if (nr > 2) w2 = load_raw<WIDE>(s.rw, r0 + 2);
                    if (nr > 3) w3 = load_raw<WIDE>(s.rw, r0 + 3);
                }
                long long C = Cprev;
                if (KIND == RECV_PULL) {
                    if (open_prev && e1 > e0) {
                        const long long g = gather_batched<PM>(s.isrc, Pprev, e0, e1);
                        C += (PM == P_BIT) ? g * s.p_common : g;
                        stat[ST_EDGES] += e1 - e0;
                    }
                } else {
                    const long long rv = st.recv[j];
                    if (rv != 0) st.recv[j] = 0;
                    if (open_prev) C += rv;
                }
                pval = light_commit<KIND, PM, CONSUME, FLIST, WIDE>(s, st, ctl, cx, j, r0, nr, w0, w1, w2, w3, C, D,
                                                                    can_sel, stat, t_fired, t_closed, t_neg, neg_idx,
                                                                    neg_val, r);
            }
            if (KIND == RECV_PULL && PM == P_BIT && sel) {
                // one 32-neuron word per warp: lanes are consecutive neurons
                const unsigned int bits = __ballot_sync(0xffffffffu, mine && pval > 0);
                const unsigned int hv = __ballot_sync(0xffffffffu, heavy);
                const unsigned int act = __ballot_sync(0xffffffffu, active);
                if ((threadIdx.x & 31) == 0 && act) {
                    const long long w = j >> 5;
                    Pzero[w] = 0u;
                    if (hv) {
                        if (bits) atomicOr(Pcur + w, bits);
                    } else {
                        Pcur[w] = bits;
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ heavy
        __shared__ long long sh_sum[kBlock / 32];
        __shared__ int sh_pick;
        __shared__ unsigned int sh_cnt[kBlock / 32];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int h = blockIdx.x - s.light_ctas; h < s.n_heavy; h += s.heavy_ctas) {
            const long long j = s.heavy[h];
            const uint32_t r0 = __ldg(s.roff + j), r1 = __ldg(s.roff + j + 1);
            long long C = st.cfg[j];
            const int dsv = st.ds[j];
            const bool open_prev = ds_open(dsv);
            __syncthreads();  // shared scratch reuse across iterations
            if (KIND == RECV_PULL) {
                long long part = 0;
                if (open_prev) {
                    const uint32_t e0 = __ldg(s.ioff + j), e1 = __ldg(s.ioff + j + 1);
                    for (uint32_t e = e0 + threadIdx.x; e < e1; e += kBlock)
                        part += p_lookup<PM>(Pprev, __ldg(s.isrc + e));
                    if (threadIdx.x == 0) stat[ST_EDGES] += e1 - e0;
                }
                part = warp_sum_ll(part);
                if (lane == 0) sh_sum[wid] = part;
                __syncthreads();
                long long g = 0;
#pragma unroll
                for (int w = 0; w < kBlock / 32; ++w) g += sh_sum[w];
                C += (PM == P_BIT) ? g * s.p_common : g;
            } else {
                const long long rv = st.recv[j];
                __syncthreads();
                if (threadIdx.x == 0 && rv != 0) st.recv[j] = 0;
                if (open_prev) C += rv;
            }
            const int D = ds_next(dsv);
            if (threadIdx.x == 0) {
                if (C < 0 && !t_neg) {
                    t_neg = true;
                    neg_idx = j;
                    neg_val = C;
                }
                if (record & REC_CONFIGS) st.tr_cfg[slot * q + j] = C;
                if (record & REC_DELAYS) st.tr_dly[slot * q + j] = D;
                t_closed |= D != 0;
            }
            int r = -1;
            if (sel && D == 0) {
                if (threadIdx.x == 0) {
                    sh_pick = -1;
                    stat[ST_OPEN] += 1;
                }
                __syncthreads();
                if (policy == 0) {
                    if (threadIdx.x < 32) {
                        const int x = heavy_first_applicable_warp(s, h, C, lane);
                        if (lane == 0) sh_pick = x < 0 ? -1 : (int)(r0 + x);
                    }
                    __syncthreads();
                    r = sh_pick;
                    if (threadIdx.x == 0) stat[ST_SCANNED] += (r >= 0) ? (uint32_t)r - r0 + 1 : r1 - r0;
                } else {
                    uint32_t total = 0;
                    for (uint32_t base = r0; base < r1; base += kBlock) {
                        const uint32_t t = base + threadIdx.x;
                        total += __syncthreads_count(t < r1 && guard_ok(rule_guard_word(s.rw, WIDE, t), C));
                    }
                    if (threadIdx.x == 0) stat[ST_SCANNED] += r1 - r0;
                    if (total) {
                        uint32_t want = (uint32_t)(mix64(seed, k, j) % total);
                        for (uint32_t base = r0; base < r1; base += kBlock) {
                            const uint32_t t = base + threadIdx.x;
                            const bool ok = t < r1 && guard_ok(rule_guard_word(s.rw, WIDE, t), C);
                            const uint32_t c = __syncthreads_count(ok);
                            if (want < c) {
                                const unsigned int b = __ballot_sync(0xffffffffu, ok);
                                if (lane == 0) sh_cnt[wid] = __popc(b);
                                __syncthreads();
                                uint32_t before = 0;
                                for (int w = 0; w < wid; ++w) before += sh_cnt[w];
                                const uint32_t rank = before + __popc(b & ((1u << lane) - 1u));
                                if (ok && rank == want) sh_pick = (int)t;
                                __syncthreads();
                                break;
                            }
                            want -= c;
                        }
                        r = sh_pick;
                    }
                }
            }
            if (threadIdx.x == 0) {
                int nds = D;
                long long Cn = C;
                long long pval = 0;
                if (r >= 0) {
                    const uint4 wr = load_rule<WIDE>(s.rw, r);
                    if (CONSUME) Cn -= (long long)wr.y;
                    pval = (long long)wr.z;
                    nds = -((int)wr.w + 1);
                    t_fired = true;
                    stat[ST_FIRED] += 1;
                    if (pval > 0) {
                        stat[ST_SENDING] += 1;
                        if (stats_on) {
                            const uint32_t od = __ldg(s.outdeg + j);
                            stat[ST_ROWS] += od + (od < (uint32_t)s.z ? 1u : 0u);
                        }
                    }
                    if (FLIST) {
                        unsigned int pos = atomicAdd(&ctl->list_count[k & 1], 1u);
                        pick2(st.list, k)[pos] = (uint32_t)r;
                    }
                }
                st.cfg[j] = Cn;
                st.ds[j] = nds;
                if (sel) {
                    if (KIND == RECV_ARRAY) st.chosen[j] = r;
                    if (record & REC_SPIKING) st.tr_chosen[slot * q + j] = r;
                    if (KIND == RECV_PULL) {
                        if (PM == P_BIT) {
                            if (pval > 0) atomicOr(Pcur + (j >> 5), 1u << (j & 31));
                        } else if (PM == P_U8) {
                            reinterpret_cast<uint8_t*>(Pcur)[j] = (uint8_t)pval;
                        } else if (PM == P_U16) {
                            reinterpret_cast<uint16_t*>(Pcur)[j] = (uint16_t)pval;
                        } else {
                            Pcur[j] = (uint32_t)pval;
                        }
                    }
                }
            }
        }
    }

    if (stats_on) flush_stats(ctl, stat);
    const bool bf = __syncthreads_or(t_fired);
    const bool bc = __syncthreads_or(t_closed);
    // negative: smallest index within the block
    __shared__ long long sh_neg_idx, sh_neg_val;
    if (threadIdx.x == 0) sh_neg_idx = 0x7fffffffffffffffll;
    __syncthreads();
    if (t_neg) atomicMin(&sh_neg_idx, neg_idx);
    __syncthreads();
    if (t_neg && sh_neg_idx == neg_idx) sh_neg_val = neg_val;
    const bool bn = __syncthreads_or(t_neg);
    if (threadIdx.x == 0) finish_step(ctl, k, sel, bf, bc, bn, sh_neg_idx, bn ? sh_neg_val : 0);
}

// ---------------------------------------------------------------------------
// TMA bulk-copy pipeline helpers (cp.async.bulk + mbarrier, sm_90+/sm_100a).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
// Producer-side wait: plain try_wait polling (no suspend hint) so the single
// TMA-issuing thread reacts to a freed stage without a wake-up delay.
#ifndef SNP_PRODUCER_POLL
#define SNP_PRODUCER_POLL 0
#endif
__device__ __forceinline__ void mbar_wait_poll(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITP_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITP_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// L2 prefetch of a global range (no smem destination, no completion):
// pulls a future ring stage's HBM bytes into L2 ahead of its TMA copy.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier over the consumer warps only (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Tiled pull step kernel (default for COMPRESSED).
//
// A CTA owns tiles of `s.tile` consecutive destinations (a whole number of
// rounds over the 148 CTAs).  A tile's in-edges are stored sorted by source
// and cut into 256-edge segments whose sources span < 2^kSrcBits (host or
// device build: build_tiles / build_tiles_device), one 32-bit word per edge =
// slot << kSrcBits | (src - seg_base).  Warp-specialised: one producer warp
// streams everything the tile needs from HBM through an s.ring-deep ring of
// kStageBytes stages in shared memory (cp.async.bulk, full/empty mbarriers);
// the consumer warps never wait on each other except at the phase
// boundaries of a tile:
//   phase 1 stages: as many segments as fit with the P_{k-1} window their
//     sources span (sorted sources make it contiguous); segments go to the
//     consumer warps round-robin across stages, lane l takes edges l, l+32,
//     ..., looks the source bit up in the staged window and adds it to the
//     destination's 8/16/32-bit counter in shared memory (one red.shared);
//   phase 2 stages: kSub destinations' Ĉ, delay state (rule offsets) and
//     rule words; each consumer thread finishes step k-1 and selects step k
//     for one destination (lean instance: branch-free over <= 4 tiny rules).
// Phase 3 selects for the tile's heavy-rule neurons (> 32 rules): a guard
// index for FirstApplicable, block-wide counts for SeededRandom.  The ring
// spans tiles, so the next tile's first stages are in flight while phases
// 2 and 3 finish.  DESIGN.md ("Tiled pull") has the measurements behind
// each choice.

constexpr int kMaxRing = 8;  // ring stages (runtime s.ring <= kMaxRing, chosen by the host)
constexpr int kWarpsC = kTileThreads / 32;              // consumer warps
#ifndef SNP_STAGE_KB
#define SNP_STAGE_KB 48
#endif
constexpr uint32_t kStageBytes = SNP_STAGE_KB * 1024u;  // one ring stage
constexpr uint32_t kHdrBytes = 512;                     // stage header (+ segment bases)
constexpr uint32_t kMaxSegPerStage = (kHdrBytes - 32) / 4;
#ifndef SNP_P2_REP
#define SNP_P2_REP 1
#endif
constexpr int kP2Rep = SNP_P2_REP;                       // phase-2 destinations per consumer thread
constexpr int kSub = kTileThreads * kP2Rep;             // destinations per phase-2 stage
#ifndef SNP_SEG_SPLIT
#define SNP_SEG_SPLIT 1
#endif
constexpr uint32_t kSegSplit = SNP_SEG_SPLIT;               // phase-1 work units per segment
constexpr int kEpl = 8 / SNP_SEG_SPLIT;                      // edges per lane per work unit

// Stage header, written by the producer thread with st.shared before the
// mbarrier arrive (release), read by consumers after the wait (acquire).
struct StageHdr {
    uint32_t kind;     // 1 = phase-1 (segments), 2 = phase-2 (destinations)
    uint32_t last;     // last stage of its phase for this tile
    uint32_t first;    // phase 1: first segment; phase 2: first destination (tile index)
    uint32_t n;        // segments / destinations in the stage
    uint32_t src0;     // phase 1: first source bit of the staged P window (multiple of 128)
    uint32_t pstaged;  // phase 1: P window staged in smem
    uint32_t r_al;     // phase 2: rule index of the first staged rule word
    uint32_t rstaged;  // phase 2: rule words staged in smem
    uint32_t bases[kMaxSegPerStage];  // phase 1: segment base sources
};
static_assert(sizeof(StageHdr) <= kHdrBytes, "header fits");

// Stage payload offsets (from the stage start)
constexpr uint32_t kPayload = kHdrBytes;
// Phase-2 stages use one fixed layout whatever their destination count n <=
// kSub (payload-relative): Ĉ int64[kSub] at 0, delay state int32[kSub] at
// kP2Ds, rule offsets u32[kSub + 1] at kP2Roff (irregular systems only), rule
// words at kP2Rules(rpn) -- constant addresses for the consumers.
constexpr uint32_t kP2Ds = (uint32_t)kSub * 8u;
constexpr uint32_t kP2Roff = (uint32_t)kSub * 12u;
__host__ __device__ constexpr uint32_t kP2Rules(bool regular) {
    return regular ? kP2Roff : kP2Roff + ((((uint32_t)kSub + 1u) * 4u + 15u) & ~15u);
}
static_assert(kP2Ds % 16 == 0 && kP2Roff % 16 == 0, "16-byte aligned bulk-copy destinations");

__device__ __forceinline__ uint32_t round16(uint32_t x) { return (x + 15u) & ~15u; }

// Phase-1 accumulation of one edge word (slot << 17 | offset) into the
// tile's counters at shared address acc_s: 32-bit counters at slot * 4, or
// 16-bit halves (word slot >> 1, half slot & 1).
template <int CB>
__device__ __forceinline__ void tile_acc_add(uint32_t acc_s, uint32_t w, uint32_t v) {
    if (CB == 16) {
        // word (slot >> 1) at byte (slot >> 1) * 4, half (slot & 1) * 16
        asm volatile(
            "{\n.reg .b32 t, a, h, x;\n"
            "and.b32 t, %0, %3;\n"
            "shr.u32 t, t, %4;\n"
            "add.u32 a, %1, t;\n"
            "shr.u32 h, %0, %5;\n"
            "and.b32 h, h, 16;\n"
            "shl.b32 x, %2, h;\n"
            "red.shared.add.u32 [a], x;\n}" ::"r"(w), "r"(acc_s), "r"(v), "n"(~((2u << kSrcBits) - 1u)),
            "n"(kSrcBits - 1), "n"(kSrcBits - 4) : "memory");
    } else if (CB == 8) {
        // word (slot >> 2) at byte (slot >> 2) * 4, byte (slot & 3) * 8
        asm volatile(
            "{\n.reg .b32 t, a, h, x;\n"
            "and.b32 t, %0, %3;\n"
            "shr.u32 t, t, %4;\n"
            "add.u32 a, %1, t;\n"
            "shr.u32 h, %0, %5;\n"
            "and.b32 h, h, 24;\n"
            "shl.b32 x, %2, h;\n"
            "red.shared.add.u32 [a], x;\n}" ::"r"(w), "r"(acc_s), "r"(v), "n"(~((4u << kSrcBits) - 1u)),
            "n"(kSrcBits), "n"(kSrcBits - 3) : "memory");
    } else {
        asm volatile(
            "{\n.reg .b32 t, a;\n"
            "and.b32 t, %0, %3;\n"
            "shr.u32 t, t, %4;\n"
            "add.u32 a, %1, t;\n"
            "red.shared.add.u32 [a], %2;\n}" ::"r"(w), "r"(acc_s), "r"(v), "n"(~((1u << kSrcBits) - 1u)),
            "n"(kSrcBits - 2) : "memory");
    }
}

// Two-pass phase 1: add v to the counter of a plain slot index.
template <int CB>
__device__ __forceinline__ void tile_acc_add_slot(uint32_t acc_s, uint32_t slot, uint32_t v) {
    if (CB == 16) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + ((slot >> 1) << 2)), "r"(v << ((slot & 1u) << 4))
                     : "memory");
    } else if (CB == 8) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + ((slot >> 2) << 2)), "r"(v << ((slot & 3u) << 3))
                     : "memory");
    } else {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + (slot << 2)), "r"(v) : "memory");
    }
}

// Counter of destination i (phase 2).
template <int CB>
__device__ __forceinline__ uint32_t tile_acc_get(const uint32_t* acc, int i) {
    if (CB == 16) return (acc[i >> 1] >> ((i & 1) << 4)) & 0xffffu;
    if (CB == 8) return (acc[i >> 2] >> ((i & 3) << 3)) & 0xffu;
    return acc[i];
}

// Shared 32-bit words holding the per-destination counters of a tile of T
// destinations plus the dummy slot T that padding edges accumulate into.
template <int CB>
__host__ __device__ constexpr int acc_words(int T) { return CB == 8 ? (T + 4) / 4 : (CB == 16 ? (T + 2) / 2 : T + 1); }

// Stage descriptor (built on the host, build_tiles): 32 bytes.
//   phase 1: {1 | last << 8, first segment, n segments, src0, P bytes, bases offset, 0, 0}
//   phase 2: {2 | last << 8, first destination, n, r_al, rule bytes (0 = not staged), 0, 0, 0}
struct StageDesc {
    uint4 a, b;
};

// CB: bits per destination counter (32, 16 or 8; 16/8-bit counters are
// packed 2/4 per 32-bit word), the narrowest the host can prove no
// destination overflows in one step; smaller counters leave shared memory
// for larger tiles and a deeper ring.
// LEAN: no trace recording and no traffic counters (compiled out; the host
// launches this instance only for runs with record == 0 and stats off).
template <int PM, int RW, int CB, bool LEAN>
__global__ void __launch_bounds__(kTileThreads + 32, 1) tiled_step_kernel(const __grid_constant__ DevSys s, DevState st) {
    constexpr bool WIDE = RW == RW_WIDE;
    constexpr bool TINY = RW == RW_TINY;
    extern __shared__ __align__(128) uint8_t smem[];
    const int nst = s.ring;                                                   // ring stages
    uint8_t* ring = smem;                                                     // nst x kStageBytes
    uint32_t* acc = reinterpret_cast<uint32_t*>(smem + nst * kStageBytes);    // [acc_words(tile)]
    __shared__ __align__(8) uint64_t full_bar[kMaxRing];
    __shared__ __align__(8) uint64_t empty_bar[kMaxRing];
    __shared__ __align__(16) StageDesc desc_s[32];
    Ctrl* ctl = st.ctrl;
    // launched with programmatic stream serialization: wait for the previous
    // step's grid to complete (and its writes to be visible) before reading
    // anything it wrote; the next step's grid may be scheduled right away
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // one parallel snapshot of the run-control block: every field the
    // prologue needs arrives in one round trip instead of a chain of
    // volatile loads per thread (K2's ncu: ~19 % of stall samples sat on
    // the prologue's Ctrl reads)
    __shared__ __align__(16) uint32_t ctl_w[(sizeof(Ctrl) + 3) / 4];
    for (int i = threadIdx.x; i < (int)((sizeof(Ctrl) + 3) / 4); i += blockDim.x)
        ctl_w[i] = reinterpret_cast<const volatile uint32_t*>(ctl)[i];
    __syncthreads();
    const Ctrl* cs = reinterpret_cast<const Ctrl*>(ctl_w);
    const int halted = cs->halted;
    const long long k = cs->step;
    if (halted || k >= cs->stop_at) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->push_armed = 0;
        return;
    }
    if (s.p2p && k > 0) {
        // peer exchange: every rank's step k-1 must be in this rank's slot
        __shared__ int x_ok;
        if (threadIdx.x == 0) x_ok = wait_peers(s, cs->epoch, k - 1) ? 1 : 0;
        __syncthreads();
        if (!x_ok) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                ctl->halted = 1;
                ctl->reason = HALT_EXCHANGE;
            }
            return;
        }
    }
    if (s.x_stride && k > 0) {
        // row partition: halting decision for step k-1 from every rank's flags
        // (all-gathered with P_{k-1}); identical on every rank
        const volatile uint32_t* Pg = pick3(st.P, (k + 2) % 3);
        uint32_t f = 0, c = 0, n = 0;
        for (int r = 0; r < s.world; ++r) {
            const volatile uint32_t* h = Pg + (long long)r * s.x_stride + s.x_stride - 4;
            f |= h[0];
            c |= h[1];
            n |= h[2];
        }
        // step k-1 had no selection (k-1 == max_steps): STEP_LIMIT unless a
        // rank saw a negative count when finishing step k-2
        const bool last = k - 1 >= cs->max_steps;
        if (n || last || (!f && !c)) {
            // the LAST CTA to get here publishes the halt: a CTA of this grid
            // that starts late reads Ctrl.halted / Ctrl.step at its top, so an
            // early writer could hand it step k-1 and a stray step
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(&ctl->blocks_done, 1u) == gridDim.x - 1) {
                    ctl->halted = 1;
                    ctl->reason = n ? HALT_NEGATIVE : (last ? HALT_STEP_LIMIT : HALT_NO_APPLICABLE);
                    if (!n) ctl->step = k - 1;
                    ctl->neg_any = n ? 1 : 0;
                    ctl->push_armed = 0;
                    ctl->blocks_done = 0;
                    __threadfence();
                }
            }
            return;
        }
    }
    const bool sel = k < cs->max_steps;
    const int policy = cs->policy;
    const unsigned long long seed = cs->seed;
    const int record = LEAN ? 0 : cs->record;
    const bool stats_on = LEAN ? false : cs->stats_on != 0;
    const long long slot = k - cs->trace_base;
    const uint32_t* __restrict__ Pprev = pick3(st.P, (k + 2) % 3);
    uint32_t* Pcur = pick3(st.P, k % 3);
    uint32_t* Pzero = pick3(st.P, (k + 1) % 3);
    const long long q = s.q;
    const StepCtx cx{k, slot, q, seed, Pcur, policy, record, sel, stats_on};
    const int T = s.tile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    using Raw = typename RuleRaw<WIDE>::T;

    unsigned int stat[ST_COUNT];
#pragma unroll
    for (int i = 0; i < ST_COUNT; ++i) stat[i] = 0;
    bool t_fired = false, t_closed = false, t_neg = false;
    long long neg_idx = 0x7fffffffffffffffll, neg_val = 0;

    if (threadIdx.x == 0) {
        for (int b = 0; b < nst; ++b) {
            mbar_init(&full_bar[b], 1);
            mbar_init(&empty_bar[b], kWarpsC);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kWarpsC) {
        // ================= producer warp: descriptors 32 at a time, lane 0 issues the TMA copies
        // P_{k-1} arrived through generic-proxy stores (this GPU's or peers');
        // order them before the bulk (async-proxy) reads of the P windows
        if (s.p2p) asm volatile("fence.proxy.async.global;" ::: "memory");
        int pb = 0;           // next ring stage to fill
        uint32_t pround = 0;  // completed passes over the ring
        const uint32_t rw_size = TINY ? 4u : (WIDE ? 16u : 8u);
        const uint8_t* rw_src = TINY ? reinterpret_cast<const uint8_t*>(s.rw4) : reinterpret_cast<const uint8_t*>(s.rw);
        // L2 prefetch cursor: s.pf stages ahead of the TMA ring, across this
        // CTA's tiles, so the ring's copies hit L2 instead of waiting on HBM
        long long pt = blockIdx.x;
        uint32_t pi = 0, pe = 0;
        if (pt < s.n_tiles) pi = __ldg(s.tstage + pt), pe = __ldg(s.tstage + pt + 1);
        auto prefetch_next = [&]() {
            if (pt >= s.n_tiles) return;
            const uint4 da = __ldg(&s.stages[pi].a), db = __ldg(&s.stages[pi].b);
            const uint32_t n = da.z;
            if ((da.x & 0xff) == 1) {
                if (n) bulk_prefetch_l2(s.seg_words + (size_t)da.y * kSegEdges, n * kSegEdges * 4u);
            } else {
                const long long j0 = pt * T + da.y;
                bulk_prefetch_l2(st.cfg + j0, round16(n * 8u));
                bulk_prefetch_l2(st.ds + j0, round16(n * 4u));
                if (db.x) bulk_prefetch_l2(rw_src + (size_t)da.w * rw_size, db.x);
            }
            if (++pi == pe) {
                pt += gridDim.x;
                if (pt < s.n_tiles) pi = __ldg(s.tstage + pt), pe = __ldg(s.tstage + pt + 1);
            }
        };
        if (lane == 0)
            for (int i = 0; i < s.pf; ++i) prefetch_next();
        for (long long tile = blockIdx.x; tile < s.n_tiles; tile += gridDim.x) {
            const long long d0 = tile * T;
            const uint32_t s0 = __ldg(s.tstage + tile), s1 = __ldg(s.tstage + tile + 1);
            for (uint32_t base = s0; base < s1; base += 32) {
                // the warp loads 32 descriptors (coalesced) into shared memory;
                // lane 0 alone walks them, so there is one warp sync per batch
                const uint32_t cnt = min(32u, s1 - base);
                if (lane < cnt) {
                    desc_s[lane].a = __ldg(&s.stages[base + lane].a);
                    desc_s[lane].b = __ldg(&s.stages[base + lane].b);
                }
                __syncwarp();
                if (lane == 0) {
                    for (uint32_t i = 0; i < cnt; ++i) {
                        const uint4 da = desc_s[i].a, db = desc_s[i].b;
                        const uint32_t kind = da.x, first = da.y, n = da.z, f3 = da.w, f4 = db.x, f5 = db.y;
                        if (s.pf) prefetch_next();
                        const int b = pb;
                        if (pround > 0) {
                            if (SNP_PRODUCER_POLL) mbar_wait_poll(&empty_bar[b], (pround - 1) & 1u);
                            else mbar_wait(&empty_bar[b], (pround - 1) & 1u);
                        }
                        if (++pb == nst) {
                            pb = 0;
                            ++pround;
                        }
                        fence_proxy_async_smem();
                        uint8_t* buf = ring + b * kStageBytes;
                        StageHdr* h = reinterpret_cast<StageHdr*>(buf);
                        h->kind = kind & 0xff;
                        h->last = kind >> 8;
                        h->first = first;
                        h->n = n;
                        if (k == 0 && (kind & 0xff) != 2) {
                            // step 0: nothing was emitted before it (P_{-1} = 0), so
                            // the receive stages are not streamed; consumers see n = 0
                            h->n = 0;
                            mbar_expect_tx(&full_bar[b], 0);
                        } else if ((kind & 0xff) == 3) {
                            // two-pass phase 1: first = group, n groups; slots + edge bits
                            const uint32_t sbytes = n * 64u, ga = first & ~3u, bbytes = round16((n + (first & 3u)) * 4u);
                            h->src0 = first & 3u;
                            if (n) {
                                mbar_expect_tx(&full_bar[b], sbytes + bbytes);
                                bulk_g2s(buf + kPayload, s.tp_slots + (size_t)first * 32, sbytes, &full_bar[b]);
                                bulk_g2s(buf + kPayload + sbytes, s.tp_bits + ga, bbytes, &full_bar[b]);
                            } else {
                                mbar_expect_tx(&full_bar[b], 0);  // empty stage: the arrival alone completes it
                            }
                        } else if ((kind & 0xff) == 1) {
                            // f3 = src0, f4 = P bytes, f5 = bases offset
                            const uint32_t wbytes = n * kSegEdges * 4u, bbytes = round16(n * 4u);
                            h->src0 = f3;
                            h->pstaged = f4 ? 1u : 0u;
                            mbar_expect_tx(&full_bar[b], wbytes + f4 + bbytes);
                            if (n) {
                                bulk_g2s(h->bases, s.stage_bases + f5, bbytes, &full_bar[b]);
                                bulk_g2s(buf + kPayload, s.seg_words + (size_t)first * kSegEdges, wbytes, &full_bar[b]);
                            }
                            if (f4) bulk_g2s(buf + kPayload + wbytes, Pprev + (f3 >> 5), f4, &full_bar[b]);
                        } else {
                            // f3 = r_al, f4 = staged rule bytes
                            const long long j0 = d0 + first;
                            const uint32_t b_cfg = round16(n * 8u), b_ds = round16(n * 4u),
                                           b_roff = s.rpn ? 0u : round16((n + 1u) * 4u);
                            h->r_al = f3;
                            h->rstaged = f4 ? 1u : 0u;
                            mbar_expect_tx(&full_bar[b], b_cfg + b_ds + b_roff + f4);
                            bulk_g2s(buf + kPayload, st.cfg + j0, b_cfg, &full_bar[b]);
                            bulk_g2s(buf + kPayload + kP2Ds, st.ds + j0, b_ds, &full_bar[b]);
                            if (b_roff) bulk_g2s(buf + kPayload + kP2Roff, s.roff + j0, b_roff, &full_bar[b]);
                            if (f4)
                                bulk_g2s(buf + kPayload + kP2Rules(s.rpn != 0),
                                         rw_src + (size_t)f3 * rw_size, f4, &full_bar[b]);
                        }
                    }
                }
                __syncwarp();
            }
        }
    } else {
        // ================= consumer warps
        int cb = 0;           // next ring stage to consume
        uint32_t cround = 0;  // completed passes over the ring
        // phase-1 segments go to the consumer warps round-robin across stages
        // (a stage's first segment goes to the warp after the one that took
        // the previous stage's last), so stages holding fewer segments than
        // there are warps -- sparse P windows -- still keep every warp busy
        uint32_t rot = 0;
        for (long long tile = blockIdx.x; tile < s.n_tiles; tile += gridDim.x) {
            const long long d0 = tile * T;
            const int nd = (int)min((long long)T, q - d0);
            for (int i = threadIdx.x; i < acc_words<CB>(T); i += kTileThreads) acc[i] = 0;
            consumer_sync(kTileThreads);

            // ---- phase 1: receive sums
            for (;;) {
                const int b = cb;
                const uint8_t* buf = ring + b * kStageBytes;
                mbar_wait(&full_bar[b], cround & 1u);
                if (++cb == nst) {
                    cb = 0;
                    ++cround;
                }
                const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
                const uint32_t n = h->n, last = h->last, src0 = h->src0;
                if (h->kind == 3) {
                    // two-pass: 32 edges per group = 32 slots + one word of edge bits
                    const uint16_t* sl = reinterpret_cast<const uint16_t*>(buf + kPayload);
                    const uint32_t* bw = reinterpret_cast<const uint32_t*>(buf + kPayload + n * 64u) + src0;
                    const uint32_t acc_s = smem_u32(acc);
                    const uint32_t groups = (s.dbg & 1) ? 0u : n;
                    uint32_t i = warp;
                    for (; i + 3u * kWarpsC < groups; i += 4u * kWarpsC) {
                        uint32_t sv[4], bv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            sv[u] = sl[(i + u * kWarpsC) * 32u + lane];
                            bv[u] = (bw[i + u * kWarpsC] >> lane) & 1u;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) tile_acc_add_slot<CB>(acc_s, sv[u], bv[u]);
                        if (stats_on) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) stat[ST_EDGES] += sv[u] != (uint32_t)T;
                        }
                    }
                    for (; i < groups; i += kWarpsC) {
                        const uint32_t sv = sl[i * 32u + lane];
                        tile_acc_add_slot<CB>(acc_s, sv, (bw[i] >> lane) & 1u);
                        if (stats_on) stat[ST_EDGES] += sv != (uint32_t)T;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[b]);
                    if (last) break;
                    continue;
                }
                const bool pst = h->pstaged != 0;
                const uint32_t* ps = reinterpret_cast<const uint32_t*>(buf + kPayload + n * kSegEdges * 4u);
                // work unit: 1/kSegSplit of a segment (kEpl edges per lane), so the
                // stage's segments spread over all consumer warps.  A warp releases
                // the stage as soon as its last unit's words and P bits are in
                // registers; the shared atomics into the counters come after.
                bool released = false;
                const uint32_t units = (s.dbg & 1) ? 0u : n * kSegSplit;
                const uint32_t c0 = ((uint32_t)warp + kWarpsC - rot) % kWarpsC;
                rot = (rot + units) % kWarpsC;
                for (uint32_t c = c0; c < units; c += kWarpsC) {
                    const uint32_t i = c / kSegSplit, part = c % kSegSplit;
                    // lane l takes edges l, l+32, ...: each instruction covers 32
                    // consecutive (source-sorted) edges, so the P-bit loads hit
                    // nearly consecutive words -- conflict-free shared loads.
                    // Padding edges are (0, slot T): a real lookup into the
                    // dummy counter, so the loop has no branches.
                    const uint32_t base = h->bases[i];
                    const uint32_t* wp = reinterpret_cast<const uint32_t*>(buf + kPayload + i * kSegEdges * 4u) +
                                         part * (kSegEdges / kSegSplit) + lane;
                    uint32_t w[kEpl], v[kEpl];
#pragma unroll
                    for (int e = 0; e < kEpl; ++e) w[e] = wp[e * 32];
                    // word = slot << 17 | source offset.  Segment bases and src0 are
                    // multiples of 32, so the offset's low 5 bits are the bit inside
                    // its P word.  Addresses are a mask and a shifted add each
                    // (LOP3 + LEA.HI, spelled in PTX so the pattern survives).
                    if (PM == P_BIT && pst) {
                        const uint32_t pseg = smem_u32(ps) + ((base - src0) >> 3);
#pragma unroll
                        for (int e = 0; e < kEpl; ++e) {
                            asm volatile(
                                "{\n.reg .b32 t, a, pw, r;\n"
                                "and.b32 t, %1, %2;\n"
                                "shr.u32 t, t, 3;\n"
                                "add.u32 a, %3, t;\n"
                                "ld.shared.u32 pw, [a];\n"
                                "shf.r.wrap.b32 r, pw, pw, %1;\n"
                                "and.b32 %0, r, 1;\n}"
                                : "=r"(v[e]) : "r"(w[e]), "n"(kSrcMask & ~31u), "r"(pseg) : "memory");
                        }
                    } else {
                        // P looked up in global memory (L1/L2): non-bit P, or
                        // windows not staged
#pragma unroll
                        for (int e = 0; e < kEpl; ++e) v[e] = (uint32_t)p_lookup<PM>(Pprev, base + (w[e] & kSrcMask));
                    }
                    if (c + kWarpsC >= units) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[b]);
                        released = true;
                    }
                    const uint32_t acc_s = smem_u32(acc);
#pragma unroll
                    for (int e = 0; e < kEpl; ++e) tile_acc_add<CB>(acc_s, w[e], v[e]);
                    if (stats_on) {
#pragma unroll
                        for (int e = 0; e < kEpl; ++e) stat[ST_EDGES] += ((w[e] >> kSrcBits) != (uint32_t)T);
                    }
                }
                if (!released) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[b]);
                }
                if (last) break;
            }
            consumer_sync(kTileThreads);  // acc complete

            // ---- phase 2: finish step k-1, select step k (one destination per thread)
            for (;;) {
                const int b = cb;
                const uint8_t* buf = ring + b * kStageBytes;
                mbar_wait(&full_bar[b], cround & 1u);
                if (++cb == nst) {
                    cb = 0;
                    ++cround;
                }
                const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
                const uint32_t n = h->n, last = h->last, first = h->first, r_al = h->r_al;
                const bool rstaged = h->rstaged != 0;  // staged words are tiny words when TINY
                const long long* cfg_s = reinterpret_cast<const long long*>(buf + kPayload);
                const int* ds_s = reinterpret_cast<const int*>(buf + kPayload + kP2Ds);
                const uint32_t* roff_s = reinterpret_cast<const uint32_t*>(buf + kPayload + kP2Roff);
                const Raw* rules_s = reinterpret_cast<const Raw*>(buf + kPayload + kP2Rules(s.rpn != 0));
                bool released = false;
                // kP2Rep destinations per consumer thread (li, li + kTileThreads, ...)
#pragma unroll 1
                for (int rep = 0; rep < kP2Rep; ++rep) {
                    const int li = threadIdx.x + rep * kTileThreads;
                    const int i = (int)first + li;
                    const long long j = d0 + i;
                    const bool active = li < (int)n;
                    uint32_t r0 = 0, r1 = 0;
                    long long Cprev = 0;
                    int dsv = 0;
                    if (active) {
                        // regular systems (s.rpn rules per neuron) have implicit offsets
                        r0 = s.rpn ? (uint32_t)(s.rpn * j) : roff_s[li];
                        r1 = s.rpn ? r0 + (uint32_t)s.rpn : roff_s[li + 1];
                        Cprev = cfg_s[li];
                        dsv = ds_s[li];
                    }
                    const uint32_t nr = r1 - r0;
                    const bool heavy = active && nr > kLightRules;
                    int r = -1;
                    long long pval = 0;
                    if (s.dbg & 2) {
                        // timing experiment only: skip phase-2 work
                    } else if (LEAN && !WIDE && rstaged && __all_sync(0xffffffffu, !active || nr <= 4u)) {
                        // lean fast path: <= 4 staged rule words per neuron, branch-free
                        // selection; the stage is released once they are in registers
                        constexpr int kW = TINY ? 4 : 8;
                        alignas(16) uint32_t wv[kW];
                        if (active) {
                            const uint32_t* rp = reinterpret_cast<const uint32_t*>(
                                reinterpret_cast<const uint8_t*>(rules_s) + (r0 - r_al) * (TINY ? 4u : 8u));
    #pragma unroll
                            for (int x = 0; x < kW; ++x) wv[x] = rp[x];
                        }
                        if (kP2Rep == 1) {
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&empty_bar[b]);
                            released = true;
                        }
                        if (active) {
                            long long C = Cprev;
                            if (ds_open(dsv)) {
                                const uint32_t gsum = tile_acc_get<CB>(acc, i);
                                C += (PM == P_BIT) ? (long long)gsum * s.p_common : (long long)gsum;
                            }
                            const int D = ds_next(dsv);
                            pval = lean_commit4<PM, TINY>(s, st, ctl, cx, j, nr, wv, C, D, sel && D == 0, t_fired, t_closed,
                                                          t_neg);
                        }
                    } else if (active) {
                        const bool open_prev = ds_open(dsv);
                        const int D = ds_next(dsv);
                        const bool can_sel = sel && D == 0 && !heavy;
                        Raw w0{}, w1{}, w2{}, w3{};
                        if (can_sel) {
                            if (rstaged && !TINY) {
                                const Raw* rp = rules_s + (r0 - r_al);
                                if (nr > 0) w0 = rp[0];
                                if (nr > 1) w1 = rp[1];
                                if (nr > 2) w2 = rp[2];
                                if (nr > 3) w3 = rp[3];
                            } else {
                                if (nr > 0) w0 = load_raw<WIDE>(s.rw, r0);
                                if (nr > 1) w1 = load_raw<WIDE>(s.rw, r0 + 1);
                                if (nr > 2) w2 = load_raw<WIDE>(s.rw, r0 + 2);
                                if (nr > 3) w3 = load_raw<WIDE>(s.rw, r0 + 3);
                            }
                        }
                        long long C = Cprev;
                        if (open_prev) {
                            const uint32_t gsum = tile_acc_get<CB>(acc, i);
                            C += (PM == P_BIT) ? (long long)gsum * s.p_common : (long long)gsum;
                        }
                        pval = light_commit<RECV_PULL, PM, true, false, WIDE>(s, st, ctl, cx, j, r0, nr, w0, w1, w2, w3,
                                                                            C, D, can_sel, stat, t_fired, t_closed, t_neg,
                                                                            neg_idx, neg_val, r);
                    }
                    if (sel && PM == P_BIT) {
                        const unsigned int bits = __ballot_sync(0xffffffffu, pval > 0);
                        const unsigned int hv = __ballot_sync(0xffffffffu, heavy);
                        const unsigned int act = __ballot_sync(0xffffffffu, active);
                        if (lane == 0 && act) {
                            const long long wd = (j + s.xbase) >> 5;
                            Pzero[wd] = 0u;
                            if (hv) {
                                if (bits) atomicOr(Pcur + wd, bits);
                            } else {
                                Pcur[wd] = bits;
                            }
                        }
                    }
                }
                if (!released) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[b]);
                }
                if (last) break;
            }
            consumer_sync(kTileThreads);  // phase-2 commits visible; acc free after phase 3

            // ---- phase 3: heavy-rule neurons of this tile (> 32 rules, e.g. the
            // sorter's detectors), one warp each: FirstApplicable through the
            // guard index (32-ary warp search), SeededRandom by two warp scans
            const uint32_t h0 = __ldg(s.theavy + tile), h1 = __ldg(s.theavy + tile + 1);
            if (sel && h1 > h0) {
                for (uint32_t hh = h0 + warp; hh < h1; hh += (uint32_t)kWarpsC) {
                    const long long j = s.heavy[hh];
                    const int D = st.ds[j];  // phase 2 stored D_k (>= 0, not fired)
                    if (D != 0) continue;
                    const long long C = st.cfg[j];
                    const uint32_t r0 = __ldg(s.roff + j), r1 = __ldg(s.roff + j + 1);
                    int r;
                    if (policy == 0) {
                        const int x = heavy_first_applicable_warp(s, (int)hh, C, lane);
                        r = x < 0 ? -1 : (int)(r0 + x);
                        if (lane == 0) stat[ST_SCANNED] += (r >= 0) ? (uint32_t)r - r0 + 1 : r1 - r0;
                    } else {
                        const int x = heavy_seeded_table(s, (int)hh, C);
                        r = x == -2 ? heavy_seeded_warp<WIDE>(s, r0, r1, C, seed, k, j + s.gbase, lane)
                                    : (x < 0 ? -1 : (int)(r0 + x));
                        if (lane == 0) stat[ST_SCANNED] += r1 - r0;
                    }
                    if (lane == 0) {
                        stat[ST_OPEN] += 1;
                        if (r >= 0) {
                            const uint4 wr = load_rule<WIDE>(s.rw, r);
                            st.cfg[j] = C - (long long)wr.y;
                            st.ds[j] = -((int)wr.w + 1);
                            t_fired = true;
                            stat[ST_FIRED] += 1;
                            if (wr.z > 0) {
                                stat[ST_SENDING] += 1;
                                if (stats_on) {
                                    const uint32_t od = __ldg(s.outdeg + j);
                                    stat[ST_ROWS] += od + (od < (uint32_t)s.z ? 1u : 0u);
                                }
                            }
                            if (record & REC_SPIKING) st.tr_chosen[slot * q + j] = r;
                            const long long jx = j + s.xbase;
                            if (PM == P_BIT) {
                                if (wr.z > 0) atomicOr(Pcur + (jx >> 5), 1u << (jx & 31));
                            } else if (PM == P_U8) {
                                reinterpret_cast<uint8_t*>(Pcur)[jx] = (uint8_t)wr.z;
                            } else if (PM == P_U16) {
                                reinterpret_cast<uint16_t*>(Pcur)[jx] = (uint16_t)wr.z;
                            } else {
                                Pcur[jx] = wr.z;
                            }
                        }
                    }
                }
                consumer_sync(kTileThreads);
            }
            if (s.p2p && sel) {
                // peer exchange: this tile's final P words (phase 2 + 3) straight
                // into every peer's slot k % 3 -- NVLink stores that overlap the
                // next tile's phases
                constexpr int kPS = PM == P_BIT ? 5 : (PM == P_U8 ? 2 : (PM == P_U16 ? 1 : 0));  // log2 P per word
                const long long wb = (d0 + s.xbase) >> kPS, we = (d0 + nd + s.xbase + (1 << kPS) - 1) >> kPS;
                const int nw = (int)(we - wb);
                for (int i = threadIdx.x; i < nw * s.world; i += kTileThreads) {
                    const int r = i / nw, w = i - r * nw;
                    if (r != s.rank) peer_slot(s, r, k % 3)[wb + w] = __ldcg(Pcur + wb + w);
                }
            }
        }
    }

    if (stats_on) flush_stats(ctl, stat);
    if (s.dbg) t_fired = true;  // timing experiments: keep the run going
    const bool bf = __syncthreads_or(t_fired);
    const bool bc = __syncthreads_or(t_closed);
    __shared__ long long sh_neg_idx, sh_neg_val;
    if (threadIdx.x == 0) sh_neg_idx = 0x7fffffffffffffffll;
    __syncthreads();
    if (t_neg) atomicMin(&sh_neg_idx, neg_idx);
    __syncthreads();
    if (t_neg && sh_neg_idx == neg_idx) sh_neg_val = neg_val;
    const bool bn = __syncthreads_or(t_neg);
    if (threadIdx.x == 0)
        finish_step(ctl, k, sel, bf, bc, bn, sh_neg_idx, bn ? sh_neg_val : 0,
                    s.x_stride ? Pcur + (long long)s.rank * s.x_stride + s.x_stride - 4 : nullptr,
                    s.p2p ? &s : nullptr);
}

// ---------------------------------------------------------------------------
// The tiled kernel's instances live in their own translation units, one per
// P mode (snp_tiled.cu, compiled with -DSNP_TILED_PM=0..3 in parallel).
using TiledFn = void (*)(DevSys, DevState);
template <int PM>
void tiled_fns(int rw, int cb, TiledFn* step, TiledFn* lean);
template <> void tiled_fns<P_BIT>(int, int, TiledFn*, TiledFn*);
template <> void tiled_fns<P_U8>(int, int, TiledFn*, TiledFn*);
template <> void tiled_fns<P_U16>(int, int, TiledFn*, TiledFn*);
template <> void tiled_fns<P_U32>(int, int, TiledFn*, TiledFn*);

// Two-pass receive, pass 1 (variant TILED2): one CTA per source window.  The
// window's P_{k-1} bits (<= 2^17 sources, 16 KB) are read once into shared
// memory; each group of 32 in-edges (window order) becomes one word of edge
// bits, stored at its tile-order position for the tiled kernel's phase 1.
constexpr int kMaxWindowWords = (1 << 17) / 32;

#ifndef SNP_TEMPLATES_ONLY
__global__ void __launch_bounds__(512) pass1_kernel(const __grid_constant__ DevSys s, DevState st) {
    __shared__ uint32_t pw[kMaxWindowWords];
    __shared__ int x_ok;
    Ctrl* ctl = st.ctrl;
    const volatile Ctrl* vc = ctl;
    const long long k = vc->step;
    if (vc->halted || k >= vc->stop_at) return;
    if (s.p2p && k > 0) {
        if (threadIdx.x == 0) x_ok = wait_peers(s, vc->epoch, k - 1) ? 1 : 0;
        __syncthreads();
        if (!x_ok) return;  // the step kernel reports the timeout
    }
    const uint32_t* __restrict__ Pprev = pick3(st.P, (k + 2) % 3);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint32_t wwords = 1u << (s.tp_wlog - 5);
    // work items: (window, group range) -- windows split so that items
    // outnumber CTAs several times (balance)
    for (long long it = blockIdx.x; it < s.tp_nitems; it += gridDim.x) {
        const uint4 item = __ldg(s.tp_items + it);
        const uint32_t w = item.x, g0 = item.y, g1 = item.z;
        const uint32_t* src = Pprev + (size_t)w * wwords;
        for (uint32_t i = threadIdx.x; i < wwords; i += blockDim.x) pw[i] = __ldcg(src + i);
        __syncthreads();
        // a warp takes 8 groups (256 edges) per round, 4 rounds in flight:
        // lane l loads 16 bytes = 8 offsets of group l / 4, makes their 8 bits,
        // and 4 lanes OR their bytes into the group's word (lane 4j writes it)
        const uint32_t j = lane >> 2;
        for (uint32_t gb = g0 + 8u * warp; gb < g1; gb += 32u * nwarps) {
            uint4 o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t gu = gb + u * 8u * nwarps;
                o[u] = make_uint4(0, 0, 0, 0);
                if (gu + j < g1) o[u] = __ldg(reinterpret_cast<const uint4*>(s.tp_off + (size_t)gu * 32) + lane);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t gu = gb + u * 8u * nwarps;
                const uint32_t ov[4] = {o[u].x, o[u].y, o[u].z, o[u].w};
                uint32_t byte = 0;
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const uint32_t lo = ov[x] & 0xffffu, hi = ov[x] >> 16;
                    byte |= ((pw[lo >> 5] >> (lo & 31u)) & 1u) << (2 * x);
                    byte |= ((pw[hi >> 5] >> (hi & 31u)) & 1u) << (2 * x + 1);
                }
                uint32_t word = byte << ((lane & 3u) << 3);
                word |= __shfl_xor_sync(0xffffffffu, word, 1);
                word |= __shfl_xor_sync(0xffffffffu, word, 2);
                if ((lane & 3u) == 0 && gu + j < g1) s.tp_bits[__ldg(s.tp_gword + gu + j)] = word;
            }
        }
        __syncthreads();
    }
}
#endif  // SNP_TEMPLATES_ONLY

// ---------------------------------------------------------------------------
// Push scatter (paper Alg. 4 ELL / Alg. 5 Optimized) for step k = step-1.
// Thread per neuron; columns longer than kLightOut go to the heavy queue.

template <bool ELL>
__global__ void __launch_bounds__(kBlock) push_kernel(const __grid_constant__ DevSys s, DevState st, long long* row_visits) {
    Ctrl* ctl = st.ctrl;
    const volatile Ctrl* vc = ctl;
    if (!vc->push_armed) return;
    const long long k = vc->step - 1;
    const bool stats_on = vc->stats_on != 0;
    unsigned long long edges = 0;
    const long long j = (long long)blockIdx.x * kBlock + threadIdx.x;
    if (j < s.q) {
        const int r = st.chosen[j];
        if (r >= 0) {
            if (ELL) {
                const uint32_t len = __ldg(s.ell_len + r);
                if (row_visits) row_visits[r] += len + (len < (uint32_t)s.ell_rows ? 1 : 0);
                if (len <= kLightOut) {
                    const int2* col = s.ell + (long long)r * s.ell_ld;
                    for (uint32_t i = 0; i < len; ++i) {
                        const int2 pr = __ldg(col + i);
                        red_add_i64(st.recv + pr.x, pr.y);
                    }
                    edges += len;
                } else {
                    unsigned int pos = atomicAdd(&ctl->heavy_count[k & 1], 1u);
                    pick2(st.list, k)[pos] = (uint32_t)j;
                }
            } else {
                const int p = __ldg(s.rrec + r).y;
                if (p > 0) {
                    const uint32_t e0 = __ldg(s.soff + j), e1 = __ldg(s.soff + j + 1);
                    if (e1 - e0 <= kLightOut) {
                        for (uint32_t e = e0; e < e1; ++e) red_add_i64(st.recv + __ldg(s.sdst + e), p);
                        edges += e1 - e0;
                    } else {
                        unsigned int pos = atomicAdd(&ctl->heavy_count[k & 1], 1u);
                        pick2(st.list, k)[pos] = (uint32_t)j;
                    }
                }
            }
        }
    }
    if (stats_on) {
        edges = warp_sum_ll((long long)edges);
        if ((threadIdx.x & 31) == 0 && edges) atomicAdd(&ctl->stats[ST_EDGES], edges);
    }
}

// Warp per queued heavy column.
template <bool ELL>
__global__ void __launch_bounds__(kBlock) push_heavy_kernel(const __grid_constant__ DevSys s, DevState st) {
    Ctrl* ctl = st.ctrl;
    const volatile Ctrl* vc = ctl;
    if (!vc->push_armed) return;
    const long long k = vc->step - 1;
    const unsigned int n = vc->heavy_count[k & 1];
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (kBlock / 32);
    unsigned long long edges = 0;
    for (long long w = (long long)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); w < n; w += warps) {
        const uint32_t j = pick2(st.list, k)[w];
        const int r = st.chosen[j];
        if (ELL) {
            const uint32_t len = __ldg(s.ell_len + r);
            const int2* col = s.ell + (long long)r * s.ell_ld;
            for (uint32_t i = lane; i < len; i += 32) {
                const int2 pr = __ldg(col + i);
                red_add_i64(st.recv + pr.x, pr.y);
            }
            edges += len;
        } else {
            const int p = __ldg(s.rrec + r).y;
            const uint32_t e0 = __ldg(s.soff + j), e1 = __ldg(s.soff + j + 1);
            for (uint32_t e = e0 + lane; e < e1; e += 32) red_add_i64(st.recv + __ldg(s.sdst + e), p);
            edges += e1 - e0;
        }
    }
    if (vc->stats_on && lane == 0 && edges) atomicAdd(&ctl->stats[ST_EDGES], edges);
}

// ---------------------------------------------------------------------------
// Fused push step (runs of ELL / COMPRESSED-push systems whose neurons all
// have <= 32 rules): ONE kernel per step that finishes step k-1 from the
// receive buffer of parity k&1, selects step k's rules, and scatters the
// chosen columns into the buffer of parity (k+1)&1 -- paper Alg. 4 (ELL,
// engine.py:269-310) / Alg. 5 (Optimized push, engine.py:313-355).
//
// The column walk is warp-cooperative: the fired lanes' columns are laid end
// to end in 16-byte chunks (ELL: 2 (target, amount) pairs; Optimized: one
// 4-byte target per lane) and each round the 32 lanes take 32 consecutive
// chunks, finding their column by a branch-free binary search over the
// warp's inclusive chunk prefix.  Reads are coalesced 128-bit loads with an
// L2 evict-first hint (the columns are streamed once per step), so the
// receive buffers (int32 when no neuron can receive 2^31 per step) stay
// L2-resident for the RED.ADDs.  Row 0 of an ELL column is the owner's
// consumption (owner, -c): it travels through the receive buffer like any
// delivery and is gated by the owner's open flag at the destination, as in
// the reference walk.

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ int4 ld_stream16(const void* p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream4(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
template <bool R64>
__device__ __forceinline__ void recv_add(void* buf, int t, int v) {
    if (R64) atomicAdd(reinterpret_cast<unsigned long long*>(buf) + t, (unsigned long long)(long long)v);
    else atomicAdd(reinterpret_cast<int*>(buf) + t, v);
}

template <bool ELL, bool WIDE, bool R64>
__global__ void __launch_bounds__(kBlock, kStepMinBlocks) push_step_kernel(const __grid_constant__ DevSys s, DevState st) {
    Ctrl* ctl = st.ctrl;
    const volatile Ctrl* vc = ctl;
    const int halted = vc->halted;
    const long long k = vc->step;
    if (halted || k >= vc->stop_at) return;
    const bool sel = k < vc->max_steps;
    const int record = vc->record;
    const bool stats_on = vc->stats_on != 0;
    const long long q = s.q;
    const StepCtx cx{k, k - vc->trace_base, q, vc->seed, nullptr, vc->policy, record, sel, stats_on};
    void* rcur = (k & 1) ? st.rbuf[1] : st.rbuf[0];
    void* rnext = (k & 1) ? st.rbuf[0] : st.rbuf[1];
    const uint64_t pol = evict_first_policy();
    const int lane = threadIdx.x & 31;

    unsigned int stat[ST_COUNT];
#pragma unroll
    for (int i = 0; i < ST_COUNT; ++i) stat[i] = 0;
    bool t_fired = false, t_closed = false, t_neg = false;
    long long neg_idx = 0x7fffffffffffffffll, neg_val = 0;
    unsigned long long edges = 0;

    for (long long tile = blockIdx.x; tile < s.light_tiles; tile += gridDim.x) {
        const long long j = tile * kBlock + threadIdx.x;
        int r = -1;
        long long pval = 0;
        if (j < q) {
            const uint32_t r0 = __ldg(s.roff + j), nr = __ldg(s.roff + j + 1) - r0;
            const long long Cprev = st.cfg[j];
            const int dsv = st.ds[j];
            const bool open_prev = ds_open(dsv);
            const int D = ds_next(dsv);
            const bool can_sel = sel && D == 0;
            using Raw = typename RuleRaw<WIDE>::T;
            Raw w0{}, w1{}, w2{}, w3{};
            if (can_sel) {
                if (nr > 0) w0 = load_raw<WIDE>(s.rw, r0);
                if (nr > 1) w1 = load_raw<WIDE>(s.rw, r0 + 1);
                if (nr > 2) w2 = load_raw<WIDE>(s.rw, r0 + 2);
                if (nr > 3) w3 = load_raw<WIDE>(s.rw, r0 + 3);
            }
            long long rv;
            if (R64) {
                long long* b = reinterpret_cast<long long*>(rcur) + j;
                rv = *b;
                if (rv != 0) *b = 0;
            } else {
                int* b = reinterpret_cast<int*>(rcur) + j;
                rv = *b;
                if (rv != 0) *b = 0;
            }
            const long long C = Cprev + (open_prev ? rv : 0);
            // no chosen / P stores: the column is pushed right here
            pval = light_commit<RECV_PULL, P_BIT, !ELL, false, WIDE>(s, st, ctl, cx, j, r0, nr, w0, w1, w2, w3, C, D,
                                                                     can_sel, stat, t_fired, t_closed, t_neg, neg_idx,
                                                                     neg_val, r);
        }
        // this lane's column: chunk count and start
        uint32_t nch = 0, len = 0;
        long long base = 0;
        if (sel && r >= 0) {
            if (ELL) {
                len = __ldg(s.ell_len + r);
                nch = (len + 1) >> 1;
                base = (long long)r * s.ell_ld;  // in pairs (ell_ld even: 16-byte aligned)
            } else if (pval > 0) {
                const uint32_t e0 = __ldg(s.soff + j);
                len = __ldg(s.soff + j + 1) - e0;
                nch = len;
                base = e0;
            }
            edges += len;
        }
        uint32_t incl = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - nch;
        const int amount = (int)pval;
        for (uint32_t g0 = 0; g0 < total; g0 += 32) {
            const uint32_t g = g0 + lane;
            int L = 0;
#pragma unroll
            for (int w = 16; w > 0; w >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, L + w - 1);
                if (v <= g) L += w;
            }
            const uint32_t c = g - __shfl_sync(0xffffffffu, excl, L);
            const long long b = __shfl_sync(0xffffffffu, base, L);
            if (ELL) {
                const uint32_t ln = __shfl_sync(0xffffffffu, len, L);
                if (g < total) {
                    const int4 v = ld_stream16(s.ell + b + 2 * c, pol);
                    recv_add<R64>(rnext, v.x, v.y);
                    if (2 * c + 1 < ln) recv_add<R64>(rnext, v.z, v.w);
                }
            } else {
                const int a = __shfl_sync(0xffffffffu, amount, L);
                if (g < total) recv_add<R64>(rnext, (int)ld_stream4(s.sdst + b + c, pol), a);
            }
        }
    }

    if (stats_on) {
        stat[ST_EDGES] = (unsigned int)edges;
        flush_stats(ctl, stat);
    }
    const bool bf = __syncthreads_or(t_fired);
    const bool bc = __syncthreads_or(t_closed);
    __shared__ long long sh_neg_idx, sh_neg_val;
    if (threadIdx.x == 0) sh_neg_idx = 0x7fffffffffffffffll;
    __syncthreads();
    if (t_neg) atomicMin(&sh_neg_idx, neg_idx);
    __syncthreads();
    if (t_neg && sh_neg_idx == neg_idx) sh_neg_val = neg_val;
    const bool bn = __syncthreads_or(t_neg);
    if (threadIdx.x == 0) finish_step(ctl, k, sel, bf, bc, bn, sh_neg_idx, bn ? sh_neg_val : 0);
}

// ---------------------------------------------------------------------------
// Binned push step (runs of ELL / COMPRESSED-push systems, every neuron <= 32
// rules): the scatter of Alg. 4 / Alg. 5 without global atomics per pair.
// L2 RED.ADD tops out near 200 G ops/s on this B200 (tools/redbench.cu), i.e.
// ~0.9 ms for K3's 160 M deliveries, so deliveries are instead binned by
// destination tile through shared memory and accumulated by the tile's owner
// in the next step's kernel with shared-memory atomics.
//
// Destinations are cut into bin_ntiles tiles of bin_T.  One kernel per step k;
// a CTA owns tiles and for each tile:
//   A. receive: the tile's bin entries written during step k-1 (main region:
//      whole 16-byte units; overflow region: single entries) -> 8/16/32-bit
//      counters in shared memory;
//   B. for kBinThreads destinations at a time: finish step k-1 (C += open ? recv),
//      update delays, select step k (sv_calc), consume (row 0 of the ELL
//      column, applied at selection like COMPRESSED);
//   C. walk the fired neurons' columns (ELL rows 1.., 16-byte loads with an
//      L2 evict-first hint; Optimized: the out-adjacency) -- each lane its own
//      column when the warp's columns are of similar length, else 32 chunks at
//      a time over the warp's concatenated columns -- and stage each
//      delivery's entry (u16 slot when every delivery carries the same
//      amount, else u32 slot << 15 | amount) in a per-destination-tile bucket
//      of kCap entries in shared memory; a full bucket sends single entries to
//      the tile's overflow region;
//   D. every kWin chunks (and at the tile's end) each bucket is flushed to the
//      tile's main region with one reservation and 16-byte stores, padded to
//      whole 16-byte units with entries that add nothing (slot T, the dummy
//      counter / amount 0).
// The bins of step k are complete at the kernel boundary; kernel k+1 reads
// them.  Region sizes: main = the tile's in-degree sum + the padding of every
// possible flush, overflow = the in-degree sum (checked on every reservation).

#ifndef SNP_BIN_THREADS
#define SNP_BIN_THREADS 1024  // 32 warps (64 registers: no spills since the walks became separate
                              // instances); same box: K3 ELL 1.022 (768) -> 0.948 ms, push 0.932 -> 0.857
#endif
constexpr int kBinThreads = SNP_BIN_THREADS;
constexpr int kBinUnroll = 4;    // column chunks in flight per lane
#ifndef SNP_BIN_GUNROLL
#define SNP_BIN_GUNROLL 4
#endif
constexpr int kBinGUnroll = SNP_BIN_GUNROLL;  // ELL column-group passes in flight per warp

template <bool UNIT>
struct BinEntry {
    using T = uint32_t;
    static constexpr int kCap = 64;   // staged entries per destination tile
    static constexpr int kWin = 1;    // 1024-destination chunks per flush
    static constexpr int kVec = 4;    // entries per 16-byte unit
};
template <>
struct BinEntry<true> {
    using T = uint16_t;
#ifndef SNP_BIN_CAP
#define SNP_BIN_CAP 256
#endif
    static constexpr int kCap = SNP_BIN_CAP;
#ifndef SNP_BIN_WIN
#define SNP_BIN_WIN 4
#endif
    static constexpr int kWin = SNP_BIN_WIN;
    static constexpr int kVec = 8;
};
// flushes per step into one tile are at most ceil(q / (kBinThreads * kWin)) + ntiles
__host__ __device__ constexpr long long bin_flush_dests(bool unit) {
    return (long long)kBinThreads * (unit ? BinEntry<true>::kWin : BinEntry<false>::kWin);
}

template <int CB>
__host__ __device__ constexpr int bin_acc_words(int T) { return (acc_words<CB>(T) + 3) & ~3; }

// GROUP: ELL column-group walk only (uniform column stride <= 16 chunks);
// else lane-own / concatenated walks -- separate instances keep the register
// budget of each (1024 threads: 64 registers) for its own path
template <bool ELL, bool WIDE, bool UNIT, int CB, bool GROUP>
__global__ void __launch_bounds__(kBinThreads, 1) ell_bin_step_kernel(const __grid_constant__ DevSys s, DevState st) {
    using BE = BinEntry<UNIT>;
    using E = typename BE::T;
    constexpr int kCap = BE::kCap, kWin = BE::kWin, kVec = BE::kVec;
    constexpr uint32_t kEsz = sizeof(E);
    extern __shared__ __align__(128) uint8_t smem[];
    const int NT = s.bin_ntiles, T = s.bin_T;
    uint32_t* acc = reinterpret_cast<uint32_t*>(smem);
    uint32_t* cnt = acc + bin_acc_words<CB>(T);
    E* stage = reinterpret_cast<E*>(cnt + ((NT + 3) & ~3));
    Ctrl* ctl = st.ctrl;
    // one parallel snapshot of the run-control block (see tiled_step_kernel)
    __shared__ __align__(16) uint32_t ctl_w[(sizeof(Ctrl) + 3) / 4];
    for (int i = threadIdx.x; i < (int)((sizeof(Ctrl) + 3) / 4); i += blockDim.x)
        ctl_w[i] = reinterpret_cast<const volatile uint32_t*>(ctl)[i];
    __syncthreads();
    const Ctrl* cs = reinterpret_cast<const Ctrl*>(ctl_w);
    const int halted = cs->halted;
    const long long k = cs->step;
    if (halted || k >= cs->stop_at) return;
    const bool sel = k < cs->max_steps;
    const int record = cs->record;
    const bool stats_on = cs->stats_on != 0;
    const long long q = s.q;
    const StepCtx cx{k, k - cs->trace_base, q, cs->seed, nullptr, cs->policy, record, sel, stats_on};
    const E* __restrict__ bin_in = reinterpret_cast<const E*>((k & 1) ? st.bins[0] : st.bins[1]);
    E* bin_out = reinterpret_cast<E*>((k & 1) ? st.bins[1] : st.bins[0]);
    uint32_t* fill_in = (k & 1) ? st.bin_fill[0] : st.bin_fill[1];
    uint32_t* fill_out = (k & 1) ? st.bin_fill[1] : st.bin_fill[0];
    const uint64_t pol = evict_first_policy();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // shared-window addresses, computed once (the bucket code is per delivery)
    const uint32_t acc_s = smem_u32(acc), cnt_s = smem_u32(cnt), stage_s = smem_u32(stage);
    const unsigned long long magic = s.bin_magic;
    const E pad = UNIT ? (E)T : (E)0;  // adds to the dummy counter / adds 0
    // ELL column groups: cpc chunks per column, `per` columns per warp pass
    __shared__ uint32_t col_r[kBinThreads / 32][32];
    const uint32_t cpc = (ELL && GROUP) ? (uint32_t)s.bin_cpc : 0u;
    const uint32_t per = cpc ? 32u / cpc : 0u, sub = cpc ? (uint32_t)lane / cpc : 0u, cc = (uint32_t)lane - sub * cpc;

    unsigned int stat[ST_COUNT];
#pragma unroll
    for (int i = 0; i < ST_COUNT; ++i) stat[i] = 0;
    bool t_fired = false, t_closed = false, t_neg = false, t_over = false;
    long long neg_idx = 0x7fffffffffffffffll, neg_val = 0;
    unsigned long long edges = 0;

    for (int i = threadIdx.x; i < NT; i += kBinThreads) cnt[i] = 0;
    for (long long tile = blockIdx.x; tile < NT; tile += gridDim.x) {
        const long long d0 = tile * T;
        const int nd = (int)min((long long)T, q - d0);
        // ---- A. receive the deliveries of step k-1 into the tile's counters
        for (int i = threadIdx.x; i < acc_words<CB>(T); i += kBinThreads) acc[i] = 0;
        __syncthreads();
        if (k > 0) {
            const uint32_t nin = *(volatile uint32_t*)(fill_in + tile);  // whole 16-byte units
            const uint32_t nov = *(volatile uint32_t*)(fill_in + NT + tile);
            const uint4* src = reinterpret_cast<const uint4*>(bin_in + __ldg(s.bin_off + tile));
            const uint32_t nv = nin / kVec;
            for (uint32_t v = threadIdx.x; v < nv; v += kBinThreads) {
                const uint4 w = __ldcs(src + v);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    if (UNIT) {
                        tile_acc_add_slot<CB>(acc_s, ws[x] & 0xffffu, 1u);
                        tile_acc_add_slot<CB>(acc_s, ws[x] >> 16, 1u);
                    } else {
                        tile_acc_add_slot<CB>(acc_s, ws[x] >> 15, ws[x] & 0x7fffu);
                    }
                }
            }
            const E* osrc = bin_in + __ldg(s.bin_ooff + tile);
            for (uint32_t i = threadIdx.x; i < nov; i += kBinThreads) {
                const uint32_t e = osrc[i];
                if (UNIT) tile_acc_add_slot<CB>(acc_s, e, 1u);
                else tile_acc_add_slot<CB>(acc_s, e >> 15, e & 0x7fffu);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && k > 0) {  // the regions are refilled in step k+1
            fill_in[tile] = 0;
            fill_in[NT + tile] = 0;
        }
        // ---- B + C (+ D every kWin chunks), kBinThreads destinations at a time
        for (int c0 = 0, win = 0; c0 < nd; c0 += kBinThreads, ++win) {
            const int li = c0 + threadIdx.x;
            const long long j = d0 + li;
            int r = -1;
            long long pval = 0;
            if (li < nd) {
                const uint32_t r0 = __ldg(s.roff + j), nr = __ldg(s.roff + j + 1) - r0;
                const long long Cprev = st.cfg[j];
                const int dsv = st.ds[j];
                const bool open_prev = ds_open(dsv);
                const int D = ds_next(dsv);
                const bool can_sel = sel && D == 0;
                using Raw = typename RuleRaw<WIDE>::T;
                Raw w0{}, w1{}, w2{}, w3{};
                if (can_sel) {
                    if (nr > 0) w0 = load_raw<WIDE>(s.rw, r0);
                    if (nr > 1) w1 = load_raw<WIDE>(s.rw, r0 + 1);
                    if (nr > 2) w2 = load_raw<WIDE>(s.rw, r0 + 2);
                    if (nr > 3) w3 = load_raw<WIDE>(s.rw, r0 + 3);
                }
                long long C = Cprev;
                if (open_prev) {
                    const uint32_t g = tile_acc_get<CB>(acc, li);
                    C += UNIT ? (long long)g * s.bin_amount : (long long)g;
                }
                pval = light_commit<RECV_PULL, P_BIT, true, false, WIDE>(s, st, ctl, cx, j, r0, nr, w0, w1, w2, w3, C, D,
                                                                        can_sel, stat, t_fired, t_closed, t_neg,
                                                                        neg_idx, neg_val, r);
            }
            // this lane's column: chunks (ELL: 16-byte pairs of rows, row 0 =
            // consumption, already applied; Optimized: one target per lane)
            uint32_t nch = 0, len = 0;
            long long base = 0;
            if (GROUP) {
                // column groups read whole padded columns (padding pairs have
                // target -1), so the per-rule length array is not read
                nch = (sel && r >= 0) ? 1u : 0u;
            } else if (sel && r >= 0) {
                if (ELL) {
                    len = __ldg(s.ell_len + r);
                    nch = len > 1 ? (len + 1) >> 1 : 0u;
                    base = (long long)r * s.ell_ld;
                    edges += len > 0 ? len - 1 : 0;
                } else if (pval > 0) {
                    const uint32_t e0 = __ldg(s.soff + j);
                    len = __ldg(s.soff + j + 1) - e0;
                    nch = len;
                    base = e0;
                    edges += len;
                }
            }
            const int amount = (int)pval;
            auto deliver = [&](uint32_t t, uint32_t a) {
                const uint32_t dt = (uint32_t)__umul64hi((unsigned long long)t, magic);
                const uint32_t slot = t - dt * (uint32_t)T;
                const uint32_t e = UNIT ? slot : ((slot << 15) | a);
                uint32_t pos;
                asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(pos) : "r"(cnt_s + dt * 4u) : "memory");
                if (pos < (uint32_t)kCap) {
                    const uint32_t addr = stage_s + (dt * (uint32_t)kCap + pos) * kEsz;
                    if (UNIT) asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)e) : "memory");
                    else asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(e) : "memory");
                } else {  // bucket full: one entry to the tile's overflow region
                    const uint32_t g = atomicAdd(fill_out + NT + dt, 1u);
                    const uint32_t o = __ldg(s.bin_ooff + dt);
                    if (o + g < __ldg(s.bin_ooff + dt + 1)) bin_out[o + g] = (E)e;
                    else t_over = true;
                }
            };
            const uint32_t total = __reduce_add_sync(0xffffffffu, nch);
            const uint32_t mx = __reduce_max_sync(0xffffffffu, nch);
            if constexpr (ELL && GROUP) {
                // column groups: the warp's fired columns, compacted in shared
                // memory, `per` at a time; lane sub * cpc + cc reads chunk cc of
                // column sub, so each column is one contiguous 16 * cpc-byte read
                const uint32_t fm = __ballot_sync(0xffffffffu, nch > 0);
                const uint32_t nf = __popc(fm);
                if (nch > 0) col_r[warp][__popc(fm & ((1u << lane) - 1u))] = (uint32_t)r;
                __syncwarp();
                for (uint32_t i0 = 0; i0 < nf; i0 += per * kBinGUnroll) {
                    int4 v[kBinGUnroll];
#pragma unroll
                    for (int u = 0; u < kBinGUnroll; ++u) {
                        const uint32_t col = i0 + u * per + sub;
                        v[u] = make_int4(-1, 0, -1, 0);
                        if (sub < per && col < nf)
                            v[u] = ld_stream16(s.ell + (long long)col_r[warp][col] * s.ell_ld + 2 * cc, pol);
                    }
#pragma unroll
                    for (int u = 0; u < kBinGUnroll; ++u) {
                        if (cc > 0 && v[u].x >= 0) deliver((uint32_t)v[u].x, (uint32_t)v[u].y);  // row 0 = consumption
                        if (v[u].z >= 0) deliver((uint32_t)v[u].z, (uint32_t)v[u].w);
                        edges += (cc > 0 && v[u].x >= 0 ? 1u : 0u) + (v[u].z >= 0 ? 1u : 0u);
                    }
                }
                __syncwarp();
            } else {
            if (mx * 32u <= 2u * total) {
                // lane-own columns: lane l walks its column, kBinUnroll chunks in flight
                for (uint32_t cb0 = 0; cb0 < mx; cb0 += kBinUnroll) {
                    int4 v[kBinUnroll];
#pragma unroll
                    for (int u = 0; u < kBinUnroll; ++u) {
                        const uint32_t c = cb0 + u;
                        v[u] = make_int4(-1, 0, -1, 0);
                        if (c < nch) {  // L1-allocating: the lane reads the rest of the sector next
                            if (ELL) v[u] = __ldg(reinterpret_cast<const int4*>(s.ell + base + 2 * c));
                            else v[u].x = (int)__ldg(s.sdst + base + c);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kBinUnroll; ++u) {
                        const uint32_t c = cb0 + u;
                        if (c >= nch) continue;
                        if (ELL) {
                            if (c > 0) deliver((uint32_t)v[u].x, (uint32_t)v[u].y);  // row 2c (row 0 = consumption)
                            if (2 * c + 1 < len) deliver((uint32_t)v[u].z, (uint32_t)v[u].w);
                        } else {
                            deliver((uint32_t)v[u].x, (uint32_t)amount);
                        }
                    }
                }
            } else {
                // uneven columns: 32 chunks at a time over the warp's concatenated columns
                uint32_t incl = nch;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const uint32_t excl = incl - nch;
                for (uint32_t g0 = 0; g0 < total; g0 += 32 * kBinUnroll) {
                    int4 v[kBinUnroll];
                    uint32_t cc[kBinUnroll], ln[kBinUnroll];
                    int am[kBinUnroll];
#pragma unroll
                    for (int u = 0; u < kBinUnroll; ++u) {
                        const uint32_t g = g0 + u * 32 + lane;
                        int L = 0;
#pragma unroll
                        for (int w = 16; w > 0; w >>= 1) {
                            const uint32_t x = __shfl_sync(0xffffffffu, incl, L + w - 1);
                            if (x <= g) L += w;
                        }
                        cc[u] = g - __shfl_sync(0xffffffffu, excl, L);
                        const long long b = __shfl_sync(0xffffffffu, base, L);
                        ln[u] = __shfl_sync(0xffffffffu, len, L);
                        am[u] = __shfl_sync(0xffffffffu, amount, L);
                        v[u] = make_int4(-1, 0, -1, 0);
                        if (g < total) {
                            if (ELL) v[u] = ld_stream16(s.ell + b + 2 * cc[u], pol);
                            else v[u].x = (int)ld_stream4(s.sdst + b + cc[u], pol);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kBinUnroll; ++u) {
                        if (g0 + u * 32 + lane >= total) continue;
                        if (ELL) {
                            if (cc[u] > 0) deliver((uint32_t)v[u].x, (uint32_t)v[u].y);
                            if (2 * cc[u] + 1 < ln[u]) deliver((uint32_t)v[u].z, (uint32_t)v[u].w);
                        } else {
                            deliver((uint32_t)v[u].x, (uint32_t)am[u]);
                        }
                    }
                }
            }
            }  // GROUP
            if ((win + 1) % kWin != 0 && c0 + kBinThreads < nd) continue;  // keep staging
            __syncthreads();
            // ---- D. flush every bucket: pad to whole 16-byte units, one reservation, vector stores
            for (int dt = warp; dt < NT; dt += kBinThreads / 32) {
                const uint32_t c = cnt[dt];
                if (c == 0) continue;
                const uint32_t n = min(c, (uint32_t)kCap);
                const uint32_t np = (n + kVec - 1) & ~(uint32_t)(kVec - 1);
                E* row = stage + dt * kCap;
                if ((uint32_t)lane < np - n) row[n + lane] = pad;
                uint32_t g = 0;
                if (lane == 0) g = atomicAdd(fill_out + dt, np);
                g = __shfl_sync(0xffffffffu, g, 0);
                __syncwarp();
                const uint32_t o = __ldg(s.bin_off + dt), cap = __ldg(s.bin_off + dt + 1) - o;
                if (g + np > cap) {
                    t_over = true;
                } else if ((uint32_t)lane < np / kVec) {
                    reinterpret_cast<uint4*>(bin_out + o + g)[lane] = reinterpret_cast<const uint4*>(row)[lane];
                }
                __syncwarp();
                if (lane == 0) cnt[dt] = 0;
            }
            __syncthreads();
        }
    }

    if (stats_on) {
        stat[ST_EDGES] = (unsigned int)edges;
        flush_stats(ctl, stat);
    }
    if (__syncthreads_or(t_over) && threadIdx.x == 0) atomicOr(&ctl->fault, 1);  // bin overflow (never expected)
    const bool bf = __syncthreads_or(t_fired);
    const bool bc = __syncthreads_or(t_closed);
    __shared__ long long sh_neg_idx, sh_neg_val;
    if (threadIdx.x == 0) sh_neg_idx = 0x7fffffffffffffffll;
    __syncthreads();
    if (t_neg) atomicMin(&sh_neg_idx, neg_idx);
    __syncthreads();
    if (t_neg && sh_neg_idx == neg_idx) sh_neg_val = neg_val;
    const bool bn = __syncthreads_or(t_neg);
    if (threadIdx.x == 0) finish_step(ctl, k, sel, bf, bc, bn, sh_neg_idx, bn ? sh_neg_val : 0);
}

// ---------------------------------------------------------------------------
// Small systems (variant SMALL; COMPRESSED, q <= kSmallMaxQ): ONE CTA runs a
// whole loop segment -- every step of [step, stop_at) -- in one launch, with
// block barriers where the other variants have kernel boundaries and the
// receive vector in shared memory.  A graph-replayed grid-wide step kernel
// costs ~10 us per step on this B200 however little a step holds (sort
// n <= 100 is far below a microsecond of work), so small systems were
// launch-bound; here a step is a handful of barriers.  Step semantics are
// step_kernel<RECV_ARRAY> + push_kernel (consumption at selection, push of
// Alg. 5, engine.py:312-356): per step k
//   A. finish step k-1 for every neuron (C += open ? recv, D, NegativeSpikes,
//      trace rows) and select the <= 32-rule neurons (light_commit);
//   B. select the > 32-rule neurons, one warp each (guard index /
//      SeededRandom scan, as the tiled kernel's phase 3);
//   C. push: each fired sending neuron adds p to its targets' counters
//      (shared-memory 64-bit atomics);
//   D. halting decision for step k (finish_step's rules), then the next step.
constexpr int kSmallThreads = 1024;
constexpr long long kSmallMaxQ = 16384;   // 128 KB of int64 receive counters
constexpr long long kSmallSmemQ = 4096;   // state in shared memory too: 4096 x (8 + 4 + 4 + 8) B

#ifndef SNP_TEMPLATES_ONLY
// R64: 64-bit receive counters (some destination can receive >= 2^31 in one
// step); else 32-bit, whose shared-memory atomics are native
// SMEM: the state itself (Ĉ, delay state, chosen rule) lives in shared memory
// for the whole launch (q <= kSmallSmemQ): every step's reads and writes of it
// are shared-memory accesses instead of L2 round trips
template <bool WIDE, bool R64, bool SMEM>
__global__ void __launch_bounds__(kSmallThreads, 1) small_run_kernel(const __grid_constant__ DevSys s, DevState st) {
    using RT = typename std::conditional<R64, unsigned long long, unsigned int>::type;
    extern __shared__ __align__(128) uint8_t smem[];
    RT* recv_s = reinterpret_cast<RT*>(smem);  // [q] deliveries of the previous step
    DevState sl = st;                          // the state the steps read and write
    __shared__ long long sh_neg_idx, sh_neg_val;
    __shared__ int sh_go;
    Ctrl* ctl = st.ctrl;
    volatile Ctrl* vc = ctl;
    if (vc->halted || vc->step >= vc->stop_at) {
        if (threadIdx.x == 0) ctl->push_armed = 0;
        return;
    }
    using Raw = typename RuleRaw<WIDE>::T;
    const long long q = s.q;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long max_steps = vc->max_steps, stop_at = vc->stop_at, trace_base = vc->trace_base;
    const int policy = vc->policy, record = vc->record;
    const bool stats_on = vc->stats_on != 0;
    const unsigned long long seed = vc->seed;
    long long k = vc->step;
    if (SMEM) {
        const size_t o = ((size_t)q * sizeof(RT) + 15) & ~(size_t)15;
        sl.cfg = reinterpret_cast<long long*>(smem + o);
        sl.ds = reinterpret_cast<int*>(smem + o + (size_t)q * 8);
        sl.chosen = reinterpret_cast<int*>(smem + o + (size_t)q * 12);
        for (long long j = threadIdx.x; j < q; j += kSmallThreads) {
            sl.cfg[j] = st.cfg[j];
            sl.ds[j] = st.ds[j];
            sl.chosen[j] = st.chosen[j];
        }
    }
    for (long long j = threadIdx.x; j < q; j += kSmallThreads) recv_s[j] = (RT)st.recv[j];
    __syncthreads();
    for (;;) {
        const bool sel = k < max_steps;
        const StepCtx cx{k, k - trace_base, q, seed, nullptr, policy, record, sel, stats_on};
        unsigned int stat[ST_COUNT];
#pragma unroll
        for (int i = 0; i < ST_COUNT; ++i) stat[i] = 0;
        bool t_fired = false, t_closed = false, t_neg = false;
        long long neg_idx = 0x7fffffffffffffffll, neg_val = 0;
        // ---- A
        for (long long j = threadIdx.x; j < q; j += kSmallThreads) {
            const uint32_t r0 = __ldg(s.roff + j), nr = __ldg(s.roff + j + 1) - r0;
            const int dsv = sl.ds[j];
            const int D = ds_next(dsv);
            long long C = sl.cfg[j];
            const long long rv = R64 ? (long long)recv_s[j] : (long long)(int)recv_s[j];
            recv_s[j] = 0;
            if (ds_open(dsv)) C += rv;
            if (nr > kLightRules) {
                if (C < 0 && j + s.gbase < neg_idx) {
                    t_neg = true;
                    neg_idx = j + s.gbase;
                    neg_val = C;
                }
                if (record & REC_CONFIGS) st.tr_cfg[cx.slot * q + j] = C;
                if (record & REC_DELAYS) st.tr_dly[cx.slot * q + j] = D;
                t_closed |= D != 0;
                sl.cfg[j] = C;
                sl.ds[j] = D;
                if (sel) {
                    sl.chosen[j] = -1;
                    if (record & REC_SPIKING) st.tr_chosen[cx.slot * q + j] = -1;
                }
            } else {
                const bool can_sel = sel && D == 0;
                Raw w0{}, w1{}, w2{}, w3{};
                if (can_sel) {
                    if (nr > 0) w0 = load_raw<WIDE>(s.rw, r0);
                    if (nr > 1) w1 = load_raw<WIDE>(s.rw, r0 + 1);
                    if (nr > 2) w2 = load_raw<WIDE>(s.rw, r0 + 2);
                    if (nr > 3) w3 = load_raw<WIDE>(s.rw, r0 + 3);
                }
                int r = -1;
                long long ni = neg_idx, nv = neg_val;
                light_commit<RECV_ARRAY, P_BIT, true, false, WIDE>(s, sl, ctl, cx, j, r0, nr, w0, w1, w2, w3, C, D, can_sel,
                                                                   stat, t_fired, t_closed, t_neg, ni, nv, r);
                if (ni < neg_idx) neg_idx = ni, neg_val = nv;
            }
        }
        __syncthreads();
        // ---- B: heavy neurons.  B1, thread per neuron: the dense tables answer
        // FirstApplicable, and SeededRandom when the choice is forced; B2,
        // warp per neuron, scans what the tables leave open (marked -3).
        auto commit_heavy = [&](long long j, long long C, uint32_t r0, uint32_t r1, int r, bool scanned_all) {
            stat[ST_SCANNED] += scanned_all ? r1 - r0 : ((r >= 0) ? (uint32_t)r - r0 + 1 : r1 - r0);
            stat[ST_OPEN] += 1;
            if (r >= 0) {
                const uint4 wr = load_rule<WIDE>(s.rw, r);
                sl.cfg[j] = C - (long long)wr.y;
                sl.ds[j] = -((int)wr.w + 1);
                sl.chosen[j] = r;
                t_fired = true;
                stat[ST_FIRED] += 1;
                if (wr.z > 0) {
                    stat[ST_SENDING] += 1;
                    if (stats_on) {
                        const uint32_t od = __ldg(s.outdeg + j);
                        stat[ST_ROWS] += od + (od < (uint32_t)s.z ? 1u : 0u);
                    }
                }
                if (record & REC_SPIKING) st.tr_chosen[cx.slot * q + j] = r;
            }
        };
        bool any_scan = false;
        if (sel) {
            for (int h = threadIdx.x; h < s.n_heavy; h += kSmallThreads) {
                const long long j = s.heavy[h];
                if (sl.ds[j] != 0) continue;  // D_k (A stored it): closed
                const long long C = sl.cfg[j];
                const int x = policy == 0 ? heavy_first_table(s, h, C) : heavy_seeded_table(s, h, C);
                if (x == -2) {
                    sl.chosen[j] = -3;  // B2 scans it
                    any_scan = true;
                    continue;
                }
                const uint32_t r0 = __ldg(s.roff + j), r1 = __ldg(s.roff + j + 1);
                commit_heavy(j, C, r0, r1, x < 0 ? -1 : (int)(r0 + x), policy != 0);
            }
        }
        if (__syncthreads_or(any_scan)) {
            for (int h = warp; h < s.n_heavy; h += kSmallThreads / 32) {
                const long long j = s.heavy[h];
                if (sl.chosen[j] != -3) continue;
                const long long C = sl.cfg[j];
                const uint32_t r0 = __ldg(s.roff + j), r1 = __ldg(s.roff + j + 1);
                int r;
                if (policy == 0) {
                    const int x = heavy_first_applicable_warp(s, h, C, lane);
                    r = x < 0 ? -1 : (int)(r0 + x);
                } else {
                    r = heavy_seeded_warp<WIDE>(s, r0, r1, C, seed, k, j + s.gbase, lane);
                }
                __syncwarp();
                if (lane == 0) {
                    sl.chosen[j] = -1;
                    commit_heavy(j, C, r0, r1, r, policy != 0);
                }
            }
        }
        __syncthreads();
        // ---- C (one warp per fired neuron, lanes over its out-edges)
        if (sel) {
            for (long long j = warp; j < q; j += kSmallThreads / 32) {
                const int r = sl.chosen[j];
                if (r < 0) continue;
                const int p = __ldg(&s.rrec[r].y);
                if (p <= 0) continue;
                const uint32_t e0 = __ldg(s.soff + j), e1 = __ldg(s.soff + j + 1);
                if (lane == 0) stat[ST_EDGES] += e1 - e0;
                for (uint32_t e = e0 + lane; e < e1; e += 32) atomicAdd(recv_s + __ldg(s.sdst + e), (RT)p);
            }
        }
        // ---- D
        if (stats_on) flush_stats(ctl, stat);
        const bool bf = __syncthreads_or(t_fired);
        const bool bc = __syncthreads_or(t_closed);
        if (threadIdx.x == 0) sh_neg_idx = 0x7fffffffffffffffll;
        __syncthreads();
        if (t_neg) atomicMin(&sh_neg_idx, neg_idx);
        __syncthreads();
        if (t_neg && sh_neg_idx == neg_idx) sh_neg_val = neg_val;
        const bool bn = __syncthreads_or(t_neg);
        if (threadIdx.x == 0) {
            int go = 0;
            if (vc->fault) {
                vc->halted = 1;
                vc->reason = HALT_FAULT;
            } else if (bn) {
                vc->neg_any = 1;
                vc->neg_index = sh_neg_idx;
                vc->neg_value = sh_neg_val;
                vc->halted = 1;
                vc->reason = HALT_NEGATIVE;
            } else if (!sel) {
                vc->halted = 1;
                vc->reason = HALT_STEP_LIMIT;
            } else if (!bf && !bc) {
                vc->halted = 1;
                vc->reason = HALT_NO_APPLICABLE;
            } else {
                vc->step = k + 1;
                if (stats_on) vc->stats[ST_STEPS] += 1;
                go = k + 1 < stop_at;
            }
            vc->push_armed = 0;
            sh_go = go;
        }
        __syncthreads();
        if (!sh_go) break;
        ++k;
    }
    for (long long j = threadIdx.x; j < q; j += kSmallThreads) {
        st.recv[j] = R64 ? (long long)recv_s[j] : (long long)(int)recv_s[j];
        if (SMEM) {
            st.cfg[j] = sl.cfg[j];
            st.ds[j] = sl.ds[j];
            st.chosen[j] = sl.chosen[j];
        }
    }
    __threadfence();
}
#endif  // SNP_TEMPLATES_ONLY

// Dense S.M (paper Alg. 3 over the fired rows only): blockIdx.x tiles 1024
// columns (int4 per thread), blockIdx.y splits the fired-rule list.
#ifndef SNP_TEMPLATES_ONLY
__global__ void __launch_bounds__(kBlock) dense_kernel(const __grid_constant__ DevSys s, DevState st) {
    Ctrl* ctl = st.ctrl;
    const volatile Ctrl* vc = ctl;
    if (!vc->push_armed) return;
    const long long k = vc->step - 1;
    const unsigned int n = vc->list_count[k & 1];
    const long long c4 = ((long long)blockIdx.x * kBlock + threadIdx.x) * 4;
    if (c4 >= s.q) return;
    const unsigned int lo = (unsigned int)((unsigned long long)n * blockIdx.y / gridDim.y);
    const unsigned int hi = (unsigned int)((unsigned long long)n * (blockIdx.y + 1) / gridDim.y);
    long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const uint32_t* lst = pick2(st.list, k);
    for (unsigned int f = lo; f < hi; ++f) {
        const uint32_t r = lst[f];
        const int4 v = __ldg(reinterpret_cast<const int4*>(s.dense + (long long)r * s.dense_ld + c4));
        a0 += v.x;
        a1 += v.y;
        a2 += v.z;
        a3 += v.w;
    }
    if (a0) red_add_i64(st.recv + c4, a0);
    if (a1 && c4 + 1 < s.q) red_add_i64(st.recv + c4 + 1, a1);
    if (a2 && c4 + 2 < s.q) red_add_i64(st.recv + c4 + 2, a2);
    if (a3 && c4 + 3 < s.q) red_add_i64(st.recv + c4 + 3, a3);
    if (vc->stats_on && blockIdx.x == 0 && threadIdx.x == 0 && blockIdx.y == 0)
        atomicAdd(&ctl->stats[ST_EDGES], (unsigned long long)n * (unsigned long long)s.q);
}

#endif  // SNP_TEMPLATES_ONLY

// ---------------------------------------------------------------------------
// Phase-API helpers.

// Load an arbitrary (C, D, chosen) as the engine state right after the
// selection of step 0 (engine.py:239-355 take the spiking vector as input).
// The source-open re-check of engine.py:252/281/321 applies: a chosen rule
// of a closed neuron is ignored.
template <int KIND, int PM, bool CONSUME, bool FLIST>
__global__ void prime_kernel(const __grid_constant__ DevSys s, DevState st, const long long* __restrict__ C,
                             const long long* __restrict__ D, const long long* __restrict__ chosen) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= s.q) return;
    long long r = chosen[j];
    const long long d = D[j];
    if (d != 0) r = -1;
    long long c = C[j];
    int nds = (int)d;
    long long pval = 0;
    if (r >= 0) {
        const int4 rec = s.rrec[r];
        if (CONSUME) c -= rec.x;
        pval = rec.y;
        nds = -(rec.z + 1);
        if (FLIST) {
            unsigned int pos = atomicAdd(&st.ctrl->list_count[0], 1u);
            st.list[0][pos] = (uint32_t)r;
        }
    }
    st.cfg[j] = c;
    st.ds[j] = nds;
    if (KIND == RECV_ARRAY) {
        st.chosen[j] = (int)r;
    } else if (PM == P_BIT) {
        if (pval > 0) atomicOr(st.P[0] + (j >> 5), 1u << (j & 31));
    } else if (PM == P_U8) {
        reinterpret_cast<uint8_t*>(st.P[0])[j] = (uint8_t)pval;
    } else if (PM == P_U16) {
        reinterpret_cast<uint16_t*>(st.P[0])[j] = (uint16_t)pval;
    } else {
        st.P[0][j] = (uint32_t)pval;
    }
}

// update_delays (engine.py:358-366): no source-open filter, like the reference.
#ifndef SNP_TEMPLATES_ONLY
__global__ void update_delays_kernel(long long q, const int4* __restrict__ rrec,
                                     const long long* __restrict__ D,
                                     const long long* __restrict__ chosen, long long* out) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= q) return;
    const long long r = chosen[j];
    const long long d = D[j];
    out[j] = r >= 0 ? (long long)rrec[r].z : (d > 0 ? d - 1 : 0);
}
#endif

// Load (C, D) so that the next step kernel finalises exactly C_k = C, D_k = D
// and then selects (sv_calc of engine.py:192-236).
// Row digests for SNP_REC_DIGEST (include/snpb200.h): grid.y = row.
__device__ __forceinline__ unsigned long long fmix64(unsigned long long z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
template <typename T>
__global__ void __launch_bounds__(256) digest_rows_kernel(const T* __restrict__ rows, long long q,
                                                          unsigned long long* out) {
    const T* row = rows + (long long)blockIdx.y * q;
    unsigned long long acc = 0;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < q; j += (long long)gridDim.x * blockDim.x)
        acc += fmix64((unsigned long long)(long long)row[j] * 0x9E3779B97F4A7C15ull +
                      (unsigned long long)(j + 1) * 0xD6E8FEB86659FD93ull);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out + blockIdx.y, acc);
}

#ifndef SNP_TEMPLATES_ONLY
__global__ void load_state_kernel(long long q, long long* cfg, int* ds, const long long* __restrict__ C,
                                  const long long* __restrict__ D) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= q) return;
    cfg[j] = C[j];
    ds[j] = (int)(D[j] + 1);  // ds_next(D+1) == D, and not "open last step"
}
#endif

#ifndef SNP_TEMPLATES_ONLY
__global__ void widen_i32_kernel(long long n, const int* __restrict__ in, long long* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}
#endif

// D_k from the delay state after a halt (the last kernel ran without selection).
#ifndef SNP_TEMPLATES_ONLY
__global__ void ds_to_delay_kernel(long long q, const int* __restrict__ ds, long long* out) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < q) {
        const int v = ds[j];
        out[j] = v < 0 ? -v - 1 : v;  // after a halt ds holds D_k directly (no firing)
    }
}
#endif

// ---------------------------------------------------------------------------
// Device-side layout builders (from the CSR out-adjacency).

// In-degree histogram of the transpose.
#ifndef SNP_TEMPLATES_ONLY
__global__ void indeg_kernel(long long S, const uint32_t* __restrict__ dst, uint32_t* indeg) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < S;
         e += (long long)gridDim.x * blockDim.x)
        atomicAdd(indeg + dst[e], 1u);
}
#endif

// Scatter sources into their destination lists (cursor = padded offsets).
#ifndef SNP_TEMPLATES_ONLY
__global__ void transpose_fill_kernel(long long q, const uint32_t* __restrict__ soff,
                                      const uint32_t* __restrict__ sdst, uint32_t* cursor,
                                      uint32_t* isrc) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= q) return;
    for (uint32_t e = soff[i]; e < soff[i + 1]; ++e) {
        const uint32_t pos = atomicAdd(cursor + sdst[e], 1u);
        isrc[pos] = (uint32_t)i;
    }
}
#endif

// ELL columns per rule: (owner, -c) then (dst, p) for sending rules.
#ifndef SNP_TEMPLATES_ONLY
__global__ void build_ell_kernel(long long m, long long ld, const uint32_t* __restrict__ owner,
                                 const int4* __restrict__ rrec, const uint32_t* __restrict__ soff,
                                 const uint32_t* __restrict__ sdst, int2* ell, uint32_t* len) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const uint32_t o = owner[r];
    const int4 rec = rrec[r];
    int2* col = ell + r * ld;
    col[0] = make_int2((int)o, -rec.x);
    uint32_t n = 1;
    if (rec.y > 0) {
        for (uint32_t e = soff[o]; e < soff[o + 1]; ++e) col[n++] = make_int2((int)sdst[e], rec.y);
    }
    len[r] = n;
}
#endif

// Dense rows: -c at the owner, +p at every out-neighbour (matrices.py:143-154).
#ifndef SNP_TEMPLATES_ONLY
__global__ void build_dense_kernel(long long m, long long ld, const uint32_t* __restrict__ owner,
                                   const int4* __restrict__ rrec, const uint32_t* __restrict__ soff,
                                   const uint32_t* __restrict__ sdst, int* dense) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const uint32_t o = owner[r];
    const int4 rec = rrec[r];
    int* row = dense + r * ld;
    row[o] = -rec.x;
    if (rec.y > 0)
        for (uint32_t e = soff[o]; e < soff[o + 1]; ++e) row[sdst[e]] = rec.y;
}
#endif

}  // namespace snp
