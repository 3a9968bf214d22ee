// snp_engine.cu -- host runtime + C ABI (include/snpb200.h) of the B200 SNP
// step engine.  Owns all device memory of an engine; builds the device
// layouts from the reference's interchange arrays (RuleVector,
// NeuronRuleMap, and either a CSR out-adjacency or the format's own matrix);
// drives the per-step kernels of snp_device.cuh as CUDA-graph segments with
// device-side halting; and implements the phase-level entry points.
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys / ncu --nvtx (no cost without a tool)
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/snpb200.h"
#include "snp_device.cuh"
#include "snp_ingest.cuh"

using namespace snp;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CU(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            return fail(e_ == cudaErrorMemoryAllocation ? SNP_ERR_CAPACITY : SNP_ERR_CUDA,        \
                        "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__,          \
                        __LINE__);                                                                \
        }                                                                                         \
    } while (0)

#define TRY(expr)                \
    do {                         \
        int rc_ = (expr);        \
        if (rc_ != SNP_OK) return rc_; \
    } while (0)

constexpr long long kInt32Max = 2147483647ll;

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// Host loops over q / m / S run on all host threads (engine creation at 10^7+).
// f(a, b) handles [a, b) and returns the first failing index there (or -1);
// the smallest failing index over all chunks is returned, so errors are the
// ones a sequential loop would report.
template <typename F>
long long parallel_first_fail(long long n, F f) {
    const long long nt = std::max<long long>(
        1, std::min<long long>((long long)std::max(1u, std::thread::hardware_concurrency()), n / (1 << 16) + 1));
    if (nt == 1) return n > 0 ? f(0, n) : -1;
    std::vector<long long> bad(nt, -1);
    std::vector<std::thread> th;
    for (long long t = 0; t < nt; ++t) th.emplace_back([&, t] { bad[t] = f(n * t / nt, n * (t + 1) / nt); });
    for (auto& x : th) x.join();
    for (long long b : bad)
        if (b >= 0) return b;
    return -1;
}

// CSR out-adjacency offsets (caller-built SystemArrays): offsets[0] == 0 and
// non-decreasing, so every out-degree and the edge count offsets[q] are
// well defined before any kernel walks them.
int check_csr_offsets(const int64_t* off, long long q) {
    if (q <= 0) return SNP_OK;
    if (off[0] != 0) return fail(SNP_ERR_BAD_ARG, "adj_offsets[0] must be 0, got %lld", (long long)off[0]);
    const long long bad = parallel_first_fail(q, [&](long long a, long long b) -> long long {
        for (long long i = a; i < b; ++i)
            if (off[i + 1] < off[i]) return i;
        return -1;
    });
    if (bad >= 0)
        return fail(SNP_ERR_BAD_ARG, "adj_offsets decrease at neuron %lld (%lld > %lld)", bad, (long long)off[bad],
                    (long long)off[bad + 1]);
    return SNP_OK;
}

using StepFn = void (*)(DevSys, DevState);
using PrimeFn = void (*)(DevSys, DevState, const long long*, const long long*, const long long*);

template <int KIND, int PM, bool CONSUME, bool FLIST>
void pick_fns(bool wide, StepFn* step, PrimeFn* prime) {
    *step = wide ? step_kernel<KIND, PM, CONSUME, FLIST, true> : step_kernel<KIND, PM, CONSUME, FLIST, false>;
    *prime = prime_kernel<KIND, PM, CONSUME, FLIST>;
}

}  // namespace

struct snp_engine {
    int format = SNP_FMT_COMPRESSED;
    int variant = SNP_VARIANT_PULL;
    int device = 0;
    long long q = 0, m = 0;
    int z = 0;
    int p_mode = P_BIT;
    long long p_common = 1;
    long long p_max = 0;      // largest produced amount
    int cbits = 32;           // tiled: destination counter bits (32, 16, 8; acc_words)
    long long in_edges = 0;
    int kind = RECV_PULL;
    bool tiled = false;
    long long p_words = 0;  // sharded: exchange words per P buffer
    uint32_t* xblock = nullptr;            // sharded: exchange block (3 slots + step flags)
    unsigned long long epoch = 0;          // runs begun (peer-exchange step flags)
    std::vector<void*> ipc_opened;         // peer blocks mapped with cudaIpcOpenMemHandle
    unsigned long long* d_peers = nullptr; // device array of every rank's block
    long long shard_lo = 0, shard_hi = 0, shard_nl = 0;
    cudaStream_t own_stream = nullptr;
    int step_block = kBlock;
    size_t step_smem = 0;
    bool wide_rules = false;
    bool tiny_rules = false;  // tiled: 4-byte staged rule words (s.rw4)
    long long resident_ctas = 0;
    cudaStream_t stream = nullptr;
    std::vector<void*> allocs;
    long long device_bytes = 0;
    std::vector<long long> initial;  // host copy of the system's C_0
    DevSys sys{};
    DevState st{};
    StepFn step_fn = nullptr;
    StepFn lean_fn = nullptr;  // tiled: instance without recording / counters
    StepFn fused_fn = nullptr; // push formats: one-kernel step (push_step_kernel) for runs
    bool recv64 = false;       // fused push: 64-bit receive buffers
    int fused_grid = 0, fused_block = 0;
    size_t fused_smem = 0;
    int bin_cb = 0;            // binned push: counter bits (0 = not binned)
    bool bin_unit = false;     // binned push: u16 slot entries
    size_t bin_smem = 0;       // binned push: dynamic shared memory
    PrimeFn prime_fn = nullptr;
    StepFn small_fn = nullptr;  // variant SMALL: one-CTA loop-segment kernel for runs
    bool pdl = true;            // tiled: programmatic dependent launch (SNPB200_PDL=0: off)
    size_t small_smem = 0;
    int step_grid = 0;
    int push_grid = 0;
    int heavy_push_grid = 0;
    dim3 dense_grid;
    // run state
    Ctrl hctrl{};
    bool begun = false;
    // graph cache
    cudaGraphExec_t graph = nullptr;
    long long graph_iters = 0;
    StepFn graph_fn = nullptr;
    long long tr_rows = 0;
    // phase scratch
    long long* scratch[4] = {nullptr, nullptr, nullptr, nullptr};
    unsigned long long* d_digest = nullptr;  // SNP_REC_DIGEST row digests (3 x digest_cap)
    long long digest_cap = 0;
    long long n_stages = 0, n_sbases = 0;   // tiled layout sizes (layout digest)
    int p1_grid = 0;                        // two-pass: pass-1 CTAs
    long long p_bit_words = 0;              // P_BIT: words per P buffer (single engine)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_ms = 0.0;

    template <typename T>
    int alloc(T** p, long long count) {
        size_t bytes = (size_t)std::max<long long>(count, 1) * sizeof(T);
        void* ptr = nullptr;
        cudaError_t e = cudaMalloc(&ptr, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(SNP_ERR_CAPACITY, "cudaMalloc of %zu bytes failed: %s", bytes,
                        cudaGetErrorString(e));
        }
        allocs.push_back(ptr);
        device_bytes += (long long)bytes;
        *p = static_cast<T*>(ptr);
        return SNP_OK;
    }

    ~snp_engine() {
        for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
        if (graph) cudaGraphExecDestroy(graph);
        for (void* p : allocs) cudaFree(p);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (own_stream) cudaStreamDestroy(own_stream);
    }
};

namespace {

// Host vectors that every element is written into before being read: the
// default-initialising allocator skips std::vector's serial zero fill (GBs at
// 10^8 neurons: the rule records alone are 6.4 GB).
template <typename T>
struct DefaultInit : std::allocator<T> {
    template <typename U>
    struct rebind {
        using other = DefaultInit<U>;
    };
    DefaultInit() = default;
    template <typename U>
    DefaultInit(const DefaultInit<U>&) {}
    template <typename U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <typename U, typename... Args>
    void construct(U* p, Args&&... args) {
        ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
};
template <typename T>
using hvec = std::vector<T, DefaultInit<T>>;

template <typename T, typename A>
int upload(snp_engine* e, T** dptr, const std::vector<T, A>& host) {
    TRY(e->alloc(dptr, (long long)host.size()));
    if (!host.empty()) CU(cudaMemcpy(*dptr, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice));
    return SNP_OK;
}

__global__ void fill_u32_kernel(long long n, uint32_t* p, uint32_t v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

int grid_for(long long n, int block = 256) {
    return (int)std::max<long long>(1, std::min<long long>(ceil_div(n, block), 1ll << 30));
}

// Row partition (multi-GPU): this engine owns global neurons [lo, hi); the
// edges into them come from every source, and sources are renumbered into the
// exchange space where rank r's chunk starts at element r * (nl + hdr): its
// nl P elements (1, 8, 16 or 32 bits each, the same width on every rank),
// then a 4-word header of step flags (hdr = 128 / element bits elements).
struct ShardInput {
    int world = 1, rank = 0;
    long long q_global = 0, nl = 0, lo = 0, hi = 0;
    int x_pbits = 0;          // agreed P element width (0: decide from this rank's rules)
    long long x_pmax = 0;     // agreed largest produced amount over every rank
    mutable long long hdr = 128;  // header elements, set once the P width is known
    hvec<uint32_t> soff, sdst;  // global out-adjacency
    uint32_t xpos(uint32_t src) const {
        return (uint32_t)((src / nl) * (nl + hdr) + src % nl);
    }
};

// Tiled-pull layout (see tiled_step_kernel): destinations are cut into
// tiles of T; each tile's in-edges, visited in ascending source order (the
// CSR out-adjacency is source-major, so a stable bucket pass keeps that
// order), are packed into 256-edge segments whose sources span < 2^17.
int build_tiles_device(snp_engine* e, const uint32_t* d_soff, const uint32_t* d_sdst, long long S, bool stage_p);
int build_tiles2(snp_engine* e, const uint32_t* d_soff, const uint32_t* d_sdst, const hvec<uint32_t>& soff,
                 const hvec<uint32_t>& sdst, const ShardInput* sh, const std::vector<uint32_t>& roff_h);

// Phase-2 stage descriptors of tile t (kSub destinations each, with their
// rule words when they fit a stage).
void append_phase2_desc(const snp_engine* e, long long t, const std::vector<uint32_t>& roff_h,
                        std::vector<StageDesc>& desc) {
    const DevSys& s = e->sys;
    const long long T = s.tile, q = e->q;
    const uint32_t rw_size = e->tiny_rules ? 4u : (e->wide_rules ? 16u : 8u);
    auto r16 = [](unsigned long long x) { return (uint32_t)((x + 15) & ~15ull); };
    const long long d0 = t * T;
    const long long nd = std::min<long long>(T, q - d0);
    for (long long dd = 0; dd < nd; dd += kSub) {
        const uint32_t n = (uint32_t)std::min<long long>(kSub, nd - dd);
        const uint32_t rf = roff_h[d0 + dd], rl = roff_h[d0 + dd + n];
        const uint32_t r_al = e->tiny_rules ? (rf & ~3u) : (e->wide_rules ? rf : (rf & ~1u));
        const uint32_t fixed = kPayload + kP2Rules(s.rpn != 0);
        uint32_t rb = r16((unsigned long long)(rl - r_al) * rw_size);
        if (fixed + rb > kStageBytes) rb = 0;
        StageDesc sd;
        sd.a = make_uint4(2u | ((dd + kSub >= nd) ? 256u : 0u), (uint32_t)dd, n, r_al);
        sd.b = make_uint4(rb, 0, 0, 0);
        desc.push_back(sd);
    }
}

int build_tiles(snp_engine* e, const snp_system_desc* d, const hvec<uint32_t>& soff_in,
                const hvec<uint32_t>& sdst_in, const std::vector<uint32_t>& roff_h,
                std::vector<uint32_t>& heavy, const ShardInput* sh, const uint32_t* d_soff = nullptr,
                const uint32_t* d_sdst = nullptr) {
    const hvec<uint32_t>& soff = sh ? sh->soff : soff_in;
    const hvec<uint32_t>& sdst = sh ? sh->sdst : sdst_in;
    const long long lo = sh ? sh->lo : 0, hi = sh ? sh->hi : e->q;
    const long long n_src = sh ? sh->q_global : e->q;
    const long long q = e->q;
    DevSys& s = e->sys;
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, e->device);
    // heavy-rule neurons only (in-degree does not matter here)
    heavy.clear();
    for (long long i = 0; i < q; ++i)
        if (d->offsets[i + 1] - d->offsets[i] > (long long)kLightRules) heavy.push_back((uint32_t)i);
    // 16-bit counters when no destination can receive 2^16 or more per step
    // (P_BIT counts sending in-neighbours; other modes sum produced amounts)
    {
        std::vector<uint32_t> indeg(std::max<long long>(q, 1), 0);
        if (!sh && d_sdst && !sdst.empty()) {
            // in-degrees on the device (the adjacency is already there)
            uint32_t* d_in;
            CU(cudaMalloc(&d_in, (size_t)q * 4));
            CU(cudaMemset(d_in, 0, (size_t)q * 4));
            indeg_kernel<<<std::min(grid_for((long long)sdst.size()), 148 * 64), 256>>>((long long)sdst.size(), d_sdst, d_in);
            cudaError_t err = cudaGetLastError();
            if (err == cudaSuccess) err = cudaMemcpy(indeg.data(), d_in, (size_t)q * 4, cudaMemcpyDeviceToHost);
            cudaFree(d_in);
            CU(err);
        } else {
            for (size_t e2 = 0; e2 < sdst.size(); ++e2)
                if ((long long)sdst[e2] >= lo && (long long)sdst[e2] < hi) indeg[sdst[e2] - lo]++;
        }
        const long long unit = e->p_mode == P_BIT ? 1 : std::max<long long>(1, e->p_max);
        long long worst = 0;
        for (uint32_t x : indeg) worst = std::max<long long>(worst, (long long)x * unit);
        // the counters are at most 32 bits: a destination that can receive
        // 2^32 or more in one step needs the 64-bit CSR-pull gather
        if (worst >= (1ll << 32))
            return fail(SNP_ERR_CAPACITY,
                        "a neuron can receive %lld spikes in one step, beyond the tiled kernel's 32-bit receive "
                        "counters; use variant \"pull\"", worst);
        e->cbits = worst < 256 ? 8 : (worst < 65536 ? 16 : 32);
        if (const char* env = getenv("SNPB200_COUNTER_BITS")) e->cbits = std::max(e->cbits, atoi(env));
    }
    // one CTA per SM; a multiple of the SM count in tiles keeps them balanced.
    // 8/16-bit counters: one tile per SM (T = q / 148; the ring keeps at
    // least 3 x 48 KB, T shrinks below if needed) -- measured on the round-2
    // kernel: K3 0.240 -> 0.229 ms, K4 0.241 -> 0.229, 10^6 neurons 0.044 ->
    // 0.040 vs two tiles per SM (profiles/r2_history.md); 32-bit counters and
    // heavy-rule systems: 4 per SM (more, smaller tiles)
    long long per_sm = (e->cbits <= 16 && heavy.empty()) ? 1 : 4;
    if (const char* env = getenv("SNPB200_TILES_PER_SM")) per_sm = std::max(1, atoi(env));
    long long T = ceil_div(std::max<long long>(q, 1), per_sm * n_sm);
    if (!heavy.empty()) T = std::min<long long>(T, std::max<long long>(32, 32ll * q / (long long)heavy.size()));
    if (const char* env = getenv("SNPB200_TILE")) T = atoll(env);
    // shared memory: the TMA ring (2..kMaxRing stages) plus the destination
    // counters; the ring gets what the counters of a T-tile leave, and T only
    // shrinks when not even two stages would fit
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device);
    cudaFuncAttributes fa{};
    {
        TiledFn probe = nullptr, probe_lean = nullptr;
        tiled_fns<P_BIT>(RW_WIDE, 32, &probe, &probe_lean);
        CU(cudaFuncGetAttributes(&fa, (const void*)probe));
    }
    const long long budget = (long long)smem_optin - (long long)fa.sharedSizeBytes - 128;
    auto acc_b = [&](long long t) {
        return 4ll * (e->cbits == 8 ? acc_words<8>((int)t) : (e->cbits == 16 ? acc_words<16>((int)t) : acc_words<32>((int)t)));
    };
    T = std::min<long long>(s.tp ? 65504 : kMaxTile, std::max<long long>(32, (T + 31) / 32 * 32));
    // large systems: cap T so that the ring keeps 3 stages
    while (T > 32 * 64 && (budget - acc_b(T)) / (long long)kStageBytes < 3 &&
           (budget - acc_b(T - 32)) / (long long)kStageBytes >= 1)
        T -= 32;
    long long ring = std::min<long long>(kMaxRing, (budget - acc_b(T)) / (long long)kStageBytes);
    if (const char* env = getenv("SNPB200_RING")) ring = std::min<long long>(ring, atoll(env));
    if (ring < 2) {
        ring = 2;
        while (T > 32 && acc_b(T) > budget - 2ll * kStageBytes) T -= 32;
    }
    T = T / 32 * 32;
    s.ring = (int)ring;
    if (acc_b(T) + ring * (long long)kStageBytes > budget) T = 0;
    if (T < 32) return fail(SNP_ERR_CAPACITY, "not enough shared memory for the tiled kernel");
    if (!getenv("SNPB200_TILE") && q > T) {
        // whole rounds: the CTA with the most tiles sets the step time, so a
        // partial last round is spread over all CTAs (smaller tiles, same
        // number of rounds; e.g. 10^8 neurons: 1199 -> 1332 tiles, 9 each)
        const long long rounds = ceil_div(ceil_div(q, T), (long long)n_sm);
        const long long T2 = (ceil_div(q, rounds * n_sm) + 31) / 32 * 32;
        if (T2 >= 32 && T2 < T) T = T2;
    }
    const long long n_tiles = std::max<long long>(1, ceil_div(q, T));
    s.tile = (int)T;
    s.n_tiles = n_tiles;
    s.pf = 0;  // measured: L2 prefetch ahead of the ring does not help (profiles/r1_history.md)
    if (const char* env = getenv("SNPB200_PREFETCH")) s.pf = std::max(0, atoi(env));
    s.dbg = 0;
    if (const char* env = getenv("SNPB200_DEBUG_SKIP")) s.dbg = atoi(env);
    if (const char* env = getenv("SNPB200_PDL")) e->pdl = atoi(env) != 0;
    // regular rule counts: offsets are implicit (rpn * local neuron)
    s.rpn = 0;
    if (q > 0) {
        const long long r = roff_h[1] - roff_h[0];
        bool regular = r >= 1 && r <= (long long)kLightRules;
        for (long long i = 0; i < q && regular; ++i) regular = (long long)roff_h[i] == r * i;
        regular = regular && (long long)roff_h[q] == r * q;
        if (const char* env = getenv("SNPB200_RPN")) regular = regular && atoi(env) != 0;
        if (regular) s.rpn = (int)r;
    }
    // P_BIT: stage the P-bit window of a stage's sources with its segments
    // (SNPB200_PSTAGE=0: look the bits up through L1/L2 instead)
    bool stage_p = e->p_mode == P_BIT;
    if (const char* env = getenv("SNPB200_PSTAGE")) stage_p = stage_p && atoi(env) != 0;
    // heavy-rule neurons per tile (heavy is ascending)
    {
        std::vector<uint32_t> theavy(n_tiles + 1, 0);
        for (uint32_t hn : heavy) theavy[hn / T + 1]++;
        for (long long t = 0; t < n_tiles; ++t) theavy[t + 1] += theavy[t];
        uint32_t* d_theavy;
        TRY(upload(e, &d_theavy, theavy));
        s.theavy = d_theavy;
    }
    // the layout itself: on the device (default for a single engine with its
    // out-adjacency on the device), or the host reference build below
    if (s.tp) return build_tiles2(e, d_soff, d_sdst, soff, sdst, sh, roff_h);
    bool dev_build = !sh && d_soff && d_sdst && sdst.size() < (1ull << 31);
    if (const char* env = getenv("SNPB200_DEVICE_BUILD")) dev_build = dev_build && atoi(env) != 0;
    if (dev_build) return build_tiles_device(e, d_soff, d_sdst, (long long)sdst.size(), stage_p);
    // bucket the edges into local destination tiles (source order preserved)
    std::vector<unsigned long long> start(n_tiles + 1, 0);
    for (size_t e2 = 0; e2 < sdst.size(); ++e2)
        if ((long long)sdst[e2] >= lo && (long long)sdst[e2] < hi) start[(sdst[e2] - lo) / T + 1]++;
    for (long long t = 0; t < n_tiles; ++t) start[t + 1] += start[t];
    const long long S = (long long)start[n_tiles];
    std::vector<unsigned long long> cur(start.begin(), start.end() - 1);
    std::vector<uint32_t> bsrc(S);
    std::vector<uint32_t> bslot(S);
    for (long long i = 0; i < n_src; ++i) {
        const uint32_t xs = sh ? sh->xpos((uint32_t)i) : (uint32_t)i;
        for (uint32_t e2 = soff[i]; e2 < soff[i + 1]; ++e2) {
            const long long dst = sdst[e2];
            if (dst < lo || dst >= hi) continue;
            const unsigned long long pos = cur[(dst - lo) / T]++;
            bsrc[pos] = xs;
            bslot[pos] = (uint32_t)((dst - lo) % T);
        }
    }
    // segments
    std::vector<uint32_t> tseg(n_tiles + 1, 0), base, last;
    std::vector<uint32_t> words;
    words.reserve((size_t)(S + S / 8 + 256));
    for (long long t = 0; t < n_tiles; ++t) {
        unsigned long long e2 = start[t];
        const unsigned long long end = start[t + 1];
        while (e2 < end) {
            // bases are multiples of 32 so that an offset's low 5 bits index
            // the bit inside a P word (tiled_step_kernel phase 1)
            const uint32_t b = bsrc[e2] & ~31u;
            base.push_back(b);
            int n = 0;
            while (e2 < end && n < kSegEdges && bsrc[e2] - b < kSrcSpan) {
                words.push_back(((uint32_t)bslot[e2] << kSrcBits) | (bsrc[e2] - b));
                ++e2;
                ++n;
            }
            last.push_back(bsrc[e2 - 1]);
            // padding: source offset 0 (inside the window), dummy counter slot T
            for (; n < kSegEdges; ++n) words.push_back((uint32_t)T << kSrcBits);
        }
        tseg[t + 1] = (uint32_t)base.size();
        if (words.size() >= (1ull << 32)) return fail(SNP_ERR_CAPACITY, "tiled layout exceeds 2^32 words");
    }
    // TMA stage descriptors (see tiled_step_kernel): phase-1 stages take as
    // many consecutive segments as fit with the P window they reference,
    // phase-2 stages kSub destinations with (when they fit) their rule words
    std::vector<StageDesc> desc;
    std::vector<uint32_t> tstage(n_tiles + 1, 0), sbases;
    auto r16 = [](unsigned long long x) { return (uint32_t)((x + 15) & ~15ull); };
    for (long long t = 0; t < n_tiles; ++t) {
        uint32_t g = tseg[t];
        const uint32_t g1 = tseg[t + 1];
        do {
            uint32_t n = 0, src0 = 0, pbytes = 0;
            if (g < g1) {
                src0 = base[g] & ~127u;
                while (g + n < g1 && n < kMaxSegPerStage) {
                    const uint32_t pb = stage_p ? r16((last[g + n] + 1u - src0 + 7u) / 8u) : 0u;
                    if (kPayload + (n + 1) * kSegEdges * 4u + pb > kStageBytes) break;
                    pbytes = pb;
                    ++n;
                }
            }
            const uint32_t boff = (uint32_t)sbases.size();
            for (uint32_t i = 0; i < n; ++i) sbases.push_back(base[g + i]);
            while (sbases.size() % 4) sbases.push_back(0);
            StageDesc sd;
            sd.a = make_uint4(1u | ((g + n >= g1) ? 256u : 0u), g, n, src0);
            sd.b = make_uint4(pbytes, boff, 0, 0);
            desc.push_back(sd);
            g += n;
        } while (g < g1);
        append_phase2_desc(e, t, roff_h, desc);
        tstage[t + 1] = (uint32_t)desc.size();
    }
    StageDesc* d_desc;
    uint32_t *d_tstage, *d_sbases;
    TRY(upload(e, &d_desc, desc));
    TRY(upload(e, &d_tstage, tstage));
    sbases.resize(sbases.size() + 4, 0);
    TRY(upload(e, &d_sbases, sbases));
    s.stages = d_desc;
    s.tstage = d_tstage;
    s.stage_bases = d_sbases;
    e->n_stages = (long long)desc.size();
    e->n_sbases = (long long)sbases.size();

    uint32_t *d_words, *d_base, *d_tseg;
    TRY(upload(e, &d_words, words));
    TRY(upload(e, &d_base, base));
    TRY(upload(e, &d_tseg, tseg));
    s.seg_words = d_words;
    s.seg_base = d_base;
    s.tseg = d_tseg;
    e->in_edges = (long long)words.size();
    return SNP_OK;
}

// Scratch device allocations freed at scope exit.
struct TmpAllocs {
    std::vector<void*> p;
    ~TmpAllocs() {
        for (void* x : p) cudaFree(x);
    }
    template <typename X>
    cudaError_t get(X** out, long long n) {
        void* v = nullptr;
        cudaError_t err = cudaMalloc(&v, (size_t)std::max<long long>(n, 1) * sizeof(X));
        if (err == cudaSuccess) p.push_back(v);
        *out = static_cast<X*>(v);
        return err;
    }
};

// Device build of the same layout (snp_ingest.cuh).  Temporaries are freed
// before returning; only the layout arrays stay with the engine.
int build_tiles_device(snp_engine* e, const uint32_t* d_soff, const uint32_t* d_sdst, long long S, bool stage_p) {
    DevSys& s = e->sys;
    const long long q = e->q, n_tiles = s.n_tiles;
    const uint32_t T = (uint32_t)s.tile;
    TmpAllocs tmp;
    // 1-2: keys, stable sort by tile
    uint32_t *k_in, *k_out;
    unsigned long long *v_in, *v_out, *tstart;
    CU(tmp.get(&k_in, S));
    CU(tmp.get(&k_out, S));
    CU(tmp.get(&v_in, S));
    CU(tmp.get(&v_out, S));
    CU(tmp.get(&tstart, n_tiles + 1));
    if (q > 0) ingest_keys_kernel<<<grid_for(q), 256>>>(q, d_soff, d_sdst, T, k_in, v_in);
    CU(cudaGetLastError());
    int bits = 1;
    while ((1ll << bits) <= n_tiles) ++bits;
    size_t temp_bytes = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, k_in, k_out, v_in, v_out, (int)S, 0, bits));
    void* temp;
    CU(tmp.get(reinterpret_cast<unsigned char**>(&temp), (long long)temp_bytes));
    if (S > 0) CU(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k_in, k_out, v_in, v_out, (int)S, 0, bits));
    ingest_tile_starts_kernel<<<grid_for(n_tiles + 1), 256>>>(S, k_out, n_tiles, tstart);
    CU(cudaGetLastError());
    // 3: segments (count, scan on the host, fill), words
    const int wgrid = (int)std::max<long long>(1, std::min<long long>(ceil_div(n_tiles * 32, 256), 148ll * 8));
    uint32_t* segc;
    CU(tmp.get(&segc, n_tiles));
    ingest_segments_kernel<<<wgrid, 256>>>(n_tiles, tstart, v_out, 0, segc, nullptr, nullptr, nullptr, nullptr, nullptr);
    CU(cudaGetLastError());
    std::vector<uint32_t> counts(n_tiles), tseg(n_tiles + 1, 0);
    CU(cudaMemcpy(counts.data(), segc, n_tiles * 4, cudaMemcpyDeviceToHost));
    for (long long t = 0; t < n_tiles; ++t) tseg[t + 1] = tseg[t] + counts[t];
    const long long nseg = tseg[n_tiles];
    if (nseg * (long long)kSegEdges >= (1ll << 32)) return fail(SNP_ERR_CAPACITY, "tiled layout exceeds 2^32 words");
    uint32_t *d_tseg, *d_words, *d_base, *d_last, *d_segn;
    unsigned long long* d_first;
    TRY(upload(e, &d_tseg, tseg));
    TRY(e->alloc(&d_words, nseg * kSegEdges));
    TRY(e->alloc(&d_base, nseg));
    CU(tmp.get(&d_last, nseg));
    CU(tmp.get(&d_segn, nseg));
    CU(tmp.get(&d_first, nseg));
    ingest_segments_kernel<<<wgrid, 256>>>(n_tiles, tstart, v_out, 1, nullptr, d_tseg, d_first, d_segn, d_base, d_last);
    CU(cudaGetLastError());
    if (nseg > 0)
        ingest_words_kernel<<<(int)std::min<long long>(ceil_div(nseg * 32, 256), 148ll * 64), 256>>>(
            nseg, d_first, d_segn, d_base, v_out, T, d_words);
    CU(cudaGetLastError());
    // 4: stage descriptors (count, scan, fill)
    IngestStageParams P{q, T, stage_p ? 1 : 0, s.rpn, e->tiny_rules ? 1 : 0, e->wide_rules ? 1 : 0, s.roff};
    uint32_t *nst, *nsb;
    CU(tmp.get(&nst, n_tiles));
    CU(tmp.get(&nsb, n_tiles));
    ingest_stages_kernel<<<wgrid, 256>>>(n_tiles, d_tseg, d_base, d_last, P, 0, nst, nsb, nullptr, nullptr, nullptr,
                                         nullptr);
    CU(cudaGetLastError());
    std::vector<uint32_t> cst(n_tiles), csb(n_tiles), tstage(n_tiles + 1, 0), tsbase(n_tiles + 1, 0);
    CU(cudaMemcpy(cst.data(), nst, n_tiles * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(csb.data(), nsb, n_tiles * 4, cudaMemcpyDeviceToHost));
    for (long long t = 0; t < n_tiles; ++t) {
        tstage[t + 1] = tstage[t] + cst[t];
        tsbase[t + 1] = tsbase[t] + csb[t];
    }
    uint32_t *d_tstage, *d_tsbase, *d_sbases;
    StageDesc* d_desc;
    TRY(upload(e, &d_tstage, tstage));
    CU(tmp.get(&d_tsbase, n_tiles + 1));
    CU(cudaMemcpy(d_tsbase, tsbase.data(), (n_tiles + 1) * 4, cudaMemcpyHostToDevice));
    TRY(e->alloc(&d_desc, tstage[n_tiles]));
    TRY(e->alloc(&d_sbases, (long long)tsbase[n_tiles] + 4));
    CU(cudaMemset(d_sbases, 0, ((size_t)tsbase[n_tiles] + 4) * 4));
    ingest_stages_kernel<<<wgrid, 256>>>(n_tiles, d_tseg, d_base, d_last, P, 1, nullptr, nullptr, d_tstage, d_tsbase,
                                         d_desc, d_sbases);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
    s.seg_words = d_words;
    s.seg_base = d_base;
    s.tseg = d_tseg;
    s.stages = d_desc;
    s.tstage = d_tstage;
    s.stage_bases = d_sbases;
    e->in_edges = nseg * kSegEdges;
    e->n_stages = tstage[n_tiles];
    e->n_sbases = (long long)tsbase[n_tiles] + 4;
    return SNP_OK;
}

// Two-pass layout (variant TILED2, snp_ingest.cuh): edges sorted by (tile,
// source window) on the device; per 32-edge group a tile-order slot block
// and a window-order offset block; host-side scans of the small per-chunk
// counts; phase-1 stage descriptors are runs of groups.
int build_tiles2(snp_engine* e, const uint32_t* d_soff, const uint32_t* d_sdst, const hvec<uint32_t>& soff,
                 const hvec<uint32_t>& sdst, const ShardInput* sh, const std::vector<uint32_t>& roff_h) {
    DevSys& s = e->sys;
    const long long q = e->q, nt = s.n_tiles, T = s.tile;
    if (T > 65535 - 1) return fail(SNP_ERR_CAPACITY, "two-pass tiles need T < 65535");
    const long long space = sh ? (long long)sh->world * (sh->nl + 128) : std::max<long long>(q, 1);
    int wlog = 12;
    while (wlog < 16 && (1ll << wlog) < 32 * space / std::max<long long>(T, 1)) ++wlog;
    if (const char* env = getenv("SNPB200_WINDOW_LOG")) wlog = std::min(16, std::max(5, atoi(env)));
    const long long nw = ceil_div(space, 1ll << wlog);
    const long long nk = nt * nw;
    if (nk >= (1ll << 32) - 1) return fail(SNP_ERR_CAPACITY, "two-pass layout: tiles x windows exceeds 2^32");
    TmpAllocs tmp;
    // edges -> keys / values on the device
    long long S;
    uint32_t *k_in, *k_out;
    unsigned long long *v_in, *v_out;
    if (!sh) {
        S = (long long)sdst.size();
        CU(tmp.get(&k_in, S));
        CU(tmp.get(&v_in, S));
        if (q > 0 && S > 0)
            tp_keys_csr_kernel<<<grid_for(q), 256>>>(q, d_soff, d_sdst, (uint32_t)T, (uint32_t)wlog, (uint32_t)nw, k_in, v_in);
    } else {
        std::vector<uint32_t> xs, ld;
        for (long long i = 0; i < sh->q_global; ++i) {
            const uint32_t x = sh->xpos((uint32_t)i);
            for (uint32_t e2 = soff[i]; e2 < soff[i + 1]; ++e2) {
                const long long dst = sdst[e2];
                if (dst < sh->lo || dst >= sh->hi) continue;
                xs.push_back(x);
                ld.push_back((uint32_t)(dst - sh->lo));
            }
        }
        S = (long long)xs.size();
        uint32_t *d_xs, *d_ld;
        CU(tmp.get(&d_xs, S));
        CU(tmp.get(&d_ld, S));
        CU(cudaMemcpy(d_xs, xs.data(), S * 4, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(d_ld, ld.data(), S * 4, cudaMemcpyHostToDevice));
        CU(tmp.get(&k_in, S));
        CU(tmp.get(&v_in, S));
        if (S > 0)
            tp_keys_list_kernel<<<grid_for(S), 256>>>(S, d_xs, d_ld, (uint32_t)T, (uint32_t)wlog, (uint32_t)nw, k_in, v_in);
    }
    CU(cudaGetLastError());
    if (S >= (1ll << 31)) return fail(SNP_ERR_CAPACITY, "two-pass layout: more than 2^31 in-edges");
    CU(tmp.get(&k_out, S));
    CU(tmp.get(&v_out, S));
    int bits = 1;
    while ((1ll << bits) <= nk) ++bits;
    size_t temp_bytes = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, k_in, k_out, v_in, v_out, (int)S, 0, bits));
    unsigned char* temp;
    CU(tmp.get(&temp, (long long)temp_bytes));
    if (S > 0) CU(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k_in, k_out, v_in, v_out, (int)S, 0, bits));
    // per-chunk counts and the three offset tables (host scans)
    uint32_t* d_cnt;
    CU(tmp.get(&d_cnt, nk));
    CU(cudaMemset(d_cnt, 0, nk * 4));
    if (S > 0) tp_hist_kernel<<<grid_for(S), 256>>>(S, k_out, d_cnt);
    CU(cudaGetLastError());
    std::vector<uint32_t> cnt(nk);
    CU(cudaMemcpy(cnt.data(), d_cnt, nk * 4, cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> off_raw(nk + 1, 0), off2(nk + 1, 0), off1(nk + 1, 0);
    for (long long k = 0; k < nk; ++k) {
        off_raw[k + 1] = off_raw[k] + cnt[k];
        off2[k + 1] = off2[k] + ((cnt[k] + 31ull) & ~31ull);
    }
    {
        unsigned long long acc = 0;
        for (long long w = 0; w < nw; ++w)
            for (long long t = 0; t < nt; ++t) {
                off1[w * nt + t] = acc;
                acc += (cnt[t * nw + w] + 31ull) & ~31ull;
            }
        off1[nk] = acc;
    }
    const long long edges = (long long)off2[nk], groups = edges / 32;
    if (edges >= (1ll << 32)) return fail(SNP_ERR_CAPACITY, "two-pass layout exceeds 2^32 edge slots");
    unsigned long long *d_raw, *d_off2, *d_off1;
    CU(tmp.get(&d_raw, nk + 1));
    CU(tmp.get(&d_off2, nk + 1));
    CU(tmp.get(&d_off1, nk + 1));
    CU(cudaMemcpy(d_raw, off_raw.data(), (nk + 1) * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_off2, off2.data(), (nk + 1) * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_off1, off1.data(), (nk + 1) * 8, cudaMemcpyHostToDevice));
    uint16_t *d_slots, *d_offs;
    uint32_t *d_gword, *d_bits;
    TRY(e->alloc(&d_slots, edges + 64));
    TRY(e->alloc(&d_offs, edges + 64));
    TRY(e->alloc(&d_gword, groups + 4));
    TRY(e->alloc(&d_bits, groups + 8));
    CU(cudaMemset(d_bits, 0, (groups + 8) * 4));
    CU(cudaMemset(d_offs, 0, (edges + 64) * 2));
    fill_u16_kernel<<<grid_for(std::min<long long>(edges + 64, 148ll * 4096)), 256>>>(edges + 64, d_slots, (uint16_t)T);
    CU(cudaGetLastError());
    if (S > 0)
        tp_fill_kernel<<<grid_for(S), 256>>>(S, k_out, v_out, d_raw, d_off2, d_off1, (uint32_t)nt, (uint32_t)nw,
                                             (uint32_t)wlog, d_slots, d_offs);
    tp_gword_kernel<<<grid_for(nk), 256>>>(nk, d_cnt, d_off2, d_off1, (uint32_t)nt, (uint32_t)nw, d_gword);
    CU(cudaGetLastError());
    // window -> first group (window order), tile -> group range (tile order)
    std::vector<uint32_t> wgroup(nw + 1), tgroup(nt + 1);
    for (long long w = 0; w <= nw; ++w) wgroup[w] = (uint32_t)(off1[std::min<long long>(w * nt, nk)] / 32);
    for (long long t = 0; t <= nt; ++t) tgroup[t] = (uint32_t)(off2[std::min<long long>(t * nw, nk)] / 32);
    uint32_t* d_wgroup;
    TRY(upload(e, &d_wgroup, wgroup));
    // pass-1 work items: windows cut into runs of <= 1024 groups
    std::vector<uint4> items;
    for (long long w = 0; w < nw; ++w)
        for (uint32_t g = wgroup[w]; g < wgroup[w + 1]; g += 1024)
            items.push_back(make_uint4((uint32_t)w, g, std::min<uint32_t>(g + 1024, wgroup[w + 1]), 0));
    uint4* d_items;
    TRY(upload(e, &d_items, items));
    s.tp_items = d_items;
    s.tp_nitems = (long long)items.size();
    // stage descriptors: phase-1 runs of groups, then the phase-2 stages
    const uint32_t G = (kStageBytes - kPayload - 32) / 68;
    std::vector<StageDesc> desc;
    std::vector<uint32_t> tstage(nt + 1, 0);
    for (long long t = 0; t < nt; ++t) {
        uint32_t g = tgroup[t];
        const uint32_t g1 = tgroup[t + 1];
        do {
            const uint32_t n = std::min<uint32_t>(G, g1 - g);
            StageDesc sd;
            sd.a = make_uint4(3u | ((g + n >= g1) ? 256u : 0u), g, n, 0);
            sd.b = make_uint4(0, 0, 0, 0);
            desc.push_back(sd);
            g += n;
        } while (g < g1);
        append_phase2_desc(e, t, roff_h, desc);
        tstage[t + 1] = (uint32_t)desc.size();
    }
    StageDesc* d_desc;
    uint32_t *d_tstage, *d_sb;
    TRY(upload(e, &d_desc, desc));
    TRY(upload(e, &d_tstage, tstage));
    TRY(e->alloc(&d_sb, 4));
    CU(cudaMemset(d_sb, 0, 16));
    CU(cudaDeviceSynchronize());
    s.stages = d_desc;
    s.tstage = d_tstage;
    s.stage_bases = d_sb;
    s.tp_wlog = wlog;
    s.tp_nw = nw;
    s.tp_slots = d_slots;
    s.tp_bits = d_bits;
    s.tp_off = d_offs;
    s.tp_gword = d_gword;
    s.tp_wgroup = d_wgroup;
    e->in_edges = edges;
    e->n_stages = (long long)desc.size();
    e->p1_grid = (int)std::max<long long>(1, std::min<long long>((long long)items.size(), 148ll * 4));
    return SNP_OK;
}

// Build every device structure.  Host-side work is O(q + m + S) with plain
// loops; the quadratic layouts (ELL pairs, dense rows) and the in-adjacency
// transpose are built on the device.
template <int PM>
void pick_tiled(snp_engine* e) {
    const int rw = e->wide_rules ? RW_WIDE : (e->tiny_rules ? RW_TINY : RW_COMPACT);
    tiled_fns<PM>(rw, e->cbits, &e->step_fn, &e->lean_fn);
    e->prime_fn = prime_kernel<RECV_PULL, PM, true, false>;
}

// The step kernel instance for the current run parameters: the lean tiled
// instance when nothing is recorded or counted.
StepFn run_fn(const snp_engine* e) {
    if (e->fused_fn) return e->fused_fn;
    if (e->lean_fn && e->hctrl.record == 0 && !e->hctrl.stats_on) return e->lean_fn;
    return e->step_fn;
}

// The step kernel of a run (the one-kernel push step when the engine has one).
void launch_main(snp_engine* e) {
    if (e->small_fn) {
        e->small_fn<<<1, kSmallThreads, e->small_smem, e->stream>>>(e->sys, e->st);
    } else if (e->fused_fn) {
        e->fused_fn<<<e->fused_grid, e->fused_block, e->fused_smem, e->stream>>>(e->sys, e->st);
    } else if (e->tiled && e->pdl) {
        // programmatic dependent launch: the step kernel's CTAs are scheduled
        // while the previous step's grid drains and wait in griddepcontrol.wait
        // (full completion + visibility of the previous grid) -- hides the
        // launch gap between consecutive steps
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(e->step_grid);
        cfg.blockDim = dim3(e->step_block);
        cfg.dynamicSmemBytes = e->step_smem;
        cfg.stream = e->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, run_fn(e), e->sys, e->st);
    } else {
        run_fn(e)<<<e->step_grid, e->step_block, e->step_smem, e->stream>>>(e->sys, e->st);
    }
}

// SNPB200_TIMING=1: per-phase host timings of engine creation on stderr
struct PhaseTimer {
    bool on = getenv("SNPB200_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    PhaseTimer() { nvtxRangePushA("snp_engine_create"); }
    ~PhaseTimer() { nvtxRangePop(); }
    void mark(const char* what) {
        nvtxMarkA(what);
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[snpb200 build] %-28s %8.1f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// Dynamic shared memory cap of a kernel: the device's opt-in maximum, not
// this engine's size -- the attribute is per function, so engines of
// different sizes in one process must not lower it under each other.
int allow_max_smem(const void* fn, int device, size_t needed) {
    int optin = 0;
    CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    cudaFuncAttributes fa;
    CU(cudaFuncGetAttributes(&fa, fn));
    const int cap = std::max((int)needed, optin - (int)fa.sharedSizeBytes);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, cap) != cudaSuccess) {
        cudaGetLastError();  // a tool (e.g. racecheck) may reserve shared memory: fall back to this engine's size
        if (fa.maxDynamicSharedSizeBytes < (int)needed)
            CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)needed));
    }
    return SNP_OK;
}

int build(snp_engine* e, const snp_system_desc* d, const ShardInput* sh = nullptr) {
    PhaseTimer tm;
    const long long q = d->q, m = d->m;
    if (q < 0 || m < 0) return fail(SNP_ERR_BAD_ARG, "q and m must be >= 0");
    if (q >= kInt32Max) return fail(SNP_ERR_CAPACITY, "q=%lld exceeds the int32 neuron index range", q);
    if (m >= (1ll << 32) - 1) return fail(SNP_ERR_CAPACITY, "m=%lld exceeds the uint32 rule index range", m);
    if (q > 0 && (!d->initial || !d->offsets)) return fail(SNP_ERR_BAD_ARG, "initial/offsets missing");
    if (m > 0 && (!d->threshold || !d->is_exact || !d->consumed || !d->produced || !d->delay))
        return fail(SNP_ERR_BAD_ARG, "rule vector arrays missing");
    e->q = q;
    e->m = m;
    e->format = d->format;
    e->initial.assign(d->initial, d->initial + q);
    for (long long i = 0; i < q; ++i)
        if (d->initial[i] < 0) return fail(SNP_ERR_BAD_ARG, "initial spike count of neuron %lld is negative", i);

    // --- rule vector + offsets (matrices.py:48-73, 115-140)
    if (q > 0 && d->offsets[0] != 0) return fail(SNP_ERR_BAD_ARG, "offsets[0] must be 0");
    // +8 tail: the TMA stages of the tiled kernel copy whole 16-byte units
    std::vector<uint32_t> roff(q + 1 + 8, 0);
    hvec<uint32_t> owner(m);  // every rule's owner is written below
    if (parallel_first_fail(q, [&](long long a0, long long a1) -> long long {
            for (long long i = a0; i < a1; ++i) {
                const long long a = d->offsets[i], b = d->offsets[i + 1];
                if (b < a || b > m) return i;
                roff[i + 1] = (uint32_t)b;
                for (long long r = a; r < b; ++r) owner[r] = (uint32_t)i;
            }
            return -1;
        }) >= 0)
        return fail(SNP_ERR_BAD_ARG, "offsets not non-decreasing within [0, m]");
    if ((q > 0 ? d->offsets[q] : 0) != m) return fail(SNP_ERR_BAD_ARG, "offsets[q] != m");
    hvec<uint32_t> rthr(m);
    hvec<int4> rrec(m);
    const long long bad_rule = parallel_first_fail(m, [&](long long a, long long b) -> long long {
        for (long long r = a; r < b; ++r) {
            const long long t = d->threshold[r], c = d->consumed[r], p = d->produced[r], dl = d->delay[r];
            if (t < 0 || t > kInt32Max || c < 0 || c > kInt32Max || p < 0 || p > kInt32Max || dl < 0 ||
                dl > kInt32Max - 2)
                return r;
            rthr[r] = (uint32_t)t | (d->is_exact[r] ? kExactBit : 0u);
            rrec[r] = make_int4((int)c, (int)p, (int)dl, 0);
        }
        return -1;
    });
    if (bad_rule >= 0) {
        const long long r = bad_rule, t = d->threshold[r], dl = d->delay[r];
        if (t < 0 || t > kInt32Max) return fail(SNP_ERR_CAPACITY, "rule %lld threshold %lld outside [0, 2^31-1]", r, t);
        const long long c = d->consumed[r], p = d->produced[r];
        if (c < 0 || c > kInt32Max || p < 0 || p > kInt32Max)
            return fail(SNP_ERR_CAPACITY, "rule %lld consumed/produced outside [0, 2^31-1]", r);
        return fail(SNP_ERR_CAPACITY, "rule %lld delay %lld outside [0, 2^31-3]", r, dl);
    }
    // compact rule words possible? largest / common produced amount (one
    // pass per host thread, then merged in order)
    bool compact = true;
    long long pmax = 0, pfirst = -1;
    bool pcommon = true;
    {
        const int nt = (int)std::max<long long>(1, std::min<long long>(std::max(1u, std::thread::hardware_concurrency()),
                                                                       m / (1 << 16) + 1));
        struct Part {
            bool compact = true, pcommon = true;
            long long pmax = 0, pfirst = -1;
        };
        std::vector<Part> parts(nt);
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                Part& P = parts[t];
                for (long long r = m * t / nt; r < m * (t + 1) / nt; ++r) {
                    const int4 x = rrec[r];
                    if (x.x >= 65536 || x.y >= 256 || x.z >= 256) P.compact = false;
                    if (x.y > 0) {
                        P.pmax = std::max<long long>(P.pmax, x.y);
                        if (P.pfirst < 0) P.pfirst = x.y;
                        else if (x.y != P.pfirst) P.pcommon = false;
                    }
                }
            });
        for (auto& x : th) x.join();
        for (const Part& P : parts) {
            compact = compact && P.compact;
            pmax = std::max(pmax, P.pmax);
            pcommon = pcommon && P.pcommon;
            if (P.pfirst >= 0) {
                if (pfirst < 0) pfirst = P.pfirst;
                else if (P.pfirst != pfirst) pcommon = false;
            }
        }
    }

    if (sh && sh->x_pbits) {
        // row partition: every rank must use the same exchange width (and, for
        // P bits, the same common amount), agreed over all ranks by the caller
        const int xb = sh->x_pbits;
        if (xb != 1 && xb != 8 && xb != 16 && xb != 32)
            return fail(SNP_ERR_BAD_ARG, "x_pbits must be 1, 8, 16 or 32, got %d", xb);
        if (pmax > sh->x_pmax || (xb == 1 && pfirst >= 0 && (!pcommon || pfirst != sh->x_pmax)))
            return fail(SNP_ERR_BAD_ARG, "this rank's produced amounts disagree with the agreed exchange (x_pbits=%d, "
                        "x_pmax=%lld)", xb, sh->x_pmax);
        const long long cap = xb == 1 ? (1ll << 31) : (xb == 32 ? (1ll << 32) : (1ll << xb));
        if (sh->x_pmax < 1 || sh->x_pmax >= cap)
            return fail(SNP_ERR_BAD_ARG, "x_pmax=%lld does not fit x_pbits=%d", sh->x_pmax, xb);
        pcommon = xb == 1;
        pfirst = sh->x_pmax;
        pmax = sh->x_pmax;
    }

    tm.mark("rule vector");
    // --- transition structure
    hvec<uint32_t> soff, sdst;
    bool have_adj = false;
    if (d->adj_offsets) {
        soff.resize(q + 1);
        TRY(check_csr_offsets(d->adj_offsets, q));
        const long long S = q > 0 ? d->adj_offsets[q] : 0;
        if (S >= (1ll << 32) - 1) return fail(SNP_ERR_CAPACITY, "synapse count %lld exceeds uint32", S);
        sdst.resize(S);
        parallel_first_fail(q + 1, [&](long long a, long long b) -> long long {
            for (long long i = a; i < b; ++i) soff[i] = (uint32_t)d->adj_offsets[i];
            return -1;
        });
        const long long bad = parallel_first_fail(S, [&](long long a, long long b) -> long long {
            for (long long x = a; x < b; ++x) {
                const long long t = d->adj_targets[x];
                if (t < 0 || t >= q) return x;
                sdst[x] = (uint32_t)t;
            }
            return -1;
        });
        if (bad >= 0) return fail(SNP_ERR_BAD_ARG, "synapse target %lld out of range", (long long)d->adj_targets[bad]);
        have_adj = true;
    } else if (d->syn_target && e->format == SNP_FMT_COMPRESSED) {
        // SynapseMatrix [rows][q]: the first NULL ends a column (matrices.py:100-112)
        soff.assign(q + 1, 0);
        for (long long i = 0; i < q; ++i) {
            long long n = 0;
            while (n < d->syn_rows && d->syn_target[n * q + i] >= 0) ++n;
            soff[i + 1] = soff[i] + (uint32_t)n;
        }
        sdst.resize(soff[q]);
        for (long long i = 0; i < q; ++i)
            for (uint32_t n = 0; n < soff[i + 1] - soff[i]; ++n) {
                const long long t = d->syn_target[(long long)n * q + i];
                if (t >= q) return fail(SNP_ERR_BAD_ARG, "synapse target %lld out of range", t);
                sdst[soff[i] + n] = (uint32_t)t;
            }
        have_adj = true;
    }
    int z = 0;
    std::vector<uint32_t> outdeg(q, 0);
    if (have_adj)
        for (long long i = 0; i < q; ++i) {
            outdeg[i] = soff[i + 1] - soff[i];
            z = std::max<int>(z, (int)outdeg[i]);
        }

    const bool ell_from_matrix = e->format == SNP_FMT_ELL && !have_adj;
    const bool dense_from_matrix = e->format == SNP_FMT_SPARSE && !have_adj;
    if (sh) {
        // local out-degrees (traffic counters) from the global adjacency
        for (long long i = 0; i < q; ++i) {
            outdeg[i] = sh->soff[sh->lo + i + 1] - sh->soff[sh->lo + i];
            z = std::max<int>(z, (int)outdeg[i]);
        }
    } else if (e->format == SNP_FMT_COMPRESSED && !have_adj && q > 0) {
        return fail(SNP_ERR_BAD_ARG, "COMPRESSED needs adj_offsets/adj_targets or syn_target");
    }
    if (ell_from_matrix && m > 0 && !(d->ell_target && d->ell_amount))
        return fail(SNP_ERR_BAD_ARG, "ELL needs adj_offsets/adj_targets or ell_target/ell_amount");
    if (dense_from_matrix && m > 0 && q > 0 && !d->sparse_data)
        return fail(SNP_ERR_BAD_ARG, "SPARSE needs adj_offsets/adj_targets or sparse_data");

    std::vector<int2> ell_host;
    std::vector<uint32_t> ell_len_host;
    long long ell_ld = 0;
    if (ell_from_matrix) {
        const long long rows = d->ell_rows;
        z = (int)std::max<long long>(0, rows - 1);
        ell_ld = std::max<long long>(2, (rows + 1) & ~1ll);  // 16-byte aligned columns
        ell_host.assign((size_t)(m * ell_ld), make_int2(-1, 0));
        ell_len_host.assign(m, 0);
        for (long long r = 0; r < m; ++r) {
            long long n = 0;
            while (n < rows && d->ell_target[n * m + r] >= 0) {
                const long long t = d->ell_target[n * m + r], a = d->ell_amount[n * m + r];
                if (t >= q) return fail(SNP_ERR_BAD_ARG, "ELL target %lld out of range", t);
                if (a < -kInt32Max || a > kInt32Max) return fail(SNP_ERR_CAPACITY, "ELL amount %lld outside int32", a);
                ell_host[r * ell_ld + n] = make_int2((int)t, (int)a);
                ++n;
            }
            ell_len_host[r] = (uint32_t)n;
            outdeg[owner[r]] = std::max<uint32_t>(outdeg[owner[r]], (uint32_t)std::max<long long>(0, n - 1));
        }
    }
    e->z = z;

    tm.mark("transition structure");
    // --- receive path and P width
    e->variant = d->variant;
    if (e->format == SNP_FMT_COMPRESSED) {
        // small systems: one CTA runs whole loop segments (small_run_kernel)
        const bool small_ok = !sh && q <= kSmallMaxQ && (long long)sdst.size() + m <= (1ll << 17);
        if (e->variant == SNP_VARIANT_AUTO && small_ok && q > 0) e->variant = SNP_VARIANT_SMALL;
        // no neurons: nothing to tile (a zero-CTA grid never decides the
        // halt); the one-CTA kernel decides NO_APPLICABLE_RULES at step 0
        if (q == 0 && !sh && e->variant != SNP_VARIANT_PULL && e->variant != SNP_VARIANT_PUSH)
            e->variant = SNP_VARIANT_SMALL;
        if (e->variant == SNP_VARIANT_SMALL && (sh || q > kSmallMaxQ))
            return fail(SNP_ERR_BAD_ARG, "variant SMALL needs an unpartitioned system of <= %lld neurons", kSmallMaxQ);
        if (e->variant == SNP_VARIANT_AUTO) {
            // tiled, heavy-rule systems included: with the dense
            // FirstApplicable table the sorter n=4096 steps in 0.057 ms tiled
            // vs 0.080 ms in the CSR pull (SeededRandom: 0.169 vs 0.154; the
            // reference's default policy is FirstApplicable, engine.py:118)
            e->variant = SNP_VARIANT_TILED;
            // a destination that can receive >= 2^32 spikes per step (several
            // large produced amounts) needs the 64-bit gather of the CSR pull
            if (!sh && !pcommon && (double)pmax * (double)sdst.size() >= 4294967296.0) {
                std::vector<uint32_t> indeg(std::max<long long>(q, 1), 0);
                uint32_t mx = 0;
                for (uint32_t t : sdst) mx = std::max(mx, ++indeg[t]);
                if ((double)pmax * (double)mx >= 4294967296.0) e->variant = SNP_VARIANT_PULL;
            }
        }
        e->kind = (e->variant == SNP_VARIANT_PUSH || e->variant == SNP_VARIANT_SMALL) ? RECV_ARRAY : RECV_PULL;
        e->tiled = e->variant == SNP_VARIANT_TILED || e->variant == SNP_VARIANT_TILED2;
        e->sys.tp = e->variant == SNP_VARIANT_TILED2 ? 1 : 0;
    } else {
        e->variant = SNP_VARIANT_PUSH;
        e->kind = RECV_ARRAY;
    }
    e->p_max = pmax;
    if (e->sys.tp && !pcommon) e->sys.tp = 0;  // two-pass receive moves P bits only
    if (pcommon) {
        e->p_mode = P_BIT;
        e->p_common = pfirst > 0 ? pfirst : 1;
    } else if (pmax <= 255 && !(sh && sh->x_pbits > 8)) {
        e->p_mode = P_U8;
    } else if (pmax <= 65535 && !(sh && sh->x_pbits > 16)) {
        e->p_mode = P_U16;
    } else {
        e->p_mode = P_U32;
    }
    if (sh) sh->hdr = 128 / (e->p_mode == P_BIT ? 1 : (e->p_mode == P_U8 ? 8 : (e->p_mode == P_U16 ? 16 : 32)));

    CU(cudaSetDevice(e->device));
    CU(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking));
    e->stream = e->own_stream;
    CU(cudaEventCreate(&e->ev0));
    CU(cudaEventCreate(&e->ev1));

    DevSys& s = e->sys;
    DevState& st = e->st;
    s.q = q;
    s.m = m;
    s.z = z;
    s.ell_rows = z + 1;
    s.p_common = e->p_common;
    uint32_t* d_roff;
    int4* d_rrec;
    uint32_t* d_outdeg;
    TRY(upload(e, &d_roff, roff));
    TRY(upload(e, &d_rrec, rrec));
    TRY(upload(e, &d_outdeg, outdeg));
    s.roff = d_roff;
    s.rrec = d_rrec;
    s.outdeg = d_outdeg;
    e->wide_rules = !compact;
    if (compact) {
        hvec<uint2> rw(m + 2);  // +2: 16-byte bulk-copy tails (written below)
        rw[m] = rw[m + 1] = make_uint2(0, 0);
        parallel_first_fail(m, [&](long long a, long long b) -> long long {
            for (long long r = a; r < b; ++r)
                rw[r] = make_uint2(rthr[r], (uint32_t)rrec[r].x | ((uint32_t)rrec[r].y << 16) | ((uint32_t)rrec[r].z << 24));
            return -1;
        });
        uint2* d_rw;
        TRY(upload(e, &d_rw, rw));
        s.rw = d_rw;
    } else {
        std::vector<uint4> rw(m + 1);
        for (long long r = 0; r < m; ++r)
            rw[r] = make_uint4(rthr[r], (uint32_t)rrec[r].x, (uint32_t)rrec[r].y, (uint32_t)rrec[r].z);
        uint4* d_rw;
        TRY(upload(e, &d_rw, rw));
        s.rw = d_rw;
    }
    // tiled: 4-byte rule words for the staged selection path when every rule
    // fits (threshold, consumed < 2^10, produced < 2^4, delay < 2^7)
    if (e->tiled && compact) {
        bool tiny = parallel_first_fail(m, [&](long long a, long long b) -> long long {
            for (long long r = a; r < b; ++r)
                if (!((rthr[r] & ~kExactBit) < 1024u && rrec[r].x < 1024 && rrec[r].y < 16 && rrec[r].z < 128)) return r;
            return -1;
        }) < 0;
        if (const char* env = getenv("SNPB200_TINY")) tiny = tiny && atoi(env) != 0;
        if (tiny) {
            hvec<uint32_t> rw4(m + 4);  // +4: 16-byte bulk-copy tails
            for (int x = 0; x < 4; ++x) rw4[m + x] = 0u;
            parallel_first_fail(m, [&](long long a, long long b) -> long long {
                for (long long r = a; r < b; ++r)
                    rw4[r] = tiny_word(rthr[r], (uint32_t)rrec[r].x, (uint32_t)rrec[r].y, (uint32_t)rrec[r].z);
                return -1;
            });
            uint32_t* d_rw4;
            TRY(upload(e, &d_rw4, rw4));
            s.rw4 = d_rw4;
            e->tiny_rules = true;
        }
    }

    tm.mark("rule words");
    uint32_t *d_soff = nullptr, *d_sdst = nullptr, *d_owner = nullptr;
    const bool need_owner = (e->format != SNP_FMT_COMPRESSED && have_adj);
    if (have_adj) {
        TRY(upload(e, &d_soff, soff));
        TRY(upload(e, &d_sdst, sdst));
    }
    if (need_owner) TRY(upload(e, &d_owner, owner));

    tm.mark("adjacency upload");
    // heavy list (CTA per neuron)
    std::vector<uint32_t> indeg;
    if (e->kind == RECV_PULL && !e->tiled && q > 0) {
        // in-adjacency = transpose of the out-adjacency, lists padded to x4
        // with the sentinel source q (whose P entry is always 0)
        uint32_t* d_indeg;
        TRY(e->alloc(&d_indeg, q));
        CU(cudaMemset(d_indeg, 0, q * sizeof(uint32_t)));
        if (!sdst.empty()) {
            indeg_kernel<<<std::min(grid_for((long long)sdst.size()), 148 * 64), 256>>>((long long)sdst.size(), d_sdst, d_indeg);
            CU(cudaGetLastError());
        }
        indeg.resize(q);
        CU(cudaMemcpy(indeg.data(), d_indeg, q * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        std::vector<uint32_t> ioff(q + 1, 0);
        unsigned long long acc = 0;
        for (long long i = 0; i < q; ++i) {
            ioff[i] = (uint32_t)acc;
            acc += (indeg[i] + 3u) & ~3u;
            if (acc >= (1ull << 32) - 4) return fail(SNP_ERR_CAPACITY, "in-adjacency exceeds uint32 offsets");
        }
        ioff[q] = (uint32_t)acc;
        e->in_edges = (long long)acc;
        uint32_t *d_ioff, *d_isrc, *d_cursor;
        TRY(upload(e, &d_ioff, ioff));
        TRY(e->alloc(&d_isrc, (long long)acc + 4));
        fill_u32_kernel<<<std::min(grid_for((long long)acc + 4), 148 * 64), 256>>>((long long)acc + 4, d_isrc, (uint32_t)q);
        CU(cudaGetLastError());
        TRY(e->alloc(&d_cursor, q));
        CU(cudaMemcpy(d_cursor, d_ioff, q * sizeof(uint32_t), cudaMemcpyDeviceToDevice));
        transpose_fill_kernel<<<grid_for(q), 256>>>(q, d_soff, d_sdst, d_cursor, d_isrc);
        CU(cudaGetLastError());
        CU(cudaDeviceSynchronize());
        s.ioff = d_ioff;
        s.isrc = d_isrc;
    }
    std::vector<uint32_t> heavy;
    for (long long i = 0; i < q; ++i) {
        const bool many_rules = roff[i + 1] - roff[i] > kLightRules;
        const bool many_in = e->kind == RECV_PULL && !e->tiled && ((indeg[i] + 3u) & ~3u) > kLightIn;
        if (many_rules || many_in) heavy.push_back((uint32_t)i);
    }
    if (sh && !e->tiled) return fail(SNP_ERR_BAD_ARG, "row partition needs COMPRESSED/tiled");
    tm.mark("in-adjacency / heavy");
    if (e->tiled) TRY(build_tiles(e, d, soff, sdst, roff, heavy, sh, d_soff, d_sdst));
    uint32_t* d_heavy;
    TRY(upload(e, &d_heavy, heavy));
    s.heavy = d_heavy;
    s.n_heavy = (int)heavy.size();
    // heavy-rule neurons: guard index for FirstApplicable (sorted exactly-
    // thresholds with their lowest rule, sorted at-least thresholds with the
    // prefix-minimum rule) -- a binary search instead of a scan over n rules
    if (!heavy.empty()) {
        std::vector<uint32_t> eoff(heavy.size() + 1, 0), aoff(heavy.size() + 1, 0);
        std::vector<uint2> ev, av;
        for (size_t h = 0; h < heavy.size(); ++h) {
            const uint32_t i = heavy[h], a = roff[i], b = roff[i + 1];
            std::vector<uint2> ex, al;
            for (uint32_t r = a; r < b; ++r)
                ((rthr[r] & kExactBit) ? ex : al).push_back(make_uint2(rthr[r] & ~kExactBit, r - a));
            auto by_t = [](const uint2& x, const uint2& y) { return x.x < y.x || (x.x == y.x && x.y < y.y); };
            std::sort(ex.begin(), ex.end(), by_t);
            std::sort(al.begin(), al.end(), by_t);
            for (size_t k = 0; k < ex.size(); ++k)
                if (k == 0 || ex[k].x != ex[k - 1].x) ev.push_back(ex[k]);  // lowest rule per threshold
            uint32_t pm = 0xffffffffu;
            for (const uint2& x : al) {
                pm = std::min(pm, x.y);
                av.push_back(make_uint2(x.x, pm));
            }
            eoff[h + 1] = (uint32_t)ev.size();
            aoff[h + 1] = (uint32_t)av.size();
        }
        // dense table over the count when a neuron's thresholds are compact
        // (max threshold <= 4 x its rules + 64): entry c = the FirstApplicable
        // rule for count c, the last entry for every count above the largest
        // threshold -- one dependent load instead of two 32-ary searches
        std::vector<uint32_t> loff(heavy.size() + 1, 0), lut;
        std::vector<uint16_t> lcnt;  // applicable rules per count (saturated): SeededRandom's table
        for (size_t h = 0; h < heavy.size(); ++h) {
            const uint32_t i = heavy[h], a = roff[i], b = roff[i + 1];
            uint32_t mt = 0;
            for (uint32_t r = a; r < b; ++r) mt = std::max(mt, rthr[r] & ~kExactBit);
            const unsigned long long need = (unsigned long long)mt + 2;
            if (mt > 4ull * (b - a) + 64 || lut.size() + need > (1ull << 28)) {
                loff[h + 1] = (uint32_t)lut.size();  // no table: the guard index
                continue;
            }
            std::vector<uint32_t> exf(mt + 2, 0xffffffffu), alf(mt + 2, 0xffffffffu), exn(mt + 2, 0), aln(mt + 2, 0);
            for (uint32_t r = a; r < b; ++r) {
                const uint32_t t = rthr[r] & ~kExactBit;
                const bool ex = (rthr[r] & kExactBit) != 0;
                uint32_t& slot = ex ? exf[t] : alf[t];
                slot = std::min(slot, r - a);
                (ex ? exn[t] : aln[t]) += 1;
            }
            uint32_t best_al = 0xffffffffu, n_al = 0;
            for (uint32_t c = 0; c <= mt; ++c) {
                best_al = std::min(best_al, alf[c]);
                n_al += aln[c];
                lut.push_back(std::min(best_al, exf[c]));
                lcnt.push_back(std::min<uint32_t>(n_al + exn[c], 0xffffu));
            }
            lut.push_back(best_al);  // counts above every threshold: at-least rules only
            lcnt.push_back(std::min<uint32_t>(n_al, 0xffffu));
            loff[h + 1] = (uint32_t)lut.size();
        }
        if (!lut.empty()) {
            uint32_t *d_loff, *d_lut;
            uint16_t* d_lcnt;
            TRY(upload(e, &d_loff, loff));
            TRY(upload(e, &d_lut, lut));
            TRY(upload(e, &d_lcnt, lcnt));
            s.hx_loff = d_loff;
            s.hx_lut = d_lut;
            s.hx_lcnt = d_lcnt;
        }
        uint32_t *d_eoff, *d_aoff;
        uint2 *d_ev, *d_av;
        TRY(upload(e, &d_eoff, eoff));
        TRY(upload(e, &d_aoff, aoff));
        TRY(upload(e, &d_ev, ev));
        TRY(upload(e, &d_av, av));
        s.hx_eoff = d_eoff;
        s.hx_aoff = d_aoff;
        s.hx_e = d_ev;
        s.hx_a = d_av;
    }
    // at least one (possibly all-idle) light tile so that q == 0 still runs
    // the halting decision on the device
    s.light_tiles = std::max<long long>(1, ceil_div(q, kBlock));

    if (e->format == SNP_FMT_COMPRESSED && e->kind == RECV_ARRAY) {
        s.soff = d_soff;
        s.sdst = d_sdst;
    }
    if (e->format == SNP_FMT_ELL) {
        uint32_t* d_len;
        int2* d_ell;
        if (ell_from_matrix) {
            TRY(upload(e, &d_ell, ell_host));
            TRY(upload(e, &d_len, ell_len_host));
        } else {
            ell_ld = std::max<long long>(2, (z + 2) & ~1ll);
            TRY(e->alloc(&d_ell, m * ell_ld));
            TRY(e->alloc(&d_len, m));
            CU(cudaMemset(d_ell, 0xff, (size_t)std::max<long long>(1, m * ell_ld) * sizeof(int2)));
            if (m > 0) build_ell_kernel<<<grid_for(m), 256>>>(m, ell_ld, d_owner, d_rrec, d_soff, d_sdst, d_ell, d_len);
            CU(cudaGetLastError());
        }
        s.ell = d_ell;
        s.ell_len = d_len;
        s.ell_ld = ell_ld;
    }
    if (e->format == SNP_FMT_SPARSE) {
        const long long ld = std::max<long long>(4, (q + 3) & ~3ll);
        int* d_dense;
        if ((double)m * (double)ld * 4.0 > 9.0e18) return fail(SNP_ERR_CAPACITY, "dense matrix too large");
        TRY(e->alloc(&d_dense, m * ld));
        CU(cudaMemset(d_dense, 0, (size_t)std::max<long long>(1, m * ld) * sizeof(int)));
        if (dense_from_matrix) {
            std::vector<int> row(ld, 0);
            for (long long r = 0; r < m; ++r) {
                for (long long i = 0; i < q; ++i) {
                    const long long v = d->sparse_data[r * q + i];
                    if (v < -kInt32Max || v > kInt32Max) return fail(SNP_ERR_CAPACITY, "dense entry outside int32");
                    row[i] = (int)v;
                }
                CU(cudaMemcpy(d_dense + r * ld, row.data(), ld * sizeof(int), cudaMemcpyHostToDevice));
            }
        } else if (m > 0) {
            build_dense_kernel<<<grid_for(m), 256>>>(m, ld, d_owner, d_rrec, d_soff, d_sdst, d_dense);
            CU(cudaGetLastError());
        }
        s.dense = d_dense;
        s.dense_ld = ld;
        const int col_tiles = (int)std::max<long long>(1, ceil_div(q, kBlock * 4));
        const int splits = std::max(1, std::min(1024, 148 * 8 / col_tiles));
        e->dense_grid = dim3(col_tiles, splits, 1);
    }

    tm.mark("tiled layout + formats");
    // --- one-kernel push step for runs (ELL / COMPRESSED-push, every neuron
    // <= 32 rules): the binned kernel (ell_bin_step_kernel) when deliveries
    // fit its entries, else the L2-atomic one (push_step_kernel).
    // SNPB200_PUSH=atomic forces the latter, =unfused the 3-kernel path.
    const char* push_env = getenv("SNPB200_PUSH");
    if (e->kind == RECV_ARRAY && e->format != SNP_FMT_SPARSE && s.n_heavy == 0 && q > 0 &&
        e->variant != SNP_VARIANT_SMALL &&
        !(push_env && !strcmp(push_env, "unfused"))) {
        // per destination: deliveries it can receive in one step (each source
        // fires at most one rule) and their largest amount
        std::vector<uint32_t> ind(q, 0);
        long long amax = 0, amin = 0, cmax = 0;
        bool amount_common = true;
        if (have_adj) {
            if (!sdst.empty()) {
                uint32_t* d_in;
                CU(cudaMalloc(&d_in, (size_t)q * 4));
                CU(cudaMemset(d_in, 0, (size_t)q * 4));
                indeg_kernel<<<std::min(grid_for((long long)sdst.size()), 148 * 64), 256>>>((long long)sdst.size(), d_sdst, d_in);
                cudaError_t err = cudaGetLastError();
                if (err == cudaSuccess) err = cudaMemcpy(ind.data(), d_in, (size_t)q * 4, cudaMemcpyDeviceToHost);
                cudaFree(d_in);
                CU(err);
            }
            amax = pmax;
            amin = pfirst;
            amount_common = pcommon;
            if (e->format == SNP_FMT_ELL)
                for (long long r = 0; r < m; ++r) cmax = std::max<long long>(cmax, rrec[r].x);
        } else {
            // ELL given as the reference matrix: count every delivery pair (an
            // upper bound: rules of one neuron never fire together)
            for (long long r = 0; r < m; ++r)
                for (uint32_t n = 1; n < ell_len_host[r]; ++n) {
                    const int2 pr = ell_host[r * ell_ld + n];
                    ind[pr.x] += 1;
                    const long long a = std::abs((long long)pr.y);
                    if (amin == 0) amin = a;
                    amount_common = amount_common && a == amin && pr.y > 0;
                    amax = std::max(amax, a);
                }
            for (long long r = 0; r < m; ++r)
                if (ell_len_host[r]) cmax = std::max<long long>(cmax, std::abs((long long)ell_host[r * ell_ld].y));
        }
        uint32_t mx = 0;
        for (uint32_t x : ind) mx = std::max(mx, x);
        // binned: u16 slots (common amount) or u32 slot << 15 | amount (< 2^15)
        const bool unit = amount_common && amin > 0;
        bool bins_ok = (unit || (amin >= 0 && amax < (1 << 15))) && !(push_env && !strcmp(push_env, "atomic"));
        if (ell_from_matrix)  // the binned kernel consumes at selection: row 0 must be (owner, -consumed)
            for (long long r = 0; r < m && bins_ok; ++r)
                bins_ok = ell_len_host[r] >= 1 && ell_host[r * ell_ld].x == (int)owner[r] &&
                          ell_host[r * ell_ld].y == -rrec[r].x;
        const long long recv_worst = (long long)mx * (unit ? 1 : std::max<long long>(1, amax));
        int n_sm = 148;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, e->device);
        int smem_optin = 0;
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device);
        bool binned = false;
        if (bins_ok && recv_worst < (1ll << 32)) {
            const int cb = recv_worst < 256 ? 8 : (recv_worst < 65536 ? 16 : 32);
            const long long tmax = unit ? 65504 : 131072;  // u16 entries: the pad slot T must fit
            long long per_sm = 2;
            if (const char* env = getenv("SNPB200_BIN_TILES_PER_SM")) per_sm = std::max(1, atoi(env));
            long long T = std::min<long long>(tmax, (ceil_div(q, per_sm * n_sm) + 31) / 32 * 32);
            const long long nt = ceil_div(q, T);
            const size_t esz = unit ? 2 : 4;
            const size_t acc_b = 4 * (size_t)(cb == 8 ? bin_acc_words<8>((int)T)
                                                      : (cb == 16 ? bin_acc_words<16>((int)T) : bin_acc_words<32>((int)T)));
            const int bcap = unit ? BinEntry<true>::kCap : BinEntry<false>::kCap;
            const size_t smem = acc_b + 4 * (size_t)((nt + 3) & ~3ll) + (size_t)nt * bcap * esz;
            if ((long long)smem + 2048 <= smem_optin) {
                binned = true;
                // bin regions per tile: main = its destinations' in-degree sum
                // plus the 16-byte padding of every flush that can reach it in
                // one step; overflow = the in-degree sum (full buckets)
                const unsigned long long pads =
                    8ull * (unsigned long long)(ceil_div(q, bin_flush_dests(unit)) + nt);
                std::vector<unsigned long long> deg(nt, 0);
                for (long long t = 0; t < nt; ++t)
                    for (long long jj = t * T; jj < std::min<long long>(q, (t + 1) * T); ++jj) deg[t] += ind[jj];
                std::vector<uint32_t> boff(nt + 1, 0), ooff(nt + 1, 0);
                unsigned long long tot = 0;
                for (long long t = 0; t < nt; ++t) {
                    boff[t] = (uint32_t)tot;
                    tot += ((deg[t] + 7) & ~7ull) + pads;
                    if (tot >= (1ull << 32) - 8) return fail(SNP_ERR_CAPACITY, "push bins exceed 2^32 entries");
                }
                boff[nt] = (uint32_t)tot;
                for (long long t = 0; t < nt; ++t) {
                    ooff[t] = (uint32_t)tot;
                    tot += deg[t];
                    if (tot >= (1ull << 32) - 8) return fail(SNP_ERR_CAPACITY, "push bins exceed 2^32 entries");
                }
                ooff[nt] = (uint32_t)tot;
                uint32_t *d_boff, *d_ooff;
                TRY(upload(e, &d_boff, boff));
                TRY(upload(e, &d_ooff, ooff));
                s.bin_ooff = d_ooff;
                for (int i = 0; i < 2; ++i) {
                    uint4* bb;
                    TRY(e->alloc(&bb, (long long)(tot * esz + 15) / 16 + 1));
                    st.bins[i] = bb;
                    TRY(e->alloc(&st.bin_fill[i], 2 * nt));
                }
                s.bin_T = (int)T;
                s.bin_ntiles = (int)nt;
                s.bin_magic = (~0ull / (unsigned long long)T) + 1ull;
                s.bin_amount = unit ? (int)amin : 1;
                s.bin_off = d_boff;
                s.bin_cpc = (e->format == SNP_FMT_ELL && ell_ld / 2 <= 16) ? (int)(ell_ld / 2) : 0;
                e->bin_cb = cb;
                e->bin_unit = unit;
                e->bin_smem = smem;
                const bool ell = e->format == SNP_FMT_ELL, w = e->wide_rules;
                const bool grp = s.bin_cpc > 0;
#define SNP_BIN_PICK(E_, W_, U_, G_)                                                                      \
    (cb == 8 ? ell_bin_step_kernel<E_, W_, U_, 8, G_> : (cb == 16 ? ell_bin_step_kernel<E_, W_, U_, 16, G_>  \
                                                                  : ell_bin_step_kernel<E_, W_, U_, 32, G_>))
#define SNP_BIN_PICK_G(W_, U_) (grp ? SNP_BIN_PICK(true, W_, U_, true) : SNP_BIN_PICK(true, W_, U_, false))
                if (ell) e->fused_fn = w ? (unit ? SNP_BIN_PICK_G(true, true) : SNP_BIN_PICK_G(true, false))
                                         : (unit ? SNP_BIN_PICK_G(false, true) : SNP_BIN_PICK_G(false, false));
                else e->fused_fn = w ? (unit ? SNP_BIN_PICK(false, true, true, false) : SNP_BIN_PICK(false, true, false, false))
                                     : (unit ? SNP_BIN_PICK(false, false, true, false) : SNP_BIN_PICK(false, false, false, false));
#undef SNP_BIN_PICK_G
#undef SNP_BIN_PICK
                TRY(allow_max_smem((const void*)e->fused_fn, e->device, smem));
            }
        }
        if (!binned) {
            // L2 atomics into int32 receive buffers unless some neuron could
            // receive 2^31 or more (in absolute value) in one step
            const long long worst = (long long)mx * std::max<long long>(1, amax) + cmax;
            e->recv64 = worst >= (1ll << 31);
            const bool ell = e->format == SNP_FMT_ELL, w = e->wide_rules, r64 = e->recv64;
            e->fused_fn = ell ? (w ? (r64 ? push_step_kernel<true, true, true> : push_step_kernel<true, true, false>)
                                   : (r64 ? push_step_kernel<true, false, true> : push_step_kernel<true, false, false>))
                              : (w ? (r64 ? push_step_kernel<false, true, true> : push_step_kernel<false, true, false>)
                                   : (r64 ? push_step_kernel<false, false, true> : push_step_kernel<false, false, false>));
            for (int i = 0; i < 2; ++i) {
                long long* bb;
                TRY(e->alloc(&bb, r64 ? q : (q + 1) / 2));
                st.rbuf[i] = bb;
            }
        }
    }

    // --- run state
    TRY(e->alloc(&st.cfg, q + 8));  // +8: 16-byte bulk-copy tails
    TRY(e->alloc(&st.ds, q + 8));
    TRY(e->alloc(&st.chosen, q));
    if (sh) {
        s.x_stride = sh->nl * 128 / sh->hdr / 32 + 4;  // P elements, then 4 header words
        s.world = sh->world;
        s.rank = sh->rank;
        s.gbase = sh->lo;
        s.xbase = (long long)sh->rank * (sh->nl + sh->hdr);  // in P elements
        // identical on every rank (peers address each other's flags at
        // 3 * p_words): the two-pass tail covers any window size <= 2^16
        e->p_words = s.x_stride * sh->world + 8 + (s.tp ? (1ll << (16 - 5)) : 0);
    }
    if (e->kind == RECV_PULL) {
        long long words;
        switch (sh ? -1 : e->p_mode) {
            case -1: words = e->p_words; break;  // row partition: the exchange space
            case P_BIT:  // +8: bulk-copy tails; two-pass: whole source windows
                words = std::max<long long>(ceil_div(q + 1, 32) + 8, s.tp ? s.tp_nw * (1ll << (s.tp_wlog - 5)) + 8 : 0);
                break;
            case P_U8: words = ceil_div(q + 1, 4) + 1; break;
            case P_U16: words = ceil_div(q + 1, 2) + 1; break;
            default: words = q + 2; break;
        }
        if (e->p_mode == P_BIT && !sh) e->p_bit_words = words;
        if (sh) {
            // one exchange block: 3 slots, then `world` 64-bit step flags (peer
            // exchange); a single allocation so it maps with one IPC handle
            uint32_t* blk;
            TRY(e->alloc(&blk, 3 * words + 2ll * sh->world + 2));
            CU(cudaMemset(blk + 3 * words, 0, (2ll * sh->world + 2) * 4));
            for (int i = 0; i < 3; ++i) st.P[i] = blk + i * words;
            e->xblock = blk;
            s.p_words = words;
        } else {
            for (int i = 0; i < 3; ++i) TRY(e->alloc(&st.P[i], words));
        }
    } else {
        TRY(e->alloc(&st.recv, q));
        TRY(e->alloc(&st.list[0], q));
        TRY(e->alloc(&st.list[1], q));
    }
    TRY(e->alloc(&st.ctrl, 1));
    e->push_grid = grid_for(q);
    e->heavy_push_grid = 148 * 4;

    tm.mark("run state");
    // kernel instances
    if (e->tiled) {
        switch (e->p_mode) {
            case P_BIT: pick_tiled<P_BIT>(e); break;
            case P_U8: pick_tiled<P_U8>(e); break;
            case P_U16: pick_tiled<P_U16>(e); break;
            default: pick_tiled<P_U32>(e); break;
        }
    } else if (e->format == SNP_FMT_COMPRESSED && e->kind == RECV_PULL) {
        switch (e->p_mode) {
            case P_BIT: pick_fns<RECV_PULL, P_BIT, true, false>(e->wide_rules, &e->step_fn, &e->prime_fn); break;
            case P_U8: pick_fns<RECV_PULL, P_U8, true, false>(e->wide_rules, &e->step_fn, &e->prime_fn); break;
            case P_U16: pick_fns<RECV_PULL, P_U16, true, false>(e->wide_rules, &e->step_fn, &e->prime_fn); break;
            default: pick_fns<RECV_PULL, P_U32, true, false>(e->wide_rules, &e->step_fn, &e->prime_fn); break;
        }
    } else if (e->format == SNP_FMT_COMPRESSED) {
        pick_fns<RECV_ARRAY, P_BIT, true, false>(e->wide_rules, &e->step_fn, &e->prime_fn);
        if (e->variant == SNP_VARIANT_SMALL) {
            // 32-bit receive counters unless a destination can get 2^31 in a step
            std::vector<uint32_t> ind(std::max<long long>(1, q), 0);
            uint32_t mx = 0;
            for (uint32_t t : sdst) mx = std::max(mx, ++ind[t]);
            const bool r64 = (double)mx * (double)std::max<long long>(1, pmax) >= 2147483648.0;
            const bool sm = q <= kSmallSmemQ;  // the state in shared memory too
#define SNP_SMALL_PICK(W_) (r64 ? (sm ? small_run_kernel<W_, true, true> : small_run_kernel<W_, true, false>) \
                                : (sm ? small_run_kernel<W_, false, true> : small_run_kernel<W_, false, false>))
            e->small_fn = e->wide_rules ? SNP_SMALL_PICK(true) : SNP_SMALL_PICK(false);
#undef SNP_SMALL_PICK
            const size_t rb = (((size_t)std::max<long long>(1, q) * (r64 ? 8 : 4)) + 15) & ~(size_t)15;
            e->small_smem = rb + (sm ? (size_t)std::max<long long>(1, q) * 16 : 0);
            TRY(allow_max_smem((const void*)e->small_fn, e->device, e->small_smem));
        }
    } else if (e->format == SNP_FMT_ELL) {
        pick_fns<RECV_ARRAY, P_BIT, false, false>(e->wide_rules, &e->step_fn, &e->prime_fn);
    } else {
        pick_fns<RECV_ARRAY, P_BIT, false, true>(e->wide_rules, &e->step_fn, &e->prime_fn);
    }
    // persistent-style grid: as many CTAs as are resident at once
    int per_sm = 0, n_sm = 0;
    CU(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, e->device));
    if (e->tiled) {
        e->step_block = kTileThreads + 32;  // consumer warps + one TMA producer warp
        e->step_smem = (size_t)s.ring * kStageBytes +
                       (size_t)(e->cbits == 8 ? acc_words<8>(s.tile)
                                                 : (e->cbits == 16 ? acc_words<16>(s.tile) : acc_words<32>(s.tile))) *
                           sizeof(uint32_t);
        TRY(allow_max_smem((const void*)e->step_fn, e->device, e->step_smem));
        TRY(allow_max_smem((const void*)e->lean_fn, e->device, e->step_smem));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e->step_fn, e->step_block, e->step_smem));
        const long long resident = (long long)std::max(1, per_sm) * std::max(1, n_sm);
        e->step_grid = (int)std::min<long long>(s.n_tiles, resident);
        e->resident_ctas = resident;
    } else {
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e->step_fn, kBlock, 0));
        const long long resident = (long long)std::max(1, per_sm) * std::max(1, n_sm);
        s.light_ctas = (int)std::min<long long>(s.light_tiles, resident);
        s.heavy_ctas = (int)std::min<long long>(s.n_heavy, resident);
        e->step_grid = s.light_ctas + s.heavy_ctas;
        e->resident_ctas = resident;
    }
    if (e->fused_fn && e->bin_cb) {
        int per = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, e->fused_fn, kBinThreads, e->bin_smem));
        e->fused_grid = (int)std::min<long long>(s.bin_ntiles, (long long)std::max(1, per) * n_sm);
        e->fused_block = kBinThreads;
        e->fused_smem = e->bin_smem;
    } else if (e->fused_fn) {
        int per = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, e->fused_fn, kBlock, 0));
        e->fused_grid = (int)std::min<long long>(s.light_tiles, (long long)std::max(1, per) * n_sm);
        e->fused_block = kBlock;
        e->fused_smem = 0;
    }
    CU(cudaDeviceSynchronize());
    return SNP_OK;
}

// Launch one step's kernels on the engine stream; returns launch count.
// Two-pass receive: pass 1 (edge bits per source window) before the step kernel.
int launch_pass1(snp_engine* e) {
    if (!e->sys.tp) return 0;
    pass1_kernel<<<e->p1_grid, 512, 0, e->stream>>>(e->sys, e->st);
    return 1;
}

// The scatter kernels that follow an unfused push-format step kernel.
int launch_push_tail(snp_engine* e, long long* row_visits = nullptr) {
    if (e->kind != RECV_ARRAY || e->fused_fn) return 0;
    if (e->format == SNP_FMT_SPARSE) {
        dense_kernel<<<e->dense_grid, kBlock, 0, e->stream>>>(e->sys, e->st);
        return 1;
    }
    if (e->format == SNP_FMT_ELL) {
        push_kernel<true><<<e->push_grid, kBlock, 0, e->stream>>>(e->sys, e->st, row_visits);
        push_heavy_kernel<true><<<e->heavy_push_grid, kBlock, 0, e->stream>>>(e->sys, e->st);
    } else {
        push_kernel<false><<<e->push_grid, kBlock, 0, e->stream>>>(e->sys, e->st, row_visits);
        push_heavy_kernel<false><<<e->heavy_push_grid, kBlock, 0, e->stream>>>(e->sys, e->st);
    }
    return 2;
}

int launch_step(snp_engine* e, long long* row_visits = nullptr) {
    if (e->small_fn) {  // one launch runs the rest of the segment (up to Ctrl.stop_at)
        launch_main(e);
        return 1;
    }
    int n = 1 + launch_pass1(e);
    launch_main(e);
    return n + launch_push_tail(e, row_visits);
}

int push_ctrl(snp_engine* e) {
    CU(cudaMemcpyAsync(e->st.ctrl, &e->hctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    return SNP_OK;
}

int pull_ctrl(snp_engine* e) {
    CU(cudaMemcpyAsync(&e->hctrl, e->st.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    if (e->hctrl.fault)
        return fail(SNP_ERR_CUDA, "internal error: a binned-push bin region overflowed at step %lld", e->hctrl.step);
    return SNP_OK;
}

int reset_state(snp_engine* e) {
    const long long q = e->q;
    DevState& st = e->st;
    if (e->kind == RECV_PULL) {
        // all three P vectors start empty: P_{-1} = 0 and the bit words are
        // OR-accumulated into zeroed buffers
        for (int i = 0; i < 3; ++i) {
            size_t bytes;
            switch (e->p_words ? -1 : e->p_mode) {
                case -1: bytes = e->p_words * 4; break;  // row partition: the exchange space
                case P_BIT: bytes = e->p_bit_words * 4; break;
                case P_U8: bytes = (ceil_div(q + 1, 4) + 1) * 4; break;
                case P_U16: bytes = (ceil_div(q + 1, 2) + 1) * 4; break;
                default: bytes = (q + 2) * 4; break;
            }
            CU(cudaMemsetAsync(st.P[i], 0, bytes, e->stream));
        }
    } else {
        CU(cudaMemsetAsync(st.recv, 0, std::max<long long>(1, q) * 8, e->stream));
        if (e->fused_fn && e->bin_cb) {
            for (int i = 0; i < 2; ++i)
                CU(cudaMemsetAsync(st.bin_fill[i], 0, (size_t)std::max(1, e->sys.bin_ntiles) * 8, e->stream));
        } else if (e->fused_fn) {
            for (int i = 0; i < 2; ++i)
                CU(cudaMemsetAsync(st.rbuf[i], 0, std::max<long long>(1, q) * (e->recv64 ? 8 : 4), e->stream));
        }
    }
    CU(cudaMemsetAsync(st.ds, 0, std::max<long long>(1, q) * 4, e->stream));
    CU(cudaMemsetAsync(st.chosen, 0xff, std::max<long long>(1, q) * 4, e->stream));
    memset(&e->hctrl, 0, sizeof(Ctrl));
    e->hctrl.neg_index = 0x7fffffffffffffffll;
    e->hctrl.max_steps = 1;
    return SNP_OK;
}

int ensure_trace(snp_engine* e, long long rows) {
    if (e->tr_rows >= rows) return SNP_OK;
    // (re)allocate the ring; the graph captures its pointers
    long long* cfg;
    int *dly, *ch;
    TRY(e->alloc(&cfg, rows * std::max<long long>(1, e->q)));
    TRY(e->alloc(&dly, rows * std::max<long long>(1, e->q)));
    TRY(e->alloc(&ch, rows * std::max<long long>(1, e->q)));
    e->st.tr_cfg = cfg;
    e->st.tr_dly = dly;
    e->st.tr_chosen = ch;
    e->st.tr_rows = rows;
    e->tr_rows = rows;
    if (e->graph) {
        cudaGraphExecDestroy(e->graph);
        e->graph = nullptr;
    }
    return SNP_OK;
}

int ensure_graph(snp_engine* e, long long iters) {
    if (e->graph && e->graph_iters == iters && e->graph_fn == run_fn(e)) return SNP_OK;
    if (e->graph) {
        cudaGraphExecDestroy(e->graph);
        e->graph = nullptr;
    }
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    for (long long i = 0; i < iters; ++i) launch_step(e);
    CU(cudaStreamEndCapture(e->stream, &g));
    cudaError_t err = cudaGraphInstantiate(&e->graph, g, 0);
    cudaGraphDestroy(g);
    CU(err);
    e->graph_iters = iters;
    e->graph_fn = run_fn(e);
    return SNP_OK;
}

int kernels_per_step(const snp_engine* e) {
    if (e->kind == RECV_PULL) return e->sys.tp ? 2 : 1;
    if (e->fused_fn) return 1;
    return e->format == SNP_FMT_SPARSE ? 2 : 3;
}

int validate_opts(const snp_run_opts* o) {
    if (!o) return fail(SNP_ERR_BAD_ARG, "options missing");
    if (o->max_steps < 1) return fail(SNP_ERR_BAD_ARG, "max_steps must be >= 1, got %lld", (long long)o->max_steps);
    if (o->policy != SNP_POLICY_FIRST && o->policy != SNP_POLICY_SEEDED)
        return fail(SNP_ERR_BAD_ARG, "unknown policy %d", o->policy);
    if (o->record & ~15) return fail(SNP_ERR_BAD_ARG, "bad record flags %d", o->record);
    return SNP_OK;
}

void fill_result(const snp_engine* e, snp_result* res) {
    if (!res) return;
    const Ctrl& c = e->hctrl;
    res->steps = c.step;
    res->halt = c.halted ? c.reason : SNP_RUNNING;
    res->error = (c.halted && c.reason == HALT_NEGATIVE) ? SNP_ERR_NEGATIVE : SNP_OK;
    res->negative_neuron = c.neg_any ? c.neg_index : -1;
    res->negative_value = c.neg_any ? c.neg_value : 0;
    for (int i = 0; i < SNP_STAT_COUNT; ++i) res->stats[i] = c.stats[i];
}

}  // namespace

// ============================================================================ C ABI

extern "C" {

int snp_abi_version(void) { return SNPB200_ABI_VERSION; }

const char* snp_last_error(void) { return g_last_error.c_str(); }

int snp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int snp_engine_create(const snp_system_desc* desc, snp_engine** out) {
    if (!desc || !out) return fail(SNP_ERR_BAD_ARG, "null argument");
    if (desc->format < SNP_FMT_SPARSE || desc->format > SNP_FMT_COMPRESSED)
        return fail(SNP_ERR_BAD_ARG, "unknown format %d", desc->format);
    if (snp_device_count() <= desc->device)
        return fail(SNP_ERR_CUDA, "no CUDA device %d visible (the B200 engine has no CPU fallback)", desc->device);
    auto e = std::make_unique<snp_engine>();
    e->device = desc->device;
    int rc;
    if (desc->world > 1) {
        // row partition: build the local slice of the global system
        const long long q = desc->q;
        if (desc->rank < 0 || desc->rank >= desc->world) return fail(SNP_ERR_BAD_ARG, "rank out of range");
        if (desc->format != SNP_FMT_COMPRESSED || !desc->adj_offsets)
            return fail(SNP_ERR_BAD_ARG, "row partition needs COMPRESSED with adj_offsets/adj_targets");
        ShardInput sh;
        sh.world = desc->world;
        sh.rank = desc->rank;
        sh.q_global = q;
        sh.nl = (ceil_div(std::max<long long>(q, 1), desc->world) + 127) / 128 * 128;
        sh.lo = std::min<long long>(q, (long long)desc->rank * sh.nl);
        sh.hi = std::min<long long>(q, sh.lo + sh.nl);
        if (sh.hi <= sh.lo)
            return fail(SNP_ERR_BAD_ARG, "row partition: rank %d of %d owns no neurons (q=%lld; rows are cut in "
                        "multiples of 128): use fewer ranks", (int)desc->rank, (int)desc->world, q);
        TRY(check_csr_offsets(desc->adj_offsets, q));
        const long long S = q > 0 ? desc->adj_offsets[q] : 0;
        sh.x_pbits = desc->x_pbits;
        sh.x_pmax = desc->x_pmax;
        if (S >= (1ll << 32) - 1 || (long long)desc->world * (sh.nl + 128) >= (1ll << 32))
            return fail(SNP_ERR_CAPACITY, "row partition exceeds 32-bit exchange positions");
        sh.soff.resize(q + 1);
        sh.sdst.resize(S);
        parallel_first_fail(q + 1, [&](long long a, long long b) -> long long {
            for (long long i = a; i < b; ++i) sh.soff[i] = (uint32_t)desc->adj_offsets[i];
            return -1;
        });
        const long long bad = parallel_first_fail(S, [&](long long a, long long b) -> long long {
            for (long long x = a; x < b; ++x) {
                const long long t = desc->adj_targets[x];
                if (t < 0 || t >= q) return x;
                sh.sdst[x] = (uint32_t)t;
            }
            return -1;
        });
        if (bad >= 0) return fail(SNP_ERR_BAD_ARG, "synapse target %lld out of range", (long long)desc->adj_targets[bad]);
        // node arrays (initial, offsets, rules) describe this rank's neurons
        // [lo, hi) only; `m` counts their rules
        snp_system_desc ld = *desc;
        ld.q = sh.hi - sh.lo;
        ld.adj_offsets = nullptr;
        ld.adj_targets = nullptr;
        ld.syn_target = nullptr;
        ld.variant = desc->variant == SNP_VARIANT_TILED2 ? SNP_VARIANT_TILED2 : SNP_VARIANT_TILED;
        e->shard_lo = sh.lo;
        e->shard_hi = sh.hi;
        e->shard_nl = sh.nl;
        rc = build(e.get(), &ld, &sh);
    } else {
        rc = build(e.get(), desc);
    }
    if (rc != SNP_OK) return rc;
    *out = e.release();
    return SNP_OK;
}

void snp_engine_destroy(snp_engine* eng) {
    if (!eng) return;
    cudaSetDevice(eng->device);
    delete eng;
}

int snp_engine_get_info(const snp_engine* e, snp_engine_info* info) {
    if (!e || !info) return fail(SNP_ERR_BAD_ARG, "null argument");
    info->q = e->q;
    info->m = e->m;
    info->z = e->z;
    info->device_bytes = e->device_bytes;
    info->format = e->format;
    info->variant = e->variant;
    info->p_mode = e->p_mode;
    info->heavy_neurons = e->sys.n_heavy;
    info->in_edges = e->in_edges;
    info->p_common = e->p_common;
    info->tile = e->sys.tile;
    info->n_tiles = e->sys.n_tiles;
    info->ring_stages = e->tiled ? e->sys.ring : 0;
    info->counter_bits = e->tiled ? e->cbits : 0;
    info->stage_bytes = e->tiled ? (int64_t)kStageBytes : 0;
    info->push_kernel = e->kind != RECV_ARRAY || e->format == SNP_FMT_SPARSE
                            ? SNP_PUSH_NONE
                            : (!e->fused_fn ? SNP_PUSH_UNFUSED : (e->bin_cb ? SNP_PUSH_BINNED : SNP_PUSH_ATOMIC));
    info->push_tiles = e->bin_cb ? e->sys.bin_ntiles : 0;
    return SNP_OK;
}

int snp_begin(snp_engine* e, const int64_t* initial) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    CU(cudaSetDevice(e->device));
    TRY(reset_state(e));
    e->hctrl.epoch = ++e->epoch;
    const long long q = e->q;
    const long long* src = initial ? reinterpret_cast<const long long*>(initial) : e->initial.data();
    // cudaMemcpyDefault (unified addressing): `initial` may be host memory
    // or a device pointer (e.g. a torch CUDA tensor), copied on the engine's stream
    if (q > 0) CU(cudaMemcpyAsync(e->st.cfg, src, q * 8, cudaMemcpyDefault, e->stream));
    TRY(push_ctrl(e));
    CU(cudaStreamSynchronize(e->stream));
    e->begun = true;
    return SNP_OK;
}

int snp_advance(snp_engine* e, const snp_run_opts* o, int64_t n_steps, snp_trace_out* tr, snp_result* res) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    TRY(validate_opts(o));
    if (!e->begun) return fail(SNP_ERR_BAD_ARG, "snp_advance before snp_begin");
    if (e->sys.x_stride) return fail(SNP_ERR_BAD_ARG, "a row-partitioned engine steps with snp_launch_step + an exchange");
    CU(cudaSetDevice(e->device));
    const long long q = e->q;
    const int record = tr ? o->record : 0;
    long long chunk = o->chunk > 0 ? o->chunk : (q >= (1ll << 20) ? 16 : (q >= (1ll << 14) ? 64 : 256));
    if (record) {
        long long budget_rows = std::max<long long>(1, (1ll << 30) / std::max<long long>(1, q * 16));
        chunk = std::min(chunk, budget_rows);
        if (tr->cap < 1) return fail(SNP_ERR_BAD_ARG, "trace capacity must be >= 1");
        chunk = std::min<long long>(chunk, tr->cap);
        TRY(ensure_trace(e, chunk));
    }
    if (tr) {
        tr->first_row_step = e->hctrl.step;
        tr->config_rows = 0;
        tr->spiking_rows = 0;
    }
    Ctrl& c = e->hctrl;
    c.max_steps = o->max_steps;
    c.policy = o->policy;
    c.seed = o->seed;
    c.record = record;
    c.stats_on = o->collect_stats ? 1 : 0;
    long long budget = (long long)n_steps;
    long long launches = 0;
    std::vector<int> tmp;
    CU(cudaEventRecord(e->ev0, e->stream));
    while (budget > 0 && !c.halted) {
        long long seg = std::min(chunk, budget);
        if (record) seg = std::min<long long>(seg, (long long)(tr->cap - tr->config_rows));
        if (seg <= 0) break;
        const long long k0 = c.step;
        c.stop_at = k0 + seg;
        c.trace_base = k0;
        nvtxRangePushA("snp_segment");
        struct Pop {
            ~Pop() { nvtxRangePop(); }
        } pop_on_exit;
        TRY(push_ctrl(e));
        if (e->small_fn) {
            launch_main(e);
            launches += 1;
        } else if (o->use_graph) {
            TRY(ensure_graph(e, chunk));
            CU(cudaGraphLaunch(e->graph, e->stream));
            launches += chunk * kernels_per_step(e);
        } else {
            for (long long i = 0; i < seg; ++i) launches += launch_step(e);
            CU(cudaGetLastError());
        }
        CU(cudaGetLastError());
        TRY(pull_ctrl(e));
        const long long k1 = c.step;  // halt step or next step
        if (k1 == k0 && !c.halted) return fail(SNP_ERR_CUDA, "device loop made no progress at step %lld", k0);
        long long cfg_rows = c.halted ? (k1 - k0 + 1) : (k1 - k0);
        long long sp_rows = k1 - k0;
        if (c.halted && c.reason == HALT_NEGATIVE) break;
        if (record && (record & SNP_REC_DIGEST)) {
            // digests only: one reduction per recorded row, 8 bytes back per row
            if (e->digest_cap < chunk) {
                TRY(e->alloc(&e->d_digest, 3 * chunk));
                e->digest_cap = chunk;
            }
            CU(cudaMemsetAsync(e->d_digest, 0, 3 * chunk * 8, e->stream));
            const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>(ceil_div(q, 256), 148));
            const long long r0 = tr->config_rows, s0 = tr->spiking_rows;
            if (cfg_rows > 0 && q > 0) {
                if (record & REC_CONFIGS)
                    digest_rows_kernel<long long><<<dim3(gx, (unsigned)cfg_rows), 256, 0, e->stream>>>(e->st.tr_cfg, q, e->d_digest);
                if (record & REC_DELAYS)
                    digest_rows_kernel<int><<<dim3(gx, (unsigned)cfg_rows), 256, 0, e->stream>>>(e->st.tr_dly, q, e->d_digest + chunk);
            }
            if (sp_rows > 0 && q > 0 && (record & REC_SPIKING))
                digest_rows_kernel<int><<<dim3(gx, (unsigned)sp_rows), 256, 0, e->stream>>>(e->st.tr_chosen, q, e->d_digest + 2 * chunk);
            CU(cudaGetLastError());
            if (tr->config_digests && cfg_rows > 0)
                CU(cudaMemcpyAsync(tr->config_digests + r0, e->d_digest, cfg_rows * 8, cudaMemcpyDeviceToHost, e->stream));
            if (tr->delay_digests && cfg_rows > 0)
                CU(cudaMemcpyAsync(tr->delay_digests + r0, e->d_digest + chunk, cfg_rows * 8, cudaMemcpyDeviceToHost, e->stream));
            if (tr->spiking_digests && sp_rows > 0)
                CU(cudaMemcpyAsync(tr->spiking_digests + s0, e->d_digest + 2 * chunk, sp_rows * 8, cudaMemcpyDeviceToHost,
                                   e->stream));
            CU(cudaStreamSynchronize(e->stream));
            tr->config_rows += cfg_rows;
            tr->spiking_rows += sp_rows;
        } else if (record && cfg_rows > 0) {
            const long long r0 = tr->config_rows;
            if (tr->configs && (record & REC_CONFIGS))
                CU(cudaMemcpy(tr->configs + r0 * q, e->st.tr_cfg, cfg_rows * q * 8, cudaMemcpyDeviceToHost));
            if (tr->delays && (record & REC_DELAYS)) {
                tmp.resize((size_t)(cfg_rows * q));
                CU(cudaMemcpy(tmp.data(), e->st.tr_dly, cfg_rows * q * 4, cudaMemcpyDeviceToHost));
                for (long long i = 0; i < cfg_rows * q; ++i) tr->delays[r0 * q + i] = tmp[i];
            }
            if (tr->spiking && (record & REC_SPIKING) && sp_rows > 0) {
                tmp.resize((size_t)(sp_rows * q));
                CU(cudaMemcpy(tmp.data(), e->st.tr_chosen, sp_rows * q * 4, cudaMemcpyDeviceToHost));
                const long long s0 = tr->spiking_rows;
                for (long long i = 0; i < sp_rows * q; ++i) tr->spiking[s0 * q + i] = tmp[i];
            }
            tr->config_rows += cfg_rows;
            tr->spiking_rows += sp_rows;
        }
        budget -= (k1 - k0) + (c.halted ? 1 : 0);
    }
    CU(cudaEventRecord(e->ev1, e->stream));
    CU(cudaEventSynchronize(e->ev1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->last_ms = ms;
    fill_result(e, res);
    if (res) res->kernel_launches = launches;
    if (c.halted && c.reason == HALT_NEGATIVE)
        return fail(SNP_ERR_NEGATIVE, "spike counts went negative (neuron %lld: %lld); the applied rule consumed more than stored",
                    c.neg_index, c.neg_value);
    return SNP_OK;
}

int snp_read_state(snp_engine* e, int64_t* config, int64_t* delays) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    if (!e->hctrl.halted) return fail(SNP_ERR_BAD_ARG, "snp_read_state needs a halted run");
    CU(cudaSetDevice(e->device));
    const long long q = e->q;
    if (q == 0) return SNP_OK;
    // host or device destinations (cudaMemcpyDefault), ordered on the engine's stream
    if (config) CU(cudaMemcpyAsync(config, e->st.cfg, q * 8, cudaMemcpyDefault, e->stream));
    if (delays) {
        if (!e->scratch[0]) TRY(e->alloc(&e->scratch[0], q));
        ds_to_delay_kernel<<<grid_for(q), 256, 0, e->stream>>>(q, e->st.ds, e->scratch[0]);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(delays, e->scratch[0], q * 8, cudaMemcpyDefault, e->stream));
    }
    CU(cudaStreamSynchronize(e->stream));
    return SNP_OK;
}

int snp_run(snp_engine* e, const int64_t* initial, const snp_run_opts* o, int64_t* final_config,
            int64_t* final_delays, snp_result* res) {
    TRY(validate_opts(o));
    TRY(snp_begin(e, initial));
    TRY(snp_advance(e, o, o->max_steps + 1, nullptr, res));
    return snp_read_state(e, final_config, final_delays);
}

double snp_last_device_ms(const snp_engine* e) { return e ? e->last_ms : 0.0; }

int snp_time_steps(snp_engine* e, const snp_run_opts* o, int64_t steps, double* total_ms, double* kernel_ms,
                   snp_result* res) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    TRY(validate_opts(o));
    if (!e->begun) return fail(SNP_ERR_BAD_ARG, "snp_time_steps before snp_begin");
    CU(cudaSetDevice(e->device));
    Ctrl& c = e->hctrl;
    c.max_steps = o->max_steps;
    c.policy = o->policy;
    c.seed = o->seed;
    c.record = 0;
    c.stats_on = o->collect_stats ? 1 : 0;
    c.stop_at = c.step + steps;
    TRY(push_ctrl(e));
    long long launches = 0;
    if (e->small_fn) {
        // one launch runs all `steps` (kernel time = the whole segment / steps)
        CU(cudaEventRecord(e->ev0, e->stream));
        launch_main(e);
        launches = 1;
        CU(cudaGetLastError());
        CU(cudaEventRecord(e->ev1, e->stream));
        CU(cudaEventSynchronize(e->ev1));
        if (kernel_ms) {
            float ms = 0;
            CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
            *kernel_ms = steps > 0 ? ms / steps : 0.0;
        }
    } else if (kernel_ms) {
        // per-kernel CUDA events around the step kernel on the engine stream
        std::vector<cudaEvent_t> ev(2 * steps);
        for (auto& x : ev) CU(cudaEventCreate(&x));
        CU(cudaEventRecord(e->ev0, e->stream));
        for (long long i = 0; i < steps; ++i) {
            launches += launch_pass1(e);
            CU(cudaEventRecord(ev[2 * i], e->stream));
            launch_main(e);
            CU(cudaEventRecord(ev[2 * i + 1], e->stream));
            launches += 1;
            // push kernels of the same step (unfused push formats), launched after the timed one
            launches += launch_push_tail(e);
        }
        CU(cudaGetLastError());
        CU(cudaEventRecord(e->ev1, e->stream));
        CU(cudaEventSynchronize(e->ev1));
        double sum = 0;
        for (long long i = 0; i < steps; ++i) {
            float ms = 0;
            CU(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
            sum += ms;
        }
        for (auto& x : ev) cudaEventDestroy(x);
        *kernel_ms = steps > 0 ? sum / steps : 0.0;
    } else {
        // whole graph replays of `chunk` steps, the remainder launched directly:
        // exactly `steps` step iterations are enqueued
        const long long chunk = std::min<long long>((long long)steps, 64ll);
        if (chunk > 0) TRY(ensure_graph(e, chunk));
        CU(cudaEventRecord(e->ev0, e->stream));
        long long done = 0;
        while (chunk > 0 && done + chunk <= steps) {
            CU(cudaGraphLaunch(e->graph, e->stream));
            launches += chunk * kernels_per_step(e);
            done += chunk;
        }
        for (; done < steps; ++done) launches += launch_step(e);
        CU(cudaGetLastError());
        CU(cudaEventRecord(e->ev1, e->stream));
        CU(cudaEventSynchronize(e->ev1));
    }
    float tot = 0;
    CU(cudaEventElapsedTime(&tot, e->ev0, e->ev1));
    if (total_ms) *total_ms = tot;
    e->last_ms = tot;
    TRY(pull_ctrl(e));
    fill_result(e, res);
    if (res) res->kernel_launches = launches;
    if (c.halted && c.reason == HALT_NEGATIVE) return fail(SNP_ERR_NEGATIVE, "spike counts went negative");
    return SNP_OK;
}

// --------------------------------------------------------------- phase API

static int phase_scratch(snp_engine* e) {
    for (int i = 0; i < 4; ++i)
        if (!e->scratch[i]) TRY(e->alloc(&e->scratch[i], std::max<long long>(1, e->q)));
    return SNP_OK;
}

int snp_sv_calc(snp_engine* e, const int64_t* config, const int64_t* delays, int32_t policy, uint64_t seed,
                int64_t step, int64_t* chosen) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    if (policy != SNP_POLICY_FIRST && policy != SNP_POLICY_SEEDED) return fail(SNP_ERR_BAD_ARG, "unknown policy");
    if (step < 0) return fail(SNP_ERR_BAD_ARG, "step must be >= 0");
    CU(cudaSetDevice(e->device));
    const long long q = e->q;
    for (long long i = 0; i < q; ++i)
        if (delays[i] < 0 || delays[i] > kInt32Max - 2) return fail(SNP_ERR_BAD_ARG, "delay out of range");
    TRY(phase_scratch(e));
    TRY(ensure_trace(e, std::max<long long>(1, e->tr_rows)));
    TRY(reset_state(e));
    if (q > 0) {
        CU(cudaMemcpyAsync(e->scratch[0], config, q * 8, cudaMemcpyHostToDevice, e->stream));
        CU(cudaMemcpyAsync(e->scratch[1], delays, q * 8, cudaMemcpyHostToDevice, e->stream));
        load_state_kernel<<<grid_for(q), 256, 0, e->stream>>>(q, e->st.cfg, e->st.ds, e->scratch[0], e->scratch[1]);
        CU(cudaGetLastError());
    }
    Ctrl& c = e->hctrl;
    c.step = step;
    c.max_steps = step + 1;
    c.stop_at = step + 1;
    c.trace_base = step;
    c.policy = policy;
    c.seed = seed;
    c.record = REC_SPIKING;
    TRY(push_ctrl(e));
    launch_pass1(e);
    e->step_fn<<<e->step_grid, e->step_block, e->step_smem, e->stream>>>(e->sys, e->st);
    CU(cudaGetLastError());
    if (q > 0) {
        widen_i32_kernel<<<grid_for(q), 256, 0, e->stream>>>(q, e->st.tr_chosen, e->scratch[2]);
        CU(cudaMemcpyAsync(chosen, e->scratch[2], q * 8, cudaMemcpyDeviceToHost, e->stream));
    }
    TRY(pull_ctrl(e));
    e->begun = false;
    return SNP_OK;
}

int snp_step(snp_engine* e, const int64_t* config, const int64_t* delays, const int64_t* chosen,
             int64_t* next_config, int64_t* row_visits) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    CU(cudaSetDevice(e->device));
    const long long q = e->q, m = e->m;
    for (long long i = 0; i < q; ++i) {
        if (delays[i] < 0 || delays[i] > kInt32Max - 2) return fail(SNP_ERR_BAD_ARG, "delay out of range");
        if (chosen[i] < -1 || chosen[i] >= m) return fail(SNP_ERR_BAD_ARG, "chosen rule %lld out of range", (long long)chosen[i]);
    }
    TRY(phase_scratch(e));
    TRY(reset_state(e));
    long long* d_visits = nullptr;
    if (row_visits && e->format == SNP_FMT_ELL && m > 0) {
        TRY(e->alloc(&d_visits, m));
        CU(cudaMemcpyAsync(d_visits, row_visits, m * 8, cudaMemcpyHostToDevice, e->stream));
    }
    if (q > 0) {
        CU(cudaMemcpyAsync(e->scratch[0], config, q * 8, cudaMemcpyHostToDevice, e->stream));
        CU(cudaMemcpyAsync(e->scratch[1], delays, q * 8, cudaMemcpyHostToDevice, e->stream));
        CU(cudaMemcpyAsync(e->scratch[2], chosen, q * 8, cudaMemcpyHostToDevice, e->stream));
    }
    Ctrl& c = e->hctrl;
    c.step = 1;  // the prime kernel plays "step 0's selection"
    c.max_steps = 1;
    c.stop_at = 2;
    c.trace_base = 1;
    c.record = 0;
    c.push_armed = 1;
    TRY(push_ctrl(e));
    if (q > 0) {
        e->prime_fn<<<grid_for(q), 256, 0, e->stream>>>(e->sys, e->st, e->scratch[0], e->scratch[1], e->scratch[2]);
        CU(cudaGetLastError());
    }
    if (e->kind == RECV_ARRAY) {
        if (e->format == SNP_FMT_SPARSE) {
            dense_kernel<<<e->dense_grid, kBlock, 0, e->stream>>>(e->sys, e->st);
        } else if (e->format == SNP_FMT_ELL) {
            push_kernel<true><<<e->push_grid, kBlock, 0, e->stream>>>(e->sys, e->st, d_visits);
            push_heavy_kernel<true><<<e->heavy_push_grid, kBlock, 0, e->stream>>>(e->sys, e->st);
        } else {
            push_kernel<false><<<e->push_grid, kBlock, 0, e->stream>>>(e->sys, e->st, nullptr);
            push_heavy_kernel<false><<<e->heavy_push_grid, kBlock, 0, e->stream>>>(e->sys, e->st);
        }
        CU(cudaGetLastError());
    }
    launch_pass1(e);
    e->step_fn<<<e->step_grid, e->step_block, e->step_smem, e->stream>>>(e->sys, e->st);  // finalize only
    CU(cudaGetLastError());
    TRY(pull_ctrl(e));
    e->begun = false;
    if (c.halted && c.reason == HALT_NEGATIVE)
        return fail(SNP_ERR_NEGATIVE, "spike counts went negative (neuron %lld: %lld); the applied rule consumed more than stored",
                    c.neg_index, c.neg_value);
    if (q > 0) CU(cudaMemcpy(next_config, e->st.cfg, q * 8, cudaMemcpyDeviceToHost));
    if (d_visits) CU(cudaMemcpy(row_visits, d_visits, m * 8, cudaMemcpyDeviceToHost));
    return SNP_OK;
}

int snp_update_delays(snp_engine* e, const int64_t* delays, const int64_t* chosen, int64_t* next_delays) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    CU(cudaSetDevice(e->device));
    const long long q = e->q;
    for (long long i = 0; i < q; ++i)
        if (chosen[i] < -1 || chosen[i] >= e->m) return fail(SNP_ERR_BAD_ARG, "chosen rule out of range");
    if (q == 0) return SNP_OK;
    TRY(phase_scratch(e));
    CU(cudaMemcpyAsync(e->scratch[0], delays, q * 8, cudaMemcpyHostToDevice, e->stream));
    CU(cudaMemcpyAsync(e->scratch[1], chosen, q * 8, cudaMemcpyHostToDevice, e->stream));
    update_delays_kernel<<<grid_for(q), 256, 0, e->stream>>>(q, e->sys.rrec, e->scratch[0], e->scratch[1], e->scratch[2]);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(next_delays, e->scratch[2], q * 8, cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    return SNP_OK;
}

// --------------------------------------------------------------- row partition

int snp_exchange_info(const snp_engine* e, snp_exchange* x) {
    if (!e || !x) return fail(SNP_ERR_BAD_ARG, "null argument");
    memset(x, 0, sizeof(*x));
    for (int i = 0; i < 3; ++i) x->slot[i] = e->st.P[i];
    x->world = std::max(1, e->sys.world);
    x->rank = e->sys.rank;
    x->lo = e->shard_lo;
    x->hi = e->sys.x_stride ? e->shard_hi : e->q;
    x->chunk_bytes = e->sys.x_stride * 4;
    x->chunk_offset_bytes = (long long)e->sys.rank * e->sys.x_stride * 4;
    x->slot_bytes = e->sys.x_stride * 4 * x->world;
    x->neurons_per_rank = e->shard_nl;
    return SNP_OK;
}

int snp_set_stream(snp_engine* e, void* stream) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    e->stream = stream ? static_cast<cudaStream_t>(stream) : e->own_stream;
    return SNP_OK;
}

int snp_configure(snp_engine* e, const snp_run_opts* o) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    TRY(validate_opts(o));
    if (!e->begun) return fail(SNP_ERR_BAD_ARG, "snp_configure before snp_begin");
    CU(cudaSetDevice(e->device));
    Ctrl& c = e->hctrl;
    c.max_steps = o->max_steps;
    c.policy = o->policy;
    c.seed = o->seed;
    // recording (row partitions, snp_read_trace): every row of the run stays
    // in the device ring -- step k's rows at slot k (trace_base 0)
    const int rec = o->record & (SNP_REC_CONFIGS | SNP_REC_DELAYS | SNP_REC_SPIKING);
    if (rec) {
        const double bytes = ((double)o->max_steps + 2.0) * (double)std::max<long long>(1, e->q) * 16.0;
        if (bytes > 64e9)
            return fail(SNP_ERR_CAPACITY, "recording %lld steps of %lld neurons keeps %.1f GB of rows on the device",
                        (long long)o->max_steps, e->q, bytes / 1e9);
        TRY(ensure_trace(e, o->max_steps + 2));
    }
    c.record = rec;
    c.stats_on = o->collect_stats ? 1 : 0;
    c.stop_at = 0x3fffffffffffffffll;
    c.trace_base = 0;
    TRY(push_ctrl(e));
    CU(cudaStreamSynchronize(e->stream));
    return SNP_OK;
}

int snp_read_trace(snp_engine* e, int64_t first_row, int64_t n_rows, int64_t* configs, int64_t* delays,
                   int64_t* chosen) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    if (!e->hctrl.record) return fail(SNP_ERR_BAD_ARG, "snp_read_trace needs a run configured with record flags");
    if (first_row < 0 || n_rows < 0 || first_row + n_rows > e->tr_rows)
        return fail(SNP_ERR_BAD_ARG, "trace rows [%lld, %lld) outside the ring of %lld", (long long)first_row,
                    (long long)(first_row + n_rows), e->tr_rows);
    CU(cudaSetDevice(e->device));
    CU(cudaStreamSynchronize(e->stream));
    const long long q = e->q, n = n_rows * q, o = first_row * q;
    if (n == 0) return SNP_OK;
    if (configs) CU(cudaMemcpy(configs, e->st.tr_cfg + o, n * 8, cudaMemcpyDefault));
    std::vector<int> tmp;
    auto widen = [&](const int* src, int64_t* dst) -> int {
        tmp.resize((size_t)n);
        CU(cudaMemcpy(tmp.data(), src + o, n * 4, cudaMemcpyDeviceToHost));
        for (long long i = 0; i < n; ++i) dst[i] = tmp[i];
        return SNP_OK;
    };
    if (delays) TRY(widen(e->st.tr_dly, delays));
    if (chosen) TRY(widen(e->st.tr_chosen, chosen));
    return SNP_OK;
}

int snp_launch_step(snp_engine* e) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    CU(cudaSetDevice(e->device));
    launch_step(e);
    CU(cudaGetLastError());
    return SNP_OK;
}

int snp_poll(snp_engine* e, snp_result* res) {
    if (!e) return fail(SNP_ERR_BAD_ARG, "null engine");
    CU(cudaSetDevice(e->device));
    TRY(pull_ctrl(e));
    fill_result(e, res);
    if (e->hctrl.halted && e->hctrl.reason == HALT_NEGATIVE)
        return fail(SNP_ERR_NEGATIVE, "spike counts went negative (row-partitioned run)");
    if (e->hctrl.halted && e->hctrl.reason == HALT_EXCHANGE)
        return fail(SNP_ERR_CUDA, "peer exchange timed out at step %lld (a rank stopped stepping)", e->hctrl.step);
    return SNP_OK;
}

static int connect_peers(snp_engine* e, const std::vector<unsigned long long>& bases) {
    DevSys& s = e->sys;
    TRY(e->alloc(&e->d_peers, (long long)bases.size()));
    CU(cudaMemcpy(e->d_peers, bases.data(), bases.size() * 8, cudaMemcpyHostToDevice));
    s.peers = e->d_peers;
    s.p2p = 1;
    if (e->graph) {
        cudaGraphExecDestroy(e->graph);
        e->graph = nullptr;
    }
    return SNP_OK;
}

int snp_engine_layout_digest(const snp_engine* e, uint64_t* out) {
    if (e && e->sys.tp) {
        // two-pass layout: slots, offsets (as u32 pairs), gword, stages, tstage, window groups
        if (!out) return fail(SNP_ERR_BAD_ARG, "null argument");
        memset(out, 0, 6 * sizeof(uint64_t));
        CU(cudaSetDevice(e->device));
        const DevSys& s = e->sys;
        unsigned long long* d;
        CU(cudaMalloc(&d, 6 * 8));
        CU(cudaMemset(d, 0, 6 * 8));
        const long long groups = e->in_edges / 32;
        const long long n[6] = {groups * 16, groups * 16, groups, e->n_stages * 8, s.n_tiles + 1, s.tp_nw + 1};
        const uint32_t* a[6] = {reinterpret_cast<const uint32_t*>(s.tp_slots), reinterpret_cast<const uint32_t*>(s.tp_off),
                                s.tp_gword, reinterpret_cast<const uint32_t*>(s.stages), s.tstage, s.tp_wgroup};
        for (int i = 0; i < 6; ++i)
            if (n[i] > 0) digest_u32_kernel<<<grid_for(std::min<long long>(n[i], 148ll * 1024)), 256>>>(n[i], a[i], d + i);
        cudaError_t err = cudaGetLastError();
        if (err == cudaSuccess) err = cudaMemcpy(out, d, 6 * 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CU(err);
        return SNP_OK;
    }
    if (!e || !out) return fail(SNP_ERR_BAD_ARG, "null argument");
    memset(out, 0, 6 * sizeof(uint64_t));
    if (!e->tiled) return SNP_OK;
    CU(cudaSetDevice(e->device));
    const DevSys& s = e->sys;
    unsigned long long* d;
    CU(cudaMalloc(&d, 6 * 8));
    CU(cudaMemset(d, 0, 6 * 8));
    const long long n[6] = {e->in_edges, e->in_edges / kSegEdges, e->n_stages * 8, s.n_tiles + 1, s.n_tiles + 1,
                            e->n_sbases};
    const uint32_t* a[6] = {s.seg_words, s.seg_base, reinterpret_cast<const uint32_t*>(s.stages), s.tstage, s.tseg,
                            s.stage_bases};
    for (int i = 0; i < 6; ++i)
        if (n[i] > 0) digest_u32_kernel<<<grid_for(std::min<long long>(n[i], 148ll * 1024)), 256>>>(n[i], a[i], d + i);
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess) err = cudaMemcpy(out, d, 6 * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    CU(err);
    return SNP_OK;
}

int snp_exchange_ipc_handle(const snp_engine* e, void* handle) {
    if (!e || !handle) return fail(SNP_ERR_BAD_ARG, "null argument");
    if (!e->xblock) return fail(SNP_ERR_BAD_ARG, "not a row-partitioned engine");
    CU(cudaSetDevice(e->device));
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, e->xblock));
    memcpy(handle, &h, sizeof(h));
    return SNP_OK;
}

int snp_exchange_connect(snp_engine* e, const void* handles, int world) {
    if (!e || !handles) return fail(SNP_ERR_BAD_ARG, "null argument");
    if (!e->xblock || world != e->sys.world) return fail(SNP_ERR_BAD_ARG, "world %d does not match the engine", world);
    if (e->sys.p2p) return fail(SNP_ERR_BAD_ARG, "peer exchange already connected");
    CU(cudaSetDevice(e->device));
    std::vector<unsigned long long> bases(world);
    for (int r = 0; r < world; ++r) {
        if (r == e->sys.rank) {
            bases[r] = (unsigned long long)e->xblock;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, static_cast<const char*>(handles) + (size_t)r * SNP_IPC_HANDLE_BYTES, sizeof(h));
        void* p = nullptr;
        CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        e->ipc_opened.push_back(p);
        bases[r] = (unsigned long long)p;
    }
    return connect_peers(e, bases);
}

int snp_exchange_connect_local(snp_engine* const* engines, int world) {
    if (!engines || world < 1) return fail(SNP_ERR_BAD_ARG, "null argument");
    std::vector<unsigned long long> bases(world);
    for (int r = 0; r < world; ++r) {
        const snp_engine* x = engines[r];
        if (!x || !x->xblock || x->sys.world != world || x->sys.rank != r)
            return fail(SNP_ERR_BAD_ARG, "engine %d is not rank %d of a %d-way row partition", r, r, world);
        bases[r] = (unsigned long long)x->xblock;
    }
    for (int r = 0; r < world; ++r) {
        if (engines[r]->sys.p2p) return fail(SNP_ERR_BAD_ARG, "peer exchange already connected");
        CU(cudaSetDevice(engines[r]->device));
        TRY(connect_peers(engines[r], bases));
    }
    return SNP_OK;
}

}  // extern "C"
