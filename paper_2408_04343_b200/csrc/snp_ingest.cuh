// snp_ingest.cuh -- device-side build of the tiled layout (SURVEY.md 8(f)
// rank 1, at-scale ingest).  Produces exactly the arrays of the host
// reference build in snp_engine.cu (build_tiles), from the out-adjacency
// already on the device:
//
//   1. edge keys:   key = destination tile, value = src << 20 | slot
//   2. stable radix sort by tile (CUB) -> each tile's in-edges in source order
//   3. segmentation (warp per tile, greedy exactly as the host): segment
//      start / count / base (src & ~31) / last source; then the 256-word
//      segments (warp per segment, coalesced)
//   4. TMA stage descriptors and stage bases (warp per tile, same greedy)
//
// Counting passes and fill passes share one kernel (mode 0 counts per tile;
// the host scans the per-tile counts, which are small, then mode 1 fills).
#pragma once

#include <cub/device/device_radix_sort.cuh>

namespace snp {

// 1. thread per source: one key / value per out-edge
__global__ void ingest_keys_kernel(long long q, const uint32_t* __restrict__ soff, const uint32_t* __restrict__ sdst,
                                   uint32_t T, uint32_t* __restrict__ key, unsigned long long* __restrict__ val) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (long long)gridDim.x * blockDim.x) {
        for (uint32_t e = soff[i]; e < soff[i + 1]; ++e) {
            const uint32_t d = sdst[e];
            key[e] = d / T;
            val[e] = ((unsigned long long)i << 20) | (d % T);
        }
    }
}

// tile starts in the sorted keys: start[t] = first index with key >= t
__global__ void ingest_tile_starts_kernel(long long S, const uint32_t* __restrict__ key, long long n_tiles,
                                          unsigned long long* __restrict__ start) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t <= n_tiles; t += (long long)gridDim.x * blockDim.x) {
        long long lo = 0, hi = S;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if ((long long)key[mid] < t) lo = mid + 1;
            else hi = mid;
        }
        start[t] = (unsigned long long)lo;
    }
}

// 3a. warp per tile: greedy segmentation (host build_tiles loop).  mode 0:
// seg_count[t]; mode 1: per segment first edge, edge count, base, last.
__global__ void ingest_segments_kernel(long long n_tiles, const unsigned long long* __restrict__ start,
                                       const unsigned long long* __restrict__ val, int mode,
                                       uint32_t* __restrict__ seg_count, const uint32_t* __restrict__ tseg,
                                       unsigned long long* __restrict__ seg_first, uint32_t* __restrict__ seg_n,
                                       uint32_t* __restrict__ seg_base, uint32_t* __restrict__ seg_last) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += warps) {
        const unsigned long long e0 = start[t], e1 = start[t + 1];
        uint32_t g = mode ? tseg[t] : 0u, count = 0;
        uint32_t b = 0, n = kSegEdges, prev = 0;
        for (unsigned long long c = e0; c < e1; c += 32) {
            const unsigned long long my = c + lane;
            const uint32_t v = my < e1 ? (uint32_t)(val[my] >> 20) : 0u;
            const int cnt = (int)min(32ull, e1 - c);
            for (int k = 0; k < cnt; ++k) {
                const uint32_t src = __shfl_sync(0xffffffffu, v, k);
                if (n >= (uint32_t)kSegEdges || src - b >= kSrcSpan) {
                    // close the previous segment, open one at this edge
                    if (count > 0 && mode && lane == 0) {
                        seg_n[g - 1] = n;
                        seg_last[g - 1] = prev;
                    }
                    b = src & ~31u;
                    n = 0;
                    if (mode && lane == 0) {
                        seg_first[g] = c + k;
                        seg_base[g] = b;
                    }
                    ++g;
                    ++count;
                }
                ++n;
                prev = src;
            }
        }
        if (lane == 0) {
            if (mode) {
                if (count > 0) {
                    seg_n[g - 1] = n;
                    seg_last[g - 1] = prev;
                }
            } else {
                seg_count[t] = count;
            }
        }
    }
}

// 3b. warp per segment: the 256 words (slot << kSrcBits | src - base, padding T << kSrcBits)
__global__ void ingest_words_kernel(long long nseg, const unsigned long long* __restrict__ seg_first,
                                    const uint32_t* __restrict__ seg_n, const uint32_t* __restrict__ seg_base,
                                    const unsigned long long* __restrict__ val, uint32_t T, uint32_t* __restrict__ words) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < nseg; g += warps) {
        const unsigned long long f = seg_first[g];
        const uint32_t n = seg_n[g], b = seg_base[g];
        for (int p = lane; p < kSegEdges; p += 32) {
            uint32_t w = T << kSrcBits;
            if ((uint32_t)p < n) {
                const unsigned long long v = val[f + p];
                w = ((uint32_t)(v & 0xfffffu) << kSrcBits) | ((uint32_t)(v >> 20) - b);
            }
            words[g * kSegEdges + p] = w;
        }
    }
}

// 4. lane 0 of a warp per tile: stage descriptors (host build_tiles greedy).
// mode 0: stages[t], sbase words[t]; mode 1: fill desc / sbases.
struct IngestStageParams {
    long long q;
    uint32_t T;
    int stage_p;        // stage the P windows (P_BIT)
    int rpn;            // implicit rule offsets
    int tiny, wide;     // rule word width
    const uint32_t* roff;
};

__global__ void ingest_stages_kernel(long long n_tiles, const uint32_t* __restrict__ tseg,
                                     const uint32_t* __restrict__ seg_base, const uint32_t* __restrict__ seg_last,
                                     IngestStageParams P, int mode, uint32_t* __restrict__ n_stage,
                                     uint32_t* __restrict__ n_sbase, const uint32_t* __restrict__ tstage,
                                     const uint32_t* __restrict__ tsbase, StageDesc* __restrict__ desc,
                                     uint32_t* __restrict__ sbases) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const uint32_t rw_size = P.tiny ? 4u : (P.wide ? 16u : 8u);
    auto r16 = [](unsigned long long x) { return (uint32_t)((x + 15) & ~15ull); };
    for (long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += warps) {
        if (lane != 0) continue;
        uint32_t g = tseg[t];
        const uint32_t g1 = tseg[t + 1];
        uint32_t ns = 0, nb = 0;
        uint32_t di = mode ? tstage[t] : 0u, bo = mode ? tsbase[t] : 0u;
        do {
            uint32_t n = 0, src0 = 0, pbytes = 0;
            if (g < g1) {
                src0 = seg_base[g] & ~127u;
                while (g + n < g1 && n < kMaxSegPerStage) {
                    const uint32_t pb = P.stage_p ? r16((seg_last[g + n] + 1u - src0 + 7u) / 8u) : 0u;
                    if (kPayload + (n + 1) * kSegEdges * 4u + pb > kStageBytes) break;
                    pbytes = pb;
                    ++n;
                }
            }
            const uint32_t padded = (n + 3u) & ~3u;
            if (mode) {
                for (uint32_t i = 0; i < padded; ++i) sbases[bo + i] = i < n ? seg_base[g + i] : 0u;
                StageDesc sd;
                sd.a = make_uint4(1u | ((g + n >= g1) ? 256u : 0u), g, n, src0);
                sd.b = make_uint4(pbytes, bo, 0, 0);
                desc[di++] = sd;
            }
            bo += padded;
            nb += padded;
            ++ns;
            g += n;
        } while (g < g1);
        const long long d0 = t * (long long)P.T;
        const long long nd = min((long long)P.T, P.q - d0);
        for (long long dd = 0; dd < nd; dd += kSub) {
            if (mode) {
                const uint32_t n = (uint32_t)min((long long)kSub, nd - dd);
                const uint32_t rf = P.roff[d0 + dd], rl = P.roff[d0 + dd + n];
                const uint32_t r_al = P.tiny ? (rf & ~3u) : (P.wide ? rf : (rf & ~1u));
                const uint32_t fixed = kPayload + kP2Rules(P.rpn != 0);
                uint32_t rb = r16((unsigned long long)(rl - r_al) * rw_size);
                if (fixed + rb > kStageBytes) rb = 0;
                StageDesc sd;
                sd.a = make_uint4(2u | ((dd + kSub >= nd) ? 256u : 0u), (uint32_t)dd, n, r_al);
                sd.b = make_uint4(rb, 0, 0, 0);
                desc[di++] = sd;
            }
            ++ns;
        }
        if (!mode) {
            n_stage[t] = ns;
            n_sbase[t] = nb;
        }
    }
}

// Layout digest (diagnostics / tests): sum of fmix64(word * A + (i + 1) * B)
__global__ void digest_u32_kernel(long long n, const uint32_t* __restrict__ a, unsigned long long* out) {
    unsigned long long acc = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc += fmix64((unsigned long long)a[i] * 0x9E3779B97F4A7C15ull + (unsigned long long)(i + 1) * 0xD6E8FEB86659FD93ull);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

}  // namespace snp

namespace snp {

// ---- two-pass layout (variant TILED2) ----------------------------------------
// key = tile * nw + window (tile order), value = xsrc << 20 | slot

__global__ void tp_keys_csr_kernel(long long q, const uint32_t* __restrict__ soff, const uint32_t* __restrict__ sdst,
                                   uint32_t T, uint32_t wlog, uint32_t nw, uint32_t* __restrict__ key,
                                   unsigned long long* __restrict__ val) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (long long)gridDim.x * blockDim.x) {
        for (uint32_t e = soff[i]; e < soff[i + 1]; ++e) {
            const uint32_t d = sdst[e];
            key[e] = (d / T) * nw + ((uint32_t)i >> wlog);
            val[e] = ((unsigned long long)i << 20) | (d % T);
        }
    }
}

__global__ void tp_keys_list_kernel(long long S, const uint32_t* __restrict__ xsrc, const uint32_t* __restrict__ ldst,
                                    uint32_t T, uint32_t wlog, uint32_t nw, uint32_t* __restrict__ key,
                                    unsigned long long* __restrict__ val) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < S; e += (long long)gridDim.x * blockDim.x) {
        const uint32_t d = ldst[e], x = xsrc[e];
        key[e] = (d / T) * nw + (x >> wlog);
        val[e] = ((unsigned long long)x << 20) | (d % T);
    }
}

__global__ void tp_hist_kernel(long long S, const uint32_t* __restrict__ key, uint32_t* __restrict__ cnt) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < S; e += (long long)gridDim.x * blockDim.x)
        atomicAdd(cnt + key[e], 1u);
}

// sorted edge i -> its tile-order slot and window-order source offset
__global__ void tp_fill_kernel(long long S, const uint32_t* __restrict__ key, const unsigned long long* __restrict__ val,
                               const unsigned long long* __restrict__ off_raw, const unsigned long long* __restrict__ off2,
                               const unsigned long long* __restrict__ off1, uint32_t nt, uint32_t nw, uint32_t wlog,
                               uint16_t* __restrict__ slots, uint16_t* __restrict__ offs) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t k = key[i], t = k / nw, w = k - t * nw;
        const unsigned long long j = (unsigned long long)i - off_raw[k];
        const unsigned long long v = val[i];
        slots[off2[k] + j] = (uint16_t)(v & 0xfffffu);
        offs[off1[(unsigned long long)w * nt + t] + j] = (uint16_t)((uint32_t)(v >> 20) - (w << wlog));
    }
}

// window-order group -> tile-order group, per chunk
__global__ void tp_gword_kernel(long long nk, const uint32_t* __restrict__ cnt, const unsigned long long* __restrict__ off2,
                                const unsigned long long* __restrict__ off1, uint32_t nt, uint32_t nw,
                                uint32_t* __restrict__ gword) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += (long long)gridDim.x * blockDim.x) {
        const uint32_t ng = (cnt[k] + 31u) >> 5;
        if (!ng) continue;
        const uint32_t t = (uint32_t)(k / nw), w = (uint32_t)(k - (long long)t * nw);
        const unsigned long long g2 = off2[k] >> 5, g1 = off1[(unsigned long long)w * nt + t] >> 5;
        for (uint32_t j = 0; j < ng; ++j) gword[g1 + j] = (uint32_t)(g2 + j);
    }
}

__global__ void fill_u16_kernel(long long n, uint16_t* p, uint16_t v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

}  // namespace snp
