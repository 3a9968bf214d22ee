// redbench.cu -- global (L2) reduction throughput for the ELL / Optimized push
// design: random RED.ADD into a 10^7-entry receive array (32- and 64-bit),
// alone and fed by a streamed pair array (the ELL column walk), with and
// without an L2 evict-first hint on the stream.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o redbench tools/redbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <typename T>
__global__ void red_hash(T* recv, uint32_t n, long long ops) {
    const long long nt = (long long)gridDim.x * blockDim.x;
    uint32_t h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ops; i += nt) {
        h = hash32(h + (uint32_t)i);
        atomicAdd(recv + (h % n), (T)1);
    }
}

__device__ __forceinline__ int4 ld_stream(const int4* p, bool ef) {
    int4 v;
    if (ef) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    } else
        v = __ldg(p);
    return v;
}

// pairs: (target, amount) int2, streamed two per lane (16 B)
template <typename T>
__global__ void red_stream(T* recv, const int4* __restrict__ pairs, long long n2, int mode, bool ef) {
    const long long nt = (long long)gridDim.x * blockDim.x;
    long long acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += nt) {
        const int4 v = ld_stream(pairs + i, ef);
        if (mode == 0) {
            acc += v.x + v.y + v.z + v.w;
        } else {
            atomicAdd(recv + v.x, (T)v.y);
            atomicAdd(recv + v.z, (T)v.w);
        }
    }
    if (acc == 0x7fffffffffffll) recv[0] = 1;
}

__global__ void fill_pairs(int2* p, long long n, uint32_t q, int local) {
    const long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += nt) {
        const uint32_t src = (uint32_t)(i / 16), k = (uint32_t)(i % 16);
        const uint32_t W = (q - 1) / 16;
        const uint32_t t = local ? (src + 1 + k * W + hash32((uint32_t)i) % W) % q : hash32((uint32_t)i * 2654435761u) % q;
        p[i] = make_int2((int)t, 1);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t q = 10000000;
    const long long E = 160000000;
    void* recv;
    int2* pairs;
    cudaMalloc(&recv, (size_t)q * 8);
    cudaMalloc(&pairs, (size_t)E * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    auto timeit = [&](auto fn) {
        fn();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        return ms / 5;
    };
    const int grid = nsm * 8, block = 256;
    float t;
    t = timeit([&] { red_hash<int><<<grid, block>>>((int*)recv, q, E); });
    printf("RED.S32 hash, 40MB array          %7.3f ms  %7.1f G ops/s\n", t, E / (t * 1e-3) / 1e9);
    t = timeit([&] { red_hash<unsigned long long><<<grid, block>>>((unsigned long long*)recv, q, E); });
    printf("RED.U64 hash, 80MB array          %7.3f ms  %7.1f G ops/s\n", t, E / (t * 1e-3) / 1e9);
    for (int local = 1; local >= 0; --local) {
        fill_pairs<<<grid, block>>>(pairs, E, q, local);
        const char* tag = local ? "synth" : "uniform";
        for (int ef = 0; ef < 2; ++ef) {
            t = timeit([&] { red_stream<int><<<grid, block>>>((int*)recv, (const int4*)pairs, E / 2, 0, ef); });
            printf("%-8s stream only (1.28 GB) ef=%d    %7.3f ms  %7.1f GB/s\n", tag, ef, t, E * 8 / (t * 1e-3) / 1e9);
            t = timeit([&] { red_stream<int><<<grid, block>>>((int*)recv, (const int4*)pairs, E / 2, 1, ef); });
            printf("%-8s stream + RED.S32 ef=%d        %7.3f ms  %7.1f G ops/s\n", tag, ef, t, E / (t * 1e-3) / 1e9);
            t = timeit([&] {
                red_stream<unsigned long long><<<grid, block>>>((unsigned long long*)recv, (const int4*)pairs, E / 2, 1, ef);
            });
            printf("%-8s stream + RED.U64 ef=%d        %7.3f ms  %7.1f G ops/s\n", tag, ef, t, E / (t * 1e-3) / 1e9);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
