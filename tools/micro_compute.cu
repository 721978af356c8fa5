// tools/micro_compute.cu -- isolate the cost of the replay kernel's compute-warp body
// (decode + running sum/max/min + Tier-E shared atomics + Bloom + chunk scan) with the
// events already resident in shared memory.  Variants toggle each part.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_compute tools/micro_compute.cu
#include <cstdio>
#include <cstdint>
#include <climits>
#include <vector>
#include <random>
#include <cuda_runtime.h>

constexpr int kHot = 1024;
__device__ unsigned long long g_sink;




__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void red_add_if(unsigned a, unsigned v, bool c) {
    asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p red.shared.add.u32 [%0], %1; }" :: "r"(a), "r"(v), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ void red_or_if(unsigned a, unsigned v, bool c) {
    asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p red.shared.or.b32 [%0], %1; }" :: "r"(a), "r"(v), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ unsigned atom_add_if(unsigned a, unsigned v, bool c) {
    unsigned o = 0;
    asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p atom.shared.add.u32 %0, [%1], %3; }" : "+r"(o) : "r"(a), "r"((unsigned)c), "r"(v) : "memory");
    return o;
}

// optimized body: predicated shared atomics, 32-bit scan + REDUX
template <bool CARRY>
__global__ void body2(const ulonglong2* __restrict__ ev, int boxes, unsigned long long* out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    ulonglong2* box = reinterpret_cast<ulonglong2*>(sm);
    unsigned* cnt = reinterpret_cast<unsigned*>(sm + 32768);
    unsigned* blo = cnt + 2 * kHot;
    unsigned* bhi = blo + 2 * kHot;
    unsigned* bloom = bhi + 2 * kHot;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < 2048; i += blockDim.x) box[i] = ev[i + 2048 * (blockIdx.x % 64)];
    for (int i = tid; i < 6 * kHot + 8 * 64 * 4; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const unsigned cnt_s = saddr(cnt), blo_s = saddr(blo), bhi_s = saddr(bhi), bl_s = saddr(bloom) + (w % 8) * 256;
    long long acc = 0;
    for (int it = 0; it < boxes; ++it) {
        const int r = (w % 8) * 32 + lane;
        const unsigned char* rowp = sm + (size_t)r * 128;
        unsigned long long ptr[8], meta[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            ulonglong2 v = *reinterpret_cast<const ulonglong2*>(rowp + ((j ^ (r & 7)) << 4));
            ptr[j] = v.x; meta[j] = v.y ^ (unsigned long long)(it & 1);
        }
        int r32 = 0, mx32 = INT_MIN, mn32 = INT_MAX;
        unsigned old[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned hi = (unsigned)(meta[j] >> 32), lo = (unsigned)meta[j] & 0x7ffffff;
            const unsigned kind = (hi >> 8) & 3u, site = (hi >> 11) & (kHot - 1);
            const bool v = kind < 2;
            r32 += kind == 0 ? (int)lo : (kind == 1 ? -(int)lo : 0);
            mx32 = max(mx32, r32); mn32 = min(mn32, r32);
            const unsigned x = ((kind & 1u) * kHot + site) * 4;
            red_add_if(cnt_s + x, 1u, v);
            if (CARRY) old[j] = atom_add_if(blo_s + x, lo, v); else red_add_if(blo_s + x, lo, v);
            const unsigned b = ((unsigned)(ptr[j] >> 4) * 0x9E3779B1u) >> 21;
            red_or_if(bl_s + (b >> 5) * 4, 1u << (b & 31), kind == 1);
        }
        if (CARRY) {
            #pragma unroll
            for (int j = 0; j < 8; ++j) {
                const unsigned hi = (unsigned)(meta[j] >> 32), lo = (unsigned)meta[j] & 0x7ffffff;
                const unsigned x = (((hi >> 8) & 1u) * kHot + ((hi >> 11) & (kHot - 1))) * 4;
                red_add_if(bhi_s + x, 1u, ((hi >> 8) & 3u) < 2 && old[j] + lo < old[j]);
            }
        }
        // 32-bit chunk summary (valid when all |lane sums| < 2^25)
        int incl = r32;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { int o = __shfl_up_sync(~0u, incl, d); if (lane >= d) incl += o; }
        const int a = __reduce_max_sync(~0u, incl - r32 + mx32), b = __reduce_min_sync(~0u, incl - r32 + mn32);
        acc += (long long)a ^ b ^ incl;
    }
    if (acc == 0x1234567) g_sink = 1;
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = cnt[0] + blo[5] + bloom[3];
}

template <bool ATOM, bool BLOOM, bool SCAN, bool CARRY>
__global__ void body(const ulonglong2* __restrict__ ev, int boxes, unsigned long long* out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    ulonglong2* box = reinterpret_cast<ulonglong2*>(sm);                 // 2048 events
    unsigned* cnt = reinterpret_cast<unsigned*>(sm + 32768);
    unsigned* blo = cnt + 2 * kHot;
    unsigned* bhi = blo + 2 * kHot;
    unsigned* bloom = bhi + 2 * kHot;                                     // 8 x 64 words
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    for (int i = tid; i < 2048; i += blockDim.x) box[i] = ev[i + 2048 * (blockIdx.x % 64)];
    for (int i = tid; i < 6 * kHot + 8 * 64 * 4; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    long long acc = 0;
    for (int it = 0; it < boxes; ++it) {
        const int r = (w % 8) * 32 + lane;
        const unsigned char* rowp = sm + (size_t)r * 128;
        unsigned long long ptr[8], meta[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            ulonglong2 v = *reinterpret_cast<const ulonglong2*>(rowp + ((j ^ (r & 7)) << 4));
            ptr[j] = v.x; meta[j] = v.y ^ (unsigned long long)(it & 1);   // defeat hoisting
        }
        int r32 = 0, mx32 = INT_MIN, mn32 = INT_MAX;
        unsigned vmask = 0;
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned kind = (unsigned)(meta[j] >> 40) & 3u;
            const int sz = (int)((unsigned)meta[j] & 0x7ffffff);
            r32 += kind == 0 ? sz : (kind == 1 ? -sz : 0);
            mx32 = max(mx32, r32); mn32 = min(mn32, r32);
            vmask |= (kind < 2 ? 1u : 0u) << j;
        }
        if (ATOM) {
            unsigned old[8];
            #pragma unroll
            for (int j = 0; j < 8; ++j) {
                const unsigned hi = (unsigned)(meta[j] >> 32);
                const unsigned kind = (hi >> 8) & 1u, site = (hi >> 11) & (kHot - 1);
                old[j] = 0;
                if ((vmask >> j) & 1u) {
                    atomicAdd(&cnt[kind * kHot + site], 1u);
                    if (CARRY) old[j] = atomicAdd(&blo[kind * kHot + site], (unsigned)meta[j]);
                    else atomicAdd(&blo[kind * kHot + site], (unsigned)meta[j]);
                }
            }
            if (CARRY) {
                #pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const unsigned hi = (unsigned)(meta[j] >> 32), szu = (unsigned)meta[j];
                    if (((vmask >> j) & 1u) && old[j] + szu < old[j]) atomicAdd(&bhi[((hi >> 8) & 1u) * kHot + ((hi >> 11) & (kHot - 1))], 1u);
                }
            }
        }
        if (BLOOM) {
            #pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (((vmask >> j) & 1u) && ((meta[j] >> 40) & 1u)) {
                    const unsigned b = ((unsigned)(ptr[j] >> 4) * 0x9E3779B1u) >> 21;
                    atomicOr(&bloom[(w % 8) * 64 + (b >> 5)], 1u << (b & 31));
                }
            }
        }
        long long run = r32, tmx = mx32, tmn = mn32;
        if (SCAN) {
            long long incl = run;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { long long o = __shfl_up_sync(~0u, incl, d); if (lane >= d) incl += o; }
            long long a = (incl - run) + tmx, b = (incl - run) + tmn;
            #pragma unroll
            for (int d = 16; d > 0; d >>= 1) { a = llmax(a, __shfl_xor_sync(~0u, a, d)); b = llmin(b, __shfl_xor_sync(~0u, b, d)); }
            acc += a ^ b ^ incl;
        } else {
            acc += run ^ tmx ^ tmn;
        }
    }
    if (acc == 0x1234567) g_sink = 1;
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = cnt[0] + blo[5] + bloom[3];
}

int main() {
    cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
    const int nsm = prop.multiProcessorCount;
    // events shaped like config 2: Zipf(0.8) sites over 1000, sizes 16..512 mostly, ~half frees
    std::vector<unsigned long long> h(2 * 2048 * 64);
    std::mt19937_64 g(1);
    std::vector<double> cdf(1000); double acc = 0;
    for (int i = 0; i < 1000; ++i) { acc += 1.0 / pow(i + 1, 0.8); cdf[i] = acc; }
    for (auto& v : cdf) v /= acc;
    for (size_t i = 0; i < h.size() / 2; ++i) {
        double u = (g() >> 11) * (1.0 / 9007199254740992.0);
        unsigned site = std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
        unsigned kind = g() & 1, size = 16 * (1 + (g() >> 59));
        h[2 * i] = 0x100000000000ull + 16 * (g() % 100000);
        h[2 * i + 1] = size | ((unsigned long long)kind << 40) | ((unsigned long long)site << 43);
    }
    ulonglong2* d; cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    unsigned long long* out; cudaMalloc(&out, 8 * 4096);
    const int smem = 32768 + 6 * kHot * 4 + 8 * 64 * 4 * 4;
    const int boxes = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](auto kern, const char* name, int warps) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0); kern<<<nsm, warps * 32, smem>>>(d, boxes, out); cudaEventRecord(e1);
            cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        }
        // each warp processes `boxes` chunks of 256 events
        double events = (double)nsm * warps * 256 * boxes;
        printf("%-34s warps/CTA=%2d: %.3g events/s  (%.0f cycles per 256-event chunk per warp)  err=%s\n", name, warps,
               events / (ms * 1e-3), ms * 1e-3 * prop.clockRate * 1e3 / boxes, cudaGetErrorString(cudaGetLastError()));
    };
    for (int warps : {8, 12, 16}) {
        run(body2<true>, "OPT: pred atomics+carry+bloom, 32b scan", warps);
        run(body2<false>, "OPT: same without carry", warps);
    }
    for (int warps : {8, 16}) {
        run(body<false, false, false, false>, "decode+sum only", warps);
        run(body<false, false, true, false>, "+scan", warps);
        run(body<true, false, true, false>, "+atomics (no carry)", warps);
        run(body<true, false, true, true>, "+atomics+carry", warps);
        run(body<true, true, true, true>, "+atomics+carry+bloom (full)", warps);
        run(body<false, true, true, false>, "bloom+scan (no tierE)", warps);
    }
    return 0;
}
