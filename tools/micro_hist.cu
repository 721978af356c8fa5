// tools/micro_hist.cu -- throughput probes for the per-site Tier-E reduce with many sites
// (config 3: 50,000 sites; DESIGN.md §5 "cold sites"): random-key updates through
//   L2 reductions (red.global.add.u64 / .u32),
//   local shared-memory atomics (ATOMS), and
//   distributed shared memory of a thread-block cluster (red.shared::cluster.add.u32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_hist tools/micro_hist.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MODE 0: two red.global.add.u64 per update (count, bytes) into [keys][4] u64
//      1: one red.global.add.u64
//      2: one red.global.add.u32 into [keys] u32
template <int MODE>
__global__ void __launch_bounds__(512) k_l2(unsigned long long* tab, int iters, uint32_t nkeys) {
    uint32_t s = hsh(blockIdx.x * 512 + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
        s = hsh(s + it);
        const uint32_t k = s % nkeys;
        if (MODE == 0) {
            asm volatile("red.global.add.u64 [%0], %1;" :: "l"(tab + 4ull * k), "l"(1ull) : "memory");
            asm volatile("red.global.add.u64 [%0], %1;" :: "l"(tab + 4ull * k + 2), "l"((unsigned long long)(s & 511)) : "memory");
        } else if (MODE == 1) {
            asm volatile("red.global.add.u64 [%0], %1;" :: "l"(tab + 4ull * k), "l"((unsigned long long)(s & 511)) : "memory");
        } else {
            asm volatile("red.global.add.u32 [%0], %1;" :: "l"((uint32_t*)tab + k), "r"(s & 511) : "memory");
        }
    }
}

// shared-memory table of words u32 per CTA; MODE 0 local ATOMS (red), 1 DSMEM red to a random CTA
// of the cluster, 2 DSMEM red, half local (own rank) half remote
template <int MODE>
__global__ void __launch_bounds__(512) k_sm(unsigned long long* out, int iters, uint32_t words) {
    extern __shared__ __align__(16) uint32_t tab[];
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) tab[i] = 0;
    uint32_t csize = 1, crank = 0;
    if (MODE) {
        asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
    uint32_t s = hsh(blockIdx.x * 512 + threadIdx.x);
    const uint32_t base = smem_u32(tab);
    for (int it = 0; it < iters; ++it) {
        s = hsh(s + it);
        const uint32_t k = (s >> 8) % words;
        const uint32_t a = base + 4 * k;
        if (MODE == 0) {
            asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a), "r"(s & 255) : "memory");
        } else {
            const uint32_t dst = MODE == 1 ? (s & (csize - 1)) : ((s & 1) ? crank : (s >> 1) & (csize - 1));
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(dst));
            asm volatile("red.shared::cluster.add.u32 [%0], %1;" :: "r"(ra), "r"(s & 255) : "memory");
        }
    }
    if (MODE) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    uint32_t acc = 0;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) acc += tab[i];
    atomicAdd(out, (unsigned long long)acc);
}

template <class K>
static float run(K kern, dim3 grid, int threads, size_t smem, int cluster, void** args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelExC(&cfg, (const void*)kern, args);
        cudaEventRecord(b);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return -1; }
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    return best;
}

int main() {
    int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* tab; CK(cudaMalloc(&tab, 200000ull * 4 * 8)); CK(cudaMemset(tab, 0, 200000ull * 32));
    unsigned long long* out; CK(cudaMalloc(&out, 8));
    const int iters = 4096, threads = 512;
    for (uint32_t nkeys : {100000u, 96000u, 20000u}) {
        int it = iters; uint32_t nk = nkeys;
        void* args[] = {&tab, &it, &nk};
        const double ops = (double)nsm * threads * iters;
        float m0 = run(k_l2<0>, dim3(nsm), threads, 0, 1, args);
        float m1 = run(k_l2<1>, dim3(nsm), threads, 0, 1, args);
        float m2 = run(k_l2<2>, dim3(nsm), threads, 0, 1, args);
        printf("L2 keys=%u: 2x red.u64 %.1f G updates/s (%.1f G reds/s) | 1x red.u64 %.1f G/s | 1x red.u32 %.1f G/s\n",
               nkeys, ops / m0 / 1e6, 2 * ops / m0 / 1e6, ops / m1 / 1e6, ops / m2 / 1e6);
    }
    CK(cudaFuncSetAttribute(k_sm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_sm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_sm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_sm<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_sm<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (uint32_t words : {12288u, 24576u, 49152u}) {
        int it = iters; uint32_t w = words;
        void* args[] = {&out, &it, &w};
        const double ops = (double)nsm * threads * iters;
        float ml = run(k_sm<0>, dim3(nsm), threads, words * 4, 1, args);
        printf("smem words=%u: local red.shared %.1f G/s (%.2f /clk/SM @1.965GHz)\n", words, ops / ml / 1e6,
               ops / ml / 1e6 / nsm / 1.965);
        for (int cs : {2, 4, 8}) {
            const int g = (nsm / cs) * cs;
            const double opc = (double)g * threads * iters;
            float mr = run(k_sm<1>, dim3(g), threads, words * 4, cs, args);
            float mh = run(k_sm<2>, dim3(g), threads, words * 4, cs, args);
            printf("   cluster %d (grid %d): DSMEM red random CTA %.1f G/s (%.2f /clk/SM) | half-own %.1f G/s\n", cs, g,
                   opc / mr / 1e6, opc / mr / 1e6 / g / 1.965, opc / mh / 1e6);
        }
    }
    return 0;
}
