// tools/microbench.cu -- B200 probes that shaped the replay kernel design
// (DESIGN.md §5): HBM streaming with LDG.128 vs cp.async.bulk (TMA bulk) into
// a shared-memory ring, and shared-memory atomic throughput (32-bit native
// ATOMS.ADD vs the 64-bit CAS loop ptxas emits for u64 atomicAdd on smem).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_sink;

__global__ void k_ldg(const int4* __restrict__ p, size_t n16) {
    int4 acc = make_int4(0, 0, 0, 0);
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        int4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
        acc.x ^= a.x ^ b.x ^ c.x ^ d.x; acc.y ^= a.y ^ b.y ^ c.y ^ d.y;
        acc.z ^= a.z ^ b.z ^ c.z ^ d.z; acc.w ^= a.w ^ b.w ^ c.w ^ d.w;
    }
    for (; i < n16; i += stride) { int4 a = __ldcs(p + i); acc.x ^= a.x; acc.y ^= a.y; acc.z ^= a.z; acc.w ^= a.w; }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) g_sink = 1;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(smem_u32(b)), "r"(phase) : "memory");
}

// TMA bulk ring: tiles of TILE bytes, STAGES deep; 256 consumer threads XOR the tile.
template <int TILE, int STAGES>
__global__ void __launch_bounds__(256) k_bulk(const char* __restrict__ p, size_t ntiles) {
    extern __shared__ __align__(128) char sm[];
    uint64_t* bar = (uint64_t*)(sm + TILE * STAGES);
    if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    size_t first = blockIdx.x, step = gridDim.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s) {
            size_t t = first + s * step;
            if (t < ntiles) { mbar_expect_tx(&bar[s], TILE); bulk_g2s(sm + s * TILE, p + t * TILE, TILE, &bar[s]); }
        }
    int4 acc = make_int4(0, 0, 0, 0);
    int k = 0;
    for (size_t t = first; t < ntiles; t += step, ++k) {
        int s = k % STAGES; uint32_t ph = (k / STAGES) & 1;
        mbar_wait(&bar[s], ph);
        const int4* q = (const int4*)(sm + s * TILE);
        #pragma unroll 4
        for (int i = threadIdx.x; i < TILE / 16; i += 256) { int4 a = q[i]; acc.x ^= a.x; acc.y ^= a.y; acc.z ^= a.z; acc.w ^= a.w; }
        __syncthreads();
        size_t tn = t + (size_t)STAGES * step;
        if (threadIdx.x == 0 && tn < ntiles) { mbar_expect_tx(&bar[s], TILE); bulk_g2s(sm + s * TILE, p + tn * TILE, TILE, &bar[s]); }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) g_sink = 1;
}

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// smem atomics: each thread ITER x 8 atomics to pseudo-random slots of a TAB-entry table
template <int MODE>   // 0: u32 add no return; 1: u32 add with return used; 2: u64 atomicAdd (CAS loop); 3: two u32 adds
__global__ void __launch_bounds__(256) k_atoms(unsigned long long* out, int iters, int tabmask) {
    extern __shared__ __align__(16) uint32_t tab[];
    for (int i = threadIdx.x; i <= tabmask * 2 + 1; i += blockDim.x) tab[i] = 0;
    __syncthreads();
    uint32_t seed = hsh(blockIdx.x * 256 + threadIdx.x), acc = 0;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t h = hsh(seed + it * 8 + j);
            uint32_t slot = h & tabmask;
            if (MODE == 0) atomicAdd(&tab[slot], h >> 20);
            else if (MODE == 1) { uint32_t o = atomicAdd(&tab[slot], h >> 8); acc += (o + (h >> 8) < o); }
            else if (MODE == 2) atomicAdd((unsigned long long*)&tab[2 * slot], (unsigned long long)(h >> 8));
            else { atomicAdd(&tab[2 * slot], 1u); atomicAdd(&tab[2 * slot + 1], h >> 8); }
        }
    }
    __syncthreads();
    unsigned long long s = acc;
    for (int i = threadIdx.x; i <= tabmask; i += blockDim.x) s += tab[i];
    atomicAdd(out, s);
}

int main() {
    int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
    int nsm = prop.multiProcessorCount;
    printf("device %s, %d SMs, clock %d kHz, L2 %d MB\n", prop.name, nsm, prop.clockRate, prop.l2CacheSize >> 20);
    size_t bytes = 4ull << 30;
    char* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
    unsigned long long* out; CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int bpsm : {4, 8, 16}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0); k_ldg<<<nsm * bpsm, 256>>>((const int4*)buf, bytes / 16); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("ldg128 grid-stride  %2d CTA/SM x256: %.1f GB/s\n", bpsm, bytes / ms / 1e6);
    }
    {
        constexpr int TILE = 16384, ST = 4;
        int smem = TILE * ST + 64;
        CK(cudaFuncSetAttribute(k_bulk<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int bpsm : {1, 2, 3}) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0); k_bulk<TILE, ST><<<nsm * bpsm, 256, smem>>>(buf, bytes / TILE); cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            }
            printf("bulk 16KBx4 ring    %2d CTA/SM: %.1f GB/s\n", bpsm, bytes / ms / 1e6);
        }
    }
    {
        constexpr int TILE = 32768, ST = 3;
        int smem = TILE * ST + 64;
        CK(cudaFuncSetAttribute(k_bulk<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int bpsm : {1, 2}) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0); k_bulk<TILE, ST><<<nsm * bpsm, 256, smem>>>(buf, bytes / TILE); cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            }
            printf("bulk 32KBx3 ring    %2d CTA/SM: %.1f GB/s\n", bpsm, bytes / ms / 1e6);
        }
    }
    const int iters = 2048;
    for (int mode = 0; mode < 4; ++mode) {
        for (int tabbits : {10, 13}) {
            int mask = (1 << tabbits) - 1, smem = (mask + 1) * 8;
            auto fn = mode == 0 ? k_atoms<0> : mode == 1 ? k_atoms<1> : mode == 2 ? k_atoms<2> : k_atoms<3>;
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0); fn<<<nsm * 4, 256, smem>>>(out, iters, mask); cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            }
            double ops = (double)nsm * 4 * 256 * iters * 8 * (mode == 3 ? 2 : 1);
            double per_sm_cyc = ops / nsm / (ms * 1e-3) / (prop.clockRate * 1e3);
            printf("atoms mode %d tab 2^%d: %.3g atom/s  = %.2f atom/cycle/SM (at %d MHz)  -> %.3g events/s at %s\n",
                   mode, tabbits, ops / (ms * 1e-3), per_sm_cyc, prop.clockRate / 1000,
                   ops / (ms * 1e-3) / (mode == 3 ? 2 : 1), mode == 3 ? "2 atoms/event" : "1 atom/event");
        }
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
