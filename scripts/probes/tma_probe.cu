// Read/write-only probe (VERDICT r1 "settle the TMA question"): does moving a
// tile's 19 x 64 values through shared memory with bulk copies (TMA engine,
// cp.async.bulk -> UBLKCP) beat the per-thread LDG/STG path of the step
// kernel's read-write-only variant (step_impl.cuh, TLBM_READ_WRITE_ONLY)?
//
// Both kernels copy t_n tiles of 19 * 64 fp64 values (9,728 B, one
// contiguous tile record of the block store, layout.py:115-132) from one
// copy to the other -- 2 x 19 x 8 = 304 B per node, the step's algorithmic
// traffic.  t_n = 262,144 is the 256^3 channel (2.55 GB per copy, > L2).
//   ldg  : 64 threads per tile, 2 tiles per CTA, 19 loads then 19 stores per
//          thread (the rw-only step minus the node word)
//   bulk : persistent, one CTA per resident slot; one elected thread runs an
//          S-stage ring: cp.async.bulk global->shared (mbarrier complete_tx)
//          then cp.async.bulk shared->global (bulk_group), reusing a stage
//          once its store has read it (cp.async.bulk.wait_group.read)
//   memcpy: cudaMemcpyAsync device->device of the same bytes
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -o scripts/probes/tma_probe scripts/probes/tma_probe.cu
// Prints one JSON line per kernel (best of R launches, CUDA events).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

constexpr int Q = 19;
constexpr int TILE = Q * 64;                 // values per tile
constexpr int TILE_BYTES = TILE * 8;         // 9,728

__global__ void __launch_bounds__(128, 8) ldg_rw(const double *__restrict__ src,
                                                 double *__restrict__ dst, long long t_n) {
    const long long t = blockIdx.x * 2LL + (threadIdx.x >> 6);
    const int j = threadIdx.x & 63;
    if (t >= t_n) return;
    const double *s = src + t * TILE + j;
    double g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = __ldg(s + q * 64);
    double *d = dst + t * TILE + j;
#pragma unroll
    for (int q = 0; q < Q; ++q) d[q * 64] = g[q];
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void *s, const void *g, unsigned bytes,
                                          unsigned long long *b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(s)), "l"(g), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_store(void *g, const void *s, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                 "r"(smem_u32(s)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int S>
__global__ void __launch_bounds__(32) bulk_rw(const double *__restrict__ src,
                                              double *__restrict__ dst, long long t_n) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long full[S];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long stride = gridDim.x;
    long long first = blockIdx.x;
    // prologue: S loads in flight
    int issued = 0;
    for (int s = 0; s < S; ++s) {
        const long long t = first + s * stride;
        if (t >= t_n) break;
        mbar_expect_tx(&full[s], TILE_BYTES);
        bulk_load(smem + s * TILE_BYTES, src + t * TILE, TILE_BYTES, &full[s]);
        ++issued;
    }
    long long i = 0;
    for (long long t = first; t < t_n; t += stride, ++i) {
        const int s = (int)(i % S);
        mbar_wait(&full[s], (unsigned)((i / S) & 1));
        bulk_store(dst + t * TILE, smem + s * TILE_BYTES, TILE_BYTES);
        // refill the stage of the previous tile once its store has read it
        if (i >= 1) {
            const long long nt = t + (S - 1) * stride;
            const int ps = (int)((i - 1) % S);
            if (nt < t_n) {
                bulk_wait_read<1>();
                mbar_expect_tx(&full[ps], TILE_BYTES);
                bulk_load(smem + ps * TILE_BYTES, src + nt * TILE, TILE_BYTES, &full[ps]);
            }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float best_ms(F launch, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r > 0 && ms < best) best = ms;   // r = 0 is the warm-up
    }
    return best;
}

template <int S>
void run_bulk(const double *src, double *dst, long long t_n, int reps, double bytes, int sms) {
    auto k = bulk_rw<S>;
    const int sm_bytes = S * TILE_BYTES;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, sm_bytes));
    const unsigned grid = (unsigned)(per_sm * sms);
    const float ms = best_ms([&] { k<<<grid, 32, sm_bytes>>>(src, dst, t_n); }, reps);
    CK(cudaGetLastError());
    printf("{\"kernel\": \"bulk_rw\", \"stages\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, "
           "\"gbs\": %.1f}\n", S, per_sm, ms, bytes / ms / 1e6);
}

int main(int argc, char **argv) {
    const long long t_n = argc > 1 ? atoll(argv[1]) : 262144;
    const int reps = argc > 2 ? atoi(argv[2]) : 21;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t n = (size_t)t_n * TILE;
    double *a, *b;
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8));
    CK(cudaMemset(a, 0, n * 8));
    CK(cudaMemset(b, 0, n * 8));
    const double bytes = 2.0 * n * 8;
    float ms = best_ms([&] { ldg_rw<<<(unsigned)((t_n + 1) / 2), 128>>>(a, b, t_n); }, reps);
    CK(cudaGetLastError());
    printf("{\"kernel\": \"ldg_rw\", \"ms\": %.4f, \"gbs\": %.1f}\n", ms, bytes / ms / 1e6);
    run_bulk<2>(a, b, t_n, reps, bytes, sms);
    run_bulk<4>(a, b, t_n, reps, bytes, sms);
    run_bulk<8>(a, b, t_n, reps, bytes, sms);
    run_bulk<12>(a, b, t_n, reps, bytes, sms);
    ms = best_ms([&] { CK(cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice)); }, reps);
    printf("{\"kernel\": \"memcpy\", \"ms\": %.4f, \"gbs\": %.1f}\n", ms, bytes / ms / 1e6);
    // correctness of the last bulk run: b == a (both zero-filled then a
    // patterned): fill a with a pattern and re-run one bulk copy
    double *h = (double *)malloc(TILE * 8 * 4);
    for (int i = 0; i < TILE * 4; ++i) h[i] = i * 0.5 + 1;
    CK(cudaMemcpy(a + (t_n - 4) * TILE, h, TILE * 8 * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(b, 0, n * 8));
    run_bulk<4>(a, b, t_n, 2, bytes, sms);
    double *g = (double *)malloc(TILE * 8 * 4);
    CK(cudaMemcpy(g, b + (t_n - 4) * TILE, TILE * 8 * 4, cudaMemcpyDeviceToHost));
    printf("{\"check\": %s}\n", memcmp(g, h, TILE * 8 * 4) == 0 ? "true" : "false");
    return 0;
}
