// Bisect TMA issue: argv[1] = variant
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ void body(const CUtensorMap* tm, double* out, int x) {
    extern __shared__ __align__(1024) unsigned char sm[];
    double* buf = (double*)sm;
    uint64_t* bar = (uint64_t*)(sm + 8192);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(32 * 18 * 8) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(buf)), "l"((uint64_t)tm), "r"(x), "r"(0), "r"(0), "r"(su32(bar)) : "memory");
    }
    uint32_t ok = 0;
    for (int it = 0; it < (1 << 24) && !ok; ++it)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(bar)), "r"(0) : "memory");
    if (!ok) { if (threadIdx.x == 0) printf("timeout\n"); return; }
    for (int i = threadIdx.x; i < 64; i += 32) out[i] = buf[i];
}
struct Maps { CUtensorMap a, b; };
__global__ void k_struct(const __grid_constant__ Maps m, double* out, int x) { body(&m.a, out, x); }
__global__ void k_direct(const __grid_constant__ CUtensorMap m, double* out, int x) { body(&m, out, x); }
__global__ void k_global(const CUtensorMap* m, double* out, int x) { body(m, out, x); }
int main(int argc, char** argv) {
    int v = atoi(argv[1]);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    int nx = 40, er = 36; size_t ep = 40, epl = 1440 + 32;
    double* S; cudaMalloc(&S, 18 * epl * 8);
    double* h = (double*)malloc(18 * epl * 8); for (size_t i = 0; i < 18 * epl; ++i) h[i] = i; cudaMemcpy(S, h, 18 * epl * 8, cudaMemcpyHostToDevice);
    Maps m;
    int rank = (v >= 6) ? 2 : 3;
    cuuint64_t dS[3] = {(cuuint64_t)nx, (cuuint64_t)er, 18}, sS[2] = {ep * 8, epl * 8};
    cuuint32_t bS[3] = {32, 1, 18}, es[3] = {1, 1, 1};
    CUresult r = fn(&m.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, S, dS, sS, bS, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    double* out; cudaMalloc(&out, 64 * 8);
    CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m.a, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    int x = (argc > 2) ? atoi(argv[2]) : ((v % 2) ? -1 : 0);
    const char* names[] = {"struct x=0", "struct x=-1", "direct x=0", "direct x=-1", "global x=0", "global x=-1"};
    if (v < 2) k_struct<<<1, 32, 8192 + 64>>>(m, out, x);
    else if (v < 4) k_direct<<<1, 32, 8192 + 64>>>(m.a, out, x);
    else k_global<<<1, 32, 8192 + 64>>>(gm, out, x);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[64] = {0}; if (!e) cudaMemcpy(ho, out, 64 * 8, cudaMemcpyDeviceToHost);
    printf("%-14s encode=%d: %s  first %g %g [32]=%g\n", names[v], (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[32]);
    return 0;
}
