// Standalone probe of the TMA load pattern used by k_subcycle_tma (debug aid).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap a, b; };
__global__ void probe(const __grid_constant__ Maps m, double* out, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    double* buf = (double*)sm;
    uint64_t* bar = (uint64_t*)(sm + 8192);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        uint32_t bytes = mode == 0 ? 32 * 18 * 8 : 66 * 3 * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(buf)), "l"((uint64_t)&m.a), "r"(-1), "r"(0), "r"(0), "r"(su32(bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"((uint64_t)&m.b), "r"(-2), "r"(0), "r"(su32(bar)) : "memory");
    }
    uint32_t ok = 0;
    for (int it = 0; it < (1 << 24) && !ok; ++it)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(bar)), "r"(0) : "memory");
    if (!ok) { if (threadIdx.x == 0) printf("timeout mode %d\n", mode); return; }
    for (int i = threadIdx.x; i < 64; i += 32) out[i] = buf[i];
}
int main() {
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    printf("entry %p q=%d\n", p, (int)q);
    int nx = 40, er = 36; size_t ep = 40, epl = 1440 + 32;
    double* S; cudaMalloc(&S, 18 * epl * 8);
    double* h = (double*)malloc(18 * epl * 8); for (size_t i = 0; i < 18 * epl; ++i) h[i] = i; cudaMemcpy(S, h, 18 * epl * 8, cudaMemcpyHostToDevice);
    Maps m;
    cuuint64_t dS[3] = {(cuuint64_t)nx, (cuuint64_t)er, 18}, sS[2] = {ep * 8, epl * 8};
    cuuint32_t bS[3] = {32, 1, 18}, es[3] = {1, 1, 1};
    CUresult r = fn(&m.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, S, dS, sS, bS, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode S: %d\n", (int)r);
    cuuint64_t dV[2] = {81, 73}, sV[1] = {96 * 8};
    cuuint32_t bV[2] = {66, 3};
    r = fn(&m.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, S, dV, sV, bV, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode V: %d\n", (int)r);
    double* out; cudaMalloc(&out, 64 * 8);
    for (int mode = 0; mode < 2; ++mode) {
        probe<<<1, 32, 8192 + 64>>>(m, out, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e) return 1;
        double ho[64]; cudaMemcpy(ho, out, 64 * 8, cudaMemcpyDeviceToHost);
        printf("  first: %g %g %g ... [32]=%g\n", ho[0], ho[1], ho[2], ho[32]);
    }
    return 0;
}
