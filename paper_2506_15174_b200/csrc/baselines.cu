// baselines.cu -- BENCH ONLY (libescs_bench.so): the library baselines the
// paper compares against (§4.1): cuSPARSE CSR SpMM and cuBLAS dense
// SGEMM (fp32; optional TF32 tensor-core "cuBlas Tensor Core" context column).
// Not on the product path; escs_* never calls into this library.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusparse.h>

#include <cstdint>
#include <cstdlib>

struct BlSparse {
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnMatDescr_t B = nullptr, C = nullptr;
    void* buf = nullptr;
    cusparseSpMMAlg_t alg = CUSPARSE_SPMM_ALG_DEFAULT;
};

// Gather ceiling (bench roofline): warps gather pseudo-random 512-byte rows
// (bCols 128, fp32; row = fmix32(i) mod k, so repeats are spread like C5's
// uniform columns and L1 reuse stays at its random-access level) of an
// L2-resident B with no index loads, no values and no FMAs -- the most B-row bytes per second the SM memory pipeline delivers
// to registers for this access pattern.  L lanes per row, 16 B per lane per
// load instruction (interleaved), U rows in flight per sub-warp.
template <int L, int U>
__global__ void __launch_bounds__(256) gather_peak_kernel(const float4* __restrict__ B, int k,
                                                          long long rows_per_warp,
                                                          float* __restrict__ sink) {
    constexpr int F4 = 32 / L, S = 32 / L;   // float4 per lane per row; rows per instruction
    const int lane = threadIdx.x & 31, sub = lane / L, lj = lane % L;
    const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (long long i = 0; i < rows_per_warp; i += S * U) {
        float4 b[U][F4];
#pragma unroll
        for (int u = 0; u < U; u++) {
            unsigned x = (unsigned)(w * rows_per_warp + i + u * S + sub);
            x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16;   // fmix32
            const unsigned r = x % (unsigned)k;
#pragma unroll
            for (int v = 0; v < F4; v++) b[u][v] = __ldg(B + (size_t)r * 32 + v * L + lj);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
            for (int v = 0; v < F4; v++) {
                acc.x += b[u][v].x; acc.y += b[u][v].y; acc.z += b[u][v].z; acc.w += b[u][v].w;
            }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[threadIdx.x] = acc.x;   // keep the loads live
}

extern "C" {

// One launch of the gather ceiling kernel: `variant` 0..5 picks (L, U) in
// {32,16,8} x {4,8}; grid = ctas x 256 threads; rows_per_warp rows each.
int bl_gather_peak(const float* B, int k, int variant, int ctas, long long rows_per_warp,
                   float* sink, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const float4* B4 = reinterpret_cast<const float4*>(B);
    switch (variant) {
        case 0: gather_peak_kernel<32, 4><<<ctas, 256, 0, st>>>(B4, k, rows_per_warp, sink); break;
        case 1: gather_peak_kernel<32, 8><<<ctas, 256, 0, st>>>(B4, k, rows_per_warp, sink); break;
        case 2: gather_peak_kernel<16, 4><<<ctas, 256, 0, st>>>(B4, k, rows_per_warp, sink); break;
        case 3: gather_peak_kernel<16, 8><<<ctas, 256, 0, st>>>(B4, k, rows_per_warp, sink); break;
        case 4: gather_peak_kernel<8, 4><<<ctas, 256, 0, st>>>(B4, k, rows_per_warp, sink); break;
        case 5: gather_peak_kernel<8, 8><<<ctas, 256, 0, st>>>(B4, k, rows_per_warp, sink); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}


// alg: 0 = DEFAULT, 1 = CSR_ALG1, 2 = CSR_ALG2, 3 = CSR_ALG3.  Row-major B/C.
// Returns NULL if this algorithm rejects the configuration.
void* bl_cusparse_create(int m, int k, int nnz, int n, const int* rowptr, const int* colidx,
                         const float* vals, const float* B, float* C, int alg, void* stream) {
    BlSparse* s = new BlSparse();
    static const cusparseSpMMAlg_t algs[4] = {CUSPARSE_SPMM_ALG_DEFAULT, CUSPARSE_SPMM_CSR_ALG1,
                                              CUSPARSE_SPMM_CSR_ALG2, CUSPARSE_SPMM_CSR_ALG3};
    s->alg = algs[alg & 3];
    float one = 1.f, zero = 0.f;
    size_t bytes = 0;
    bool ok = cusparseCreate(&s->h) == CUSPARSE_STATUS_SUCCESS &&
              cusparseSetStream(s->h, (cudaStream_t)stream) == CUSPARSE_STATUS_SUCCESS &&
              cusparseCreateCsr(&s->A, m, k, nnz, (void*)rowptr, (void*)colidx, (void*)vals,
                                CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO,
                                CUDA_R_32F) == CUSPARSE_STATUS_SUCCESS &&
              cusparseCreateDnMat(&s->B, k, n, n, (void*)B, CUDA_R_32F, CUSPARSE_ORDER_ROW) ==
                  CUSPARSE_STATUS_SUCCESS &&
              cusparseCreateDnMat(&s->C, m, n, n, (void*)C, CUDA_R_32F, CUSPARSE_ORDER_ROW) ==
                  CUSPARSE_STATUS_SUCCESS &&
              cusparseSpMM_bufferSize(s->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                      CUSPARSE_OPERATION_NON_TRANSPOSE, &one, s->A, s->B, &zero,
                                      s->C, CUDA_R_32F, s->alg, &bytes) == CUSPARSE_STATUS_SUCCESS;
    if (ok && bytes) ok = cudaMalloc(&s->buf, bytes) == cudaSuccess;
    if (ok && (s->alg == CUSPARSE_SPMM_CSR_ALG3 || s->alg == CUSPARSE_SPMM_CSR_ALG2))
        ok = cusparseSpMM_preprocess(s->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                     CUSPARSE_OPERATION_NON_TRANSPOSE, &one, s->A, s->B, &zero,
                                     s->C, CUDA_R_32F, s->alg, s->buf) == CUSPARSE_STATUS_SUCCESS;
    if (ok)
        ok = cusparseSpMM(s->h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE,
                          &one, s->A, s->B, &zero, s->C, CUDA_R_32F, s->alg,
                          s->buf) == CUSPARSE_STATUS_SUCCESS;
    if (ok) ok = cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess;
    if (!ok) {
        if (s->buf) cudaFree(s->buf);
        if (s->A) cusparseDestroySpMat(s->A);
        if (s->B) cusparseDestroyDnMat(s->B);
        if (s->C) cusparseDestroyDnMat(s->C);
        if (s->h) cusparseDestroy(s->h);
        delete s;
        cudaGetLastError();
        return nullptr;
    }
    return s;
}

int bl_cusparse_run(void* hs, void* stream) {
    BlSparse* s = (BlSparse*)hs;
    float one = 1.f, zero = 0.f;
    cusparseSetStream(s->h, (cudaStream_t)stream);
    return (int)cusparseSpMM(s->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                             CUSPARSE_OPERATION_NON_TRANSPOSE, &one, s->A, s->B, &zero, s->C,
                             CUDA_R_32F, s->alg, s->buf);
}

void bl_cusparse_destroy(void* hs) {
    BlSparse* s = (BlSparse*)hs;
    if (!s) return;
    if (s->buf) cudaFree(s->buf);
    cusparseDestroySpMat(s->A);
    cusparseDestroyDnMat(s->B);
    cusparseDestroyDnMat(s->C);
    cusparseDestroy(s->h);
    delete s;
}

void* bl_cublas_create(void) {
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    // fixed workspace so that calls are CUDA-graph capturable
    void* ws = nullptr;
    const size_t bytes = 64u << 20;
    if (cudaMalloc(&ws, bytes) == cudaSuccess) cublasSetWorkspace(h, ws, bytes);
    cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);
    return h;
}

// Row-major C[m x n] = A[m x k] * B[k x n] via column-major C^T = B^T A^T.
int bl_cublas_sgemm(void* hv, int m, int n, int k, const float* A, const float* B, float* C,
                    int tf32, void* stream) {
    cublasHandle_t h = (cublasHandle_t)hv;
    cublasSetStream(h, (cudaStream_t)stream);
    const float one = 1.f, zero = 0.f;
    cublasComputeType_t ct = tf32 ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F;
    return (int)cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &one, B, CUDA_R_32F, n, A,
                             CUDA_R_32F, k, &zero, C, CUDA_R_32F, n, ct, CUBLAS_GEMM_DEFAULT);
}

void bl_cublas_destroy(void* hv) {
    if (hv) cublasDestroy((cublasHandle_t)hv);
}

}  // extern "C"
