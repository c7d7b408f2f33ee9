// tools/tc_selftest.cu -- development check of the tcgen05 building blocks in csrc/tc.cuh:
// D[128][N] = A[128][K] . W[K][N] with bf16x3 on the tensor cores vs an fp64 host GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2509_23043_b200/csrc \
//        tools/tc_selftest.cu -o /tmp/tc_selftest && /tmp/tc_selftest
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tc.cuh"

using namespace tapt_tc;

template <int N, int K>
__global__ void k_selftest(const float* A, const float* W, float* D) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* ah = sm;
    uint8_t* al = ah + 128 * K * 2;
    uint8_t* bh = al + 128 * K * 2;
    uint8_t* bl = bh + N * K * 2;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    // operands: A row r = tid; B row n = W[:, n]
    for (int k0 = 0; k0 < K; k0 += 8) {
        float x[8];
        for (int i = 0; i < 8; ++i) x[i] = A[tid * K + k0 + i];
        store_row8(ah, al, tid, k0, K, x);
    }
    for (int n = tid; n < N; n += 128)
        for (int k0 = 0; k0 < K; k0 += 8) {
            float x[8];
            for (int i = 0; i < 8; ++i) x[i] = W[(k0 + i) * N + n];
            store_row8(bh, bl, n, k0, K, x);
        }
    if (tid == 0) bar_init(&bar, 1);
    if (warp == 0) tmem_alloc(&tbase, 256);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t t0 = tbase;
    if (tid == 0) {
        mma_x3<N, K>(t0, ah, al, bh, bl);
        mma_commit(&bar);
    }
    bar_wait(&bar, 0);
    fence_after();
    for (int c = 0; c < N; c += 16) {
        float v[16];
        tmem_ld16(t0 + ((uint32_t)(32 * (warp & 3)) << 16) + c, v);
        for (int i = 0; i < 16; ++i) D[tid * N + c + i] = v[i];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_free(t0, 256);
}

template <int N, int K>
int run() {
    std::vector<float> A(128 * K), W(K * N), D(128 * N);
    srand(N * 7 + K);
    for (auto& x : A) x = (float)(rand() / (double)RAND_MAX * 2 - 1);
    for (auto& x : W) x = (float)(rand() / (double)RAND_MAX * 2 - 1) * 0.1f;
    float *dA, *dW, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dW, W.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)(2 * 128 * K + 2 * N * K) * 2;
    cudaFuncSetAttribute(k_selftest<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_selftest<N, K><<<1, 128, smem>>>(dA, dW, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)A[r * K + k] * W[k * N + n];
            maxerr = fmax(maxerr, fabs(ref - D[r * N + n]));
            maxref = fmax(maxref, fabs(ref));
        }
    printf("N=%d K=%d: max |err| %.3e (max |ref| %.3e) %s\n", N, K, maxerr, maxref, maxerr < 1e-5 * maxref ? "OK" : "FAIL");
    cudaFree(dA);
    cudaFree(dW);
    cudaFree(dD);
    return maxerr < 1e-5 * maxref ? 0 : 1;
}

int main() {
    int bad = 0;
    bad += run<192, 64>();
    bad += run<64, 64>();
    bad += run<128, 64>();
    bad += run<64, 128>();
    return bad;
}
