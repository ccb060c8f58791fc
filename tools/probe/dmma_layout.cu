// Verify the mma.sync.m8n8k4 f64 fragment layout assumed by fast_kernels.cuh:
//   A (8x4): a0 = A[lane>>2][lane&3];  B (4x8): b0 = B[lane&3][lane>>2]
//   C (8x8): c{0,1} = C[lane>>2][2*(lane&3) + {0,1}]
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* C) {
    const int lane = threadIdx.x;
    double a = A[(lane >> 2) * 4 + (lane & 3)];
    double b = B[(lane & 3) * 8 + (lane >> 2)];
    double c0 = 0, c1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    C[(lane >> 2) * 8 + 2 * (lane & 3)] = c0;
    C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;
}

int main() {
    double hA[32], hB[32], hC[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i; hB[i] = 0.5 * i - 3.0; }
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int t = 0; t < 4; ++t) s += hA[r * 4 + t] * hB[t * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *A, *B, *C;
    cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
    cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(A, B, C);
    cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 64; ++i) if (hC[i] != ref[i]) ++bad;
    std::printf("m8n8k4 f64 layout check: %d mismatches (%s)\n", bad, bad ? "LAYOUT WRONG" : "ok");
    return bad != 0;
}
