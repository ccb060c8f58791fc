// chain_kernel with the products pinned ahead of the next batch's loads
// (PIN=1) vs the production schedule (PIN=0): static SASS + timing.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o chain_pin_probe chain_pin_probe.cu
#include <cstdio>
#include <vector>
#include "exact_kernels.cuh"
using namespace coopcg_gpu;

template <int P, int T, int S, int PIN>
__global__ void __launch_bounds__(kChainThreads)
    chain_pin_kernel(const double* __restrict__ s0, const double* __restrict__ s1,
                 const double* __restrict__ s2, int nsrc, int n,
                 const ChainDesc* __restrict__ descs, int nchains, double* __restrict__ out,
                 const int* __restrict__ stop, int kzero) {
    pdl_wait();
    constexpr int U = kChainU;
    static_assert(T % (2 * U) == 0, "tile rows must be an even number of batches");
    constexpr int NBT = T / U;  // batches per tile
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* buf = reinterpret_cast<double*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(buf + static_cast<size_t>(S) * nsrc * T * P);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntiles = (n + T - 1) / T;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kChainWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int rows = min(T, n - t * T);
                const uint32_t bytes = static_cast<uint32_t>(rows) * P * 8u;
                mbar_arrive_expect_tx(&full[s], bytes * nsrc);
                double* dst = buf + static_cast<size_t>(s) * nsrc * T * P;
                bulk_g2s(dst, s0 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (nsrc > 1) bulk_g2s(dst + T * P, s1 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (nsrc > 2) bulk_g2s(dst + 2 * T * P, s2 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int c = blockIdx.x * (kChainWarps * 32) + (tid - 32);
    ChainDesc d{0, 0, 0, 0, 0, 0, 0};
    if (c < nchains) d = descs[c];
    const int xoff = d.sx * T * P + d.a;
    const int yoff = d.sy * T * P + d.b;
    const int nb = (n + U - 1) / U;  // batches; all full except possibly the last
    auto tile_wait = [&](int t) {
        if (t < ntiles) mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
    };
    // operands of batch j (may lie past the last tile: stale ring data that
    // is multiplied but never added)
    auto batch_base = [&](int j) -> const double* {
        return buf + static_cast<size_t>((j / NBT) % S) * nsrc * T * P + (j % NBT) * U * P;
    };
    double acc = 0.0;
    // pr: products of the batch being added; operands of batch j live in the
    // even (xe/ye) or odd (xo/yo) register set by the parity of j, so a step
    // reads one set and loads into the other (no WAR hazard to serialise the
    // loads behind the DMULs)
    double pr[U], xe[U], ye[U], xo[U], yo[U];
    // add batch b, form batch b+1 (from xr/yr), load batch b+2 (into xw/yw)
    auto step = [&](int b, const double (&xr)[U], const double (&yr)[U], double (&xw)[U], double (&yw)[U]) {
        const double* b2 = batch_base(b + 2);
        if (PIN == 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc = __dadd_rn(acc, pr[u]);
                pr[u] = __dmul_rn(xr[u], yr[u]);
                xw[u] = b2[xoff + u * P];
                yw[u] = b2[yoff + u * P];
            }
        } else if (PIN == 1) {
            // products of batch b+1 first; the loads of batch b+2 take their
            // address through (product bits & kzero) == 0, so ptxas must keep
            // every DMUL ahead of them (no sinking to the consuming DADD)
            unsigned z = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc = __dadd_rn(acc, pr[u]);
                pr[u] = __dmul_rn(xr[u], yr[u]);
                z |= static_cast<unsigned>(__double2loint(pr[u]));
            }
            z &= static_cast<unsigned>(kzero);
            const double* b2z = b2 + z;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                xw[u] = b2z[xoff + u * P];
                yw[u] = b2z[yoff + u * P];
            }
        } else if (PIN == 3) {
            // the add of (batch b, u) takes its operand through the product of
            // (batch b+1, u): lo | (next.lo & kzero) == lo, so the DMUL of the
            // next batch must be issued before this DADD (it cannot sink to its
            // own consumer); the merge waits only where the DADD waits anyway
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double nx = __dmul_rn(xr[u], yr[u]);
                const double cur = __hiloint2double(__double2hiint(pr[u]),
                                                    __double2loint(pr[u]) | (__double2loint(nx) & kzero));
                acc = __dadd_rn(acc, cur);
                pr[u] = nx;
                xw[u] = b2[xoff + u * P];
                yw[u] = b2[yoff + u * P];
            }
        } else {
            // per step: load u of batch b+2 is addressed through product u
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc = __dadd_rn(acc, pr[u]);
                pr[u] = __dmul_rn(xr[u], yr[u]);
                const unsigned z = static_cast<unsigned>(__double2loint(pr[u])) & static_cast<unsigned>(kzero);
                const double* b2z = b2 + z;
                xw[u] = b2z[xoff + u * P];
                yw[u] = b2z[yoff + u * P];
            }
        }
    };
    tile_wait(0);
    {
        const double* b0 = batch_base(0);
        const double* b1 = batch_base(1);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pr[u] = __dmul_rn(b0[xoff + u * P], b0[yoff + u * P]);
            xo[u] = b1[xoff + u * P];
            yo[u] = b1[yoff + u * P];
        }
    }
    // One iteration per tile: tile t+1 is waited for first (the steps load up
    // to two batches ahead), the NBT steps run straight-line (one basic block
    // for ptxas to schedule), and tile t is released once its last batch has
    // been multiplied.
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
        tile_wait(t + 1);
        const int b0 = t * NBT;
        if ((t + 1) * T <= n) {
#pragma unroll
            for (int q = 0; q < NBT; q += 2) {
                step(b0 + q, xo, yo, xe, ye);
                step(b0 + q + 1, xe, ye, xo, yo);
            }
        } else {
            // partial last tile: the batches that hold rows, the last one masked
            for (int q = 0; q < NBT && b0 + q < nb; ++q) {
                const int b = b0 + q;
                if (b == nb - 1) {
                    const int rem = n - b * U;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u < rem) acc = __dadd_rn(acc, pr[u]);
                } else if (q & 1) {
                    step(b, xe, ye, xo, yo);
                } else {
                    step(b, xo, yo, xe, ye);
                }
            }
        }
        __syncwarp();
        mbar_arrive_lane0(&empty[t % S], lane);
    }
    if (c < nchains) out[d.out] = d.neg ? -acc : acc;
}


template <int P, int T, int S, int PIN>
float run(const double* s0, const double* s1, const double* s2, int n, const ChainDesc* d, int nch, double* out) {
    auto k = chain_pin_kernel<P, T, S, PIN>;
    size_t smem = chain_smem_bytes(P, T, S, 3);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<(nch + 63) / 64, kChainThreads, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k<<<(nch + 63) / 64, kChainThreads, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return ms / 10;
}

int main() {
    constexpr int P = 8;
    const int n = 16384, p = 8;
    double *s[3], *out;
    std::vector<double> h(n * P);
    for (int q = 0; q < 3; ++q) {
        cudaMalloc(&s[q], (size_t)n * P * 8);
        for (size_t e = 0; e < h.size(); ++e) h[e] = ((e * 2654435761ull + q * 97) % 1000003) / 1000003.0 - 0.45;
        cudaMemcpy(s[q], h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    }
    cudaMalloc(&out, 8192 * 8);
    std::vector<ChainDesc> hd;
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) hd.push_back(ChainDesc{0, (uint8_t)i, 1, (uint8_t)j, (uint16_t)(i * P + j), 0, 0});
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) hd.push_back(ChainDesc{2, (uint8_t)i, 0, (uint8_t)j, (uint16_t)(P * P + i * P + j), 1, 0});
    for (int i = 0; i < p; ++i) hd.push_back(ChainDesc{0, (uint8_t)i, 0, (uint8_t)i, (uint16_t)(2 * P * P + i), 0, 0});
    ChainDesc* d;
    cudaMalloc(&d, hd.size() * sizeof(ChainDesc));
    cudaMemcpy(d, hd.data(), hd.size() * sizeof(ChainDesc), cudaMemcpyHostToDevice);
    const int nch = (int)hd.size();
    std::vector<double> o0(nch), o1(nch);
    for (int w = 0; w < 2; ++w) {
        float t0 = run<8, 384, 3, 0>(s[0], s[1], s[2], n, d, nch, out);
        cudaMemcpy(o0.data(), out, nch * 8, cudaMemcpyDeviceToHost);
        float t1 = run<8, 384, 3, 1>(s[0], s[1], s[2], n, d, nch, out);
        cudaMemcpy(o1.data(), out, nch * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int c = 0; c < nch; ++c) bad += o0[c] != o1[c];
        float t2 = run<8, 384, 3, 3>(s[0], s[1], s[2], n, d, nch, out);
        cudaMemcpy(o1.data(), out, nch * 8, cudaMemcpyDeviceToHost);
        for (int c = 0; c < nch; ++c) bad += o0[c] != o1[c];
        float t3 = run<8, 512, 3, 3>(s[0], s[1], s[2], n, d, nch, out);
        std::printf("T=512 PIN=3: %.1f us\n", t3 * 1e3);
        std::printf("T=384 PIN=0: %.1f us   PIN=1: %.1f us   PIN=3: %.1f us   mismatches %d\n", t0 * 1e3, t1 * 1e3,
                    t2 * 1e3, bad);
    }
    return 0;
}
