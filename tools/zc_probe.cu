// zc_probe.cu — host<->device transfer microbenchmark for the host-buffer
// pair (config-3 vector: 2,231,184 doubles per direction).
//
//   ce_chunks  : cudaMemcpyAsync of the vector in G chunks on one stream
//                (H2D alone, D2H alone, both on two streams), direct enqueue
//   kernel     : an SM copy kernel reading pinned host memory (UVA) into HBM,
//                or writing HBM into pinned host memory, with C CTAs
//   both_kernel: H2D and D2H kernels side by side
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/zc_probe tools/zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e_));                   \
            return 1;                                                              \
        }                                                                          \
    } while (0)

// grid-stride 16-byte copy, U vectors in flight per thread
template <int U>
__global__ void __launch_bounds__(256) k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
    const size_t N = 2231184, B = N * 8;
    double *h_in, *h_out, *d_in, *d_out;
    CK(cudaHostAlloc(&h_in, B, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h_out, B, cudaHostAllocMapped));
    CK(cudaMalloc(&d_in, B));
    CK(cudaMalloc(&d_out, B));
    for (size_t i = 0; i < N; ++i) h_in[i] = double(i);
    CK(cudaMemset(d_out, 0, B));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int reps = 20;
    auto timeit = [&](auto&& body) {
        body();
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        for (int r = 0; r < reps; ++r) body();
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        return double(ms) * 1e3 / reps;  // us
    };
    // the legacy default stream orders s1 / s2 work between timing events:
    // join them into stream 0 explicitly
    cudaEvent_t j1, j2;
    CK(cudaEventCreateWithFlags(&j1, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&j2, cudaEventDisableTiming));
    auto fork = [&] {
        cudaEventRecord(j1, 0);
        cudaStreamWaitEvent(s1, j1, 0);
        cudaStreamWaitEvent(s2, j1, 0);
    };
    auto join = [&] {
        cudaEventRecord(j1, s1);
        cudaEventRecord(j2, s2);
        cudaStreamWaitEvent(0, j1, 0);
        cudaStreamWaitEvent(0, j2, 0);
    };
    for (int G : {1, 2, 4, 8, 16, 48}) {
        auto chunks = [&](bool h2d, bool d2h) {
            return timeit([&] {
                fork();
                for (int g = 0; g < G; ++g) {
                    const size_t lo = N * g / G, hi = N * (g + 1) / G;
                    if (h2d) cudaMemcpyAsync(d_in + lo, h_in + lo, 8 * (hi - lo), cudaMemcpyHostToDevice, s1);
                    if (d2h) cudaMemcpyAsync(h_out + lo, d_out + lo, 8 * (hi - lo), cudaMemcpyDeviceToHost, s2);
                }
                join();
            });
        };
        const double th = chunks(true, false), td = chunks(false, true), tb = chunks(true, true);
        std::printf("{\"ce_chunks\": %d, \"h2d_gbs\": %.1f, \"d2h_gbs\": %.1f, \"both_total_gbs\": %.1f, "
                    "\"both_us\": %.1f}\n",
                    G, B / th / 1e3, B / td / 1e3, 2 * B / tb / 1e3, tb);
    }
    const size_t n16 = B / 16;
    for (int C : {8, 16, 32, 64, 148, 296}) {
        const double th = timeit([&] {
            k_copy<4><<<C, 256>>>(reinterpret_cast<const uint4*>(h_in), reinterpret_cast<uint4*>(d_in), n16);
        });
        const double td = timeit([&] {
            k_copy<4><<<C, 256>>>(reinterpret_cast<const uint4*>(d_out), reinterpret_cast<uint4*>(h_out), n16);
        });
        const double tb = timeit([&] {
            fork();
            k_copy<4><<<C, 256, 0, s1>>>(reinterpret_cast<const uint4*>(h_in), reinterpret_cast<uint4*>(d_in), n16);
            k_copy<4><<<C, 256, 0, s2>>>(reinterpret_cast<const uint4*>(d_out), reinterpret_cast<uint4*>(h_out), n16);
            join();
        });
        std::printf("{\"kernel_ctas\": %d, \"h2d_gbs\": %.1f, \"d2h_gbs\": %.1f, \"both_total_gbs\": %.1f, "
                    "\"both_us\": %.1f}\n",
                    C, B / th / 1e3, B / td / 1e3, 2 * B / tb / 1e3, tb);
    }
    // CE H2D beside a kernel D2H, and the reverse
    for (int C : {32, 64}) {
        const double t1 = timeit([&] {
            fork();
            cudaMemcpyAsync(d_in, h_in, B, cudaMemcpyHostToDevice, s1);
            k_copy<4><<<C, 256, 0, s2>>>(reinterpret_cast<const uint4*>(d_out), reinterpret_cast<uint4*>(h_out), n16);
            join();
        });
        const double t2 = timeit([&] {
            fork();
            k_copy<4><<<C, 256, 0, s1>>>(reinterpret_cast<const uint4*>(h_in), reinterpret_cast<uint4*>(d_in), n16);
            cudaMemcpyAsync(h_out, d_out, B, cudaMemcpyDeviceToHost, s2);
            join();
        });
        std::printf("{\"mixed_ctas\": %d, \"ce_h2d_kernel_d2h_total_gbs\": %.1f, \"kernel_h2d_ce_d2h_total_gbs\": %.1f}\n",
                    C, 2 * B / t1 / 1e3, 2 * B / t2 / 1e3);
    }
    // the pair pipeline's shape: G chunks, CE H2D on s1, D2H chunk g after
    // H2D chunk g on s2 (CE copy or a C-CTA copy kernel)
    cudaEvent_t ev[64];
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int G : {1, 2, 4, 8}) {
        auto pipe = [&](int C) {
            return timeit([&] {
                fork();
                for (int g = 0; g < G; ++g) {
                    const size_t lo = N * g / G, hi = N * (g + 1) / G;
                    cudaMemcpyAsync(d_in + lo, h_in + lo, 8 * (hi - lo), cudaMemcpyHostToDevice, s1);
                    cudaEventRecord(ev[g], s1);
                    cudaStreamWaitEvent(s2, ev[g], 0);
                    if (C == 0)
                        cudaMemcpyAsync(h_out + lo, d_out + lo, 8 * (hi - lo), cudaMemcpyDeviceToHost, s2);
                    else
                        k_copy<4><<<C, 256, 0, s2>>>(reinterpret_cast<const uint4*>(d_out + lo),
                                                     reinterpret_cast<uint4*>(h_out + lo), (hi - lo) / 2);
                }
                join();
            });
        };
        std::printf("{\"pipe_chunks\": %d, \"ce_ce_us\": %.1f, \"ce_k16_us\": %.1f, \"ce_k32_us\": %.1f, "
                    "\"ce_k64_us\": %.1f}\n", G, pipe(0), pipe(16), pipe(32), pipe(64));
    }
    // the queue's shape without kernels: pairs i = 0..Q-1, each y then x in on
    // s1 and both out on s2 (out after in), host buffers cycling over R sets
    for (int R : {1, 4}) {
        double *hi[4][2], *ho[4][2], *dI[2][2], *dO[2][2];
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < 2; ++d) {
                CK(cudaHostAlloc(&hi[r][d], B, 0));
                CK(cudaHostAlloc(&ho[r][d], B, 0));
            }
        for (int k = 0; k < 2; ++k)
            for (int d = 0; d < 2; ++d) {
                CK(cudaMalloc(&dI[k][d], B));
                CK(cudaMalloc(&dO[k][d], B));
            }
        const int Q = 20;
        const double t = timeit([&] {
            fork();
            for (int i = 0; i < Q; ++i)
                for (int d : {1, 0}) {
                    const int k = i & 1, r = i % R;
                    cudaMemcpyAsync(dI[k][d], hi[r][d], B, cudaMemcpyHostToDevice, s1);
                    cudaEventRecord(ev[2 * k + d], s1);
                    cudaStreamWaitEvent(s2, ev[2 * k + d], 0);
                    cudaMemcpyAsync(ho[r][d], dO[k][d], B, cudaMemcpyDeviceToHost, s2);
                }
            join();
        });
        std::printf("{\"queue_copies_ring\": %d, \"us_per_pair\": %.1f, \"pairs_per_s\": %.1f}\n", R, t / Q,
                    1e6 * Q / t);
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < 2; ++d) {
                cudaFreeHost(hi[r][d]);
                cudaFreeHost(ho[r][d]);
            }
        for (int k = 0; k < 2; ++k)
            for (int d = 0; d < 2; ++d) {
                cudaFree(dI[k][d]);
                cudaFree(dO[k][d]);
            }
    }
    // correctness of the kernel copies
    CK(cudaDeviceSynchronize());
    double chk = 0;
    CK(cudaMemcpy(&chk, d_in + N - 1, 8, cudaMemcpyDeviceToHost));
    std::printf("{\"check\": %s}\n", chk == double(N - 1) ? "true" : "false");
    return 0;
}
