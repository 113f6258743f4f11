// Serial fold microbenchmark (development tool): one thread folds n shared-
// memory doubles in order (the chain-solve pattern), several code shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/fb tools/fold_bench.cu
#include <cstdio>

template <int V>
__global__ void fold(const double* g, double* out, int n, long long* cyc) {
    __shared__ double v[2048];
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = g[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    double acc = -0.0;
    if (V == 0) {  // plain
        for (int k = 0; k < n; ++k) { acc = v[k] + acc; v[k] = acc; }
    } else if (V == 1) {  // 8-batch double buffer, in place
        double cur[8], nxt[8];
        for (int u = 0; u < 8; ++u) cur[u] = u < n ? v[u] : 0.0;
        for (int k0 = 0; k0 < n; k0 += 8) {
            for (int u = 0; u < 8; ++u) nxt[u] = k0 + 8 + u < n ? v[k0 + 8 + u] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < n) { acc = cur[u] + acc; v[k0 + u] = acc; }
#pragma unroll
            for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
        }
    } else if (V == 2) {  // 8-batch, no store
        double cur[8], nxt[8];
        for (int u = 0; u < 8; ++u) cur[u] = u < n ? v[u] : 0.0;
        for (int k0 = 0; k0 < n; k0 += 8) {
            for (int u = 0; u < 8; ++u) nxt[u] = k0 + 8 + u < n ? v[k0 + 8 + u] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < n) acc = cur[u] + acc;
#pragma unroll
            for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
        }
    } else if (V == 3) {  // full batches without predicates, 16-wide
        int k0 = 0;
        for (; k0 + 16 <= n; k0 += 16) {
            double t[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) t[u] = v[k0 + u];
#pragma unroll
            for (int u = 0; u < 16; ++u) { acc = t[u] + acc; v[k0 + u] = acc; }
        }
        for (; k0 < n; ++k0) { acc = v[k0] + acc; v[k0] = acc; }
    }
    long long t1 = clock64();
    out[0] = acc + v[n - 1];
    cyc[0] = t1 - t0;
}

int main() {
    const int n = 1081;
    double* g; double* out; long long* cyc;
    cudaMalloc(&g, 8 * 2048); cudaMalloc(&out, 8); cudaMallocManaged(&cyc, 8);
    cudaMemset(g, 0, 8 * 2048);
    const char* names[] = {"plain", "batch8 inplace", "batch8 nostore", "batch16 nopred"};
    for (int v = 0; v < 4; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) fold<0><<<1, 256>>>(g, out, n, cyc);
            if (v == 1) fold<1><<<1, 256>>>(g, out, n, cyc);
            if (v == 2) fold<2><<<1, 256>>>(g, out, n, cyc);
            if (v == 3) fold<3><<<1, 256>>>(g, out, n, cyc);
            cudaDeviceSynchronize();
        }
        printf("%-18s %8.2f cycles/element\n", names[v], double(*cyc) / n);
    }
    return 0;
}
