// Dependent-chain latency microbenchmark (development tool): cycles per
// operation of serial DADD / DMUL / DFMA / FADD / IADD chains and of a
// serial smem-load + DADD chain, one thread.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/lat tools/microbench_latency.cu
#include <cstdio>

template <int OP>
__global__ void chain(double* out, double a, double b, int n, long long* cyc) {
    double x = a, y = b;
    float xf = float(a), yf = float(b);
    long long xi = (long long)a, yi = 3;
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-9 * i;
    __syncthreads();
    long long t0 = clock64();
    if (OP == 0)
        for (int i = 0; i < n; ++i) x = x + y;
    if (OP == 1)
        for (int i = 0; i < n; ++i) x = x * y;
    if (OP == 2)
        for (int i = 0; i < n; ++i) x = fma(x, y, b);
    if (OP == 3)
        for (int i = 0; i < n; ++i) xf = xf + yf;
    if (OP == 4)
        for (int i = 0; i < n; ++i) xi = xi + yi;
    if (OP == 5)
        for (int i = 0; i < n; ++i) x = sm[i & 1023] + x;
    if (OP == 6)  // recurrence with a compare/select like the chain solve
        for (int i = 0; i < n; ++i) x = (x != 0.0) ? sm[i & 1023] - (-1.0) * x : sm[i & 1023];
    if (OP == 7)  // IEEE fp64 division (regret matching r / sumPos)
        for (int i = 0; i < n; ++i) x = y / x;
    if (OP == 8)  // global load chain (L2 latency)
        for (int i = 0; i < n; ++i) x = out[(long long)(x) & 1] + 1e-300;
    long long t1 = clock64();
    out[0] = x + xf + double(xi);
    cyc[0] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMallocManaged(&cyc, 8);
    const char* names[] = {"DADD", "DMUL", "DFMA", "FADD", "IADD64", "LDS+DADD", "LDS+DMUL+DADD+select", "DDIV", "LDG chain"};
    const int n = 100000;
    for (int op = 0; op < 9; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: chain<0><<<1, 1>>>(out, 1.0, 1e-9, n, cyc); break;
                case 1: chain<1><<<1, 1>>>(out, 1.0, 1.0000001, n, cyc); break;
                case 2: chain<2><<<1, 1>>>(out, 1.0, 0.999999, n, cyc); break;
                case 3: chain<3><<<1, 1>>>(out, 1.0, 1e-7, n, cyc); break;
                case 4: chain<4><<<1, 1>>>(out, 1.0, 3, n, cyc); break;
                case 5: chain<5><<<1, 1>>>(out, 1.0, 1e-9, n, cyc); break;
                case 6: chain<6><<<1, 1>>>(out, 1.0, 1e-9, n, cyc); break;
                case 7: chain<7><<<1, 1>>>(out, 1.5, 1.25, n, cyc); break;
                case 8: chain<8><<<1, 1>>>(out, 0.0, 1.0, n, cyc); break;
            }
            cudaDeviceSynchronize();
        }
        printf("%-22s %7.2f cycles/op\n", names[op], double(*cyc) / n);
    }
    return 0;
}
