// FP64 latency/throughput microbenchmark (single dependent chain per thread).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_fma(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.999999999, 1e-12);
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_exp(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = exp(x) * 1e-3;
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_log(double* out, double a, int n, long long* cyc) {
    double x = a + 2.0 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = log(x) + 2.5;
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_log1p(double* out, double a, int n, long long* cyc) {
    double x = a + 0.3 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = log1p(x) + 0.1;
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_div(double* out, double a, int n, long long* cyc) {
    double x = a + 1.5 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(double* out, int n, long long* cyc) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) j = idx[j];
    long long t1 = clock64();
    out[threadIdx.x] = j; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_bar(double* out, int n, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <class K> void run(const char* name, K k, int threads, int n, double* d, long long* c) {
    long long h;
    k<<<1, threads>>>(d, 0.5, n, c);
    cudaDeviceSynchronize();
    k<<<1, threads>>>(d, 0.5, n, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-8s threads=%4d  %.1f cycles/op\n", name, threads, (double)h / n);
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 8 * 2048); cudaMalloc(&c, 8);
    for (int t : {32, 512}) {
        run("dfma", k_fma, t, 4096, d, c);
        run("exp", k_exp, t, 1024, d, c);
        run("log", k_log, t, 1024, d, c);
        run("log1p", k_log1p, t, 1024, d, c);
        run("div", k_div, t, 1024, d, c);
    }
    long long h;
    for (int t : {32, 512}) {
        k_lds<<<1, t>>>(d, 4096, c); cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("lds      threads=%4d  %.1f cycles/op\n", t, (double)h / 4096);
        k_bar<<<1, t>>>(d, 4096, c); cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("barrier  threads=%4d  %.1f cycles/op\n", t, (double)h / 4096);
    }
    return 0;
}
