// D2H bandwidth into page-locked memory with 1 / 2 / 4 concurrent streams
// (the J / P level downloads of a C3 solve).  nvcc -O2 -o /tmp/d2h_bw tools/d2h_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

int main() {
    const size_t chunk = size_t(291) << 20, total = size_t(20) * chunk;
    char *d, *h;
    cudaMalloc(&d, chunk * 4);
    cudaMemset(d, 1, chunk * 4);
    cudaHostAlloc(reinterpret_cast<void**>(&h), total, cudaHostAllocDefault);
    for (size_t i = 0; i < total; i += 4096) h[i] = 0;
    cudaStream_t s[4];
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int ns : {1, 2, 4}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, 0);
            for (int i = 0; i < 20; ++i) {
                cudaStream_t q = s[i % ns];
                cudaStreamWaitEvent(q, a, 0);
                cudaMemcpyAsync(h + i * chunk, d + (i % 4) * chunk, chunk, cudaMemcpyDeviceToHost, q);
            }
            for (int i = 0; i < ns; ++i) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, s[i]);
                cudaStreamWaitEvent(0, e, 0);
            }
            cudaEventRecord(b, 0);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            std::printf("streams %d: %.1f GB in %.1f ms = %.1f GB/s\n", ns, total / 1e9, ms, total / 1e6 / ms);
        }
    }
    // chunked: 16 MB pieces round-robin over 2 streams
    for (size_t piece : {size_t(4) << 20, size_t(32) << 20}) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        int j = 0;
        for (size_t off = 0; off < total; off += piece, ++j) {
            cudaStream_t q = s[j & 1];
            cudaStreamWaitEvent(q, a, 0);
            cudaMemcpyAsync(h + off, d + (off % (chunk * 4 - piece)), piece, cudaMemcpyDeviceToHost, q);
        }
        for (int i = 0; i < 2; ++i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s[i]);
            cudaStreamWaitEvent(0, e, 0);
        }
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("pieces %zu MB x2 streams: %.1f GB/s\n", piece >> 20, total / 1e6 / ms);
    }
    return 0;
}
