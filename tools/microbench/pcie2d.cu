// H2D bandwidth of cudaMemcpy2DAsync from pinned memory vs the copied row width
// (the host path's column-block uploads are 2D copies of narrow rows).
//   nvcc -O2 -o tools/microbench/pcie2d tools/microbench/pcie2d.cu && tools/microbench/pcie2d
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>

int main() {
    const size_t pitch = 128 << 10;                // 128 KB host rows (n = 16384 fp64)
    const size_t rows = 8192;                      // 1 GiB host buffer
    char* h = nullptr; char* d = nullptr;
    cudaMallocHost(&h, pitch * rows);
    cudaMalloc(&d, pitch * rows);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    printf("[");
    const size_t widths[] = {256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072};
    bool first = true;
    for (size_t w : widths) {
        size_t r = std::min(rows, (size_t)(256u << 20) / w);   // 256 MB per copy (or all rows)
        for (int dir = 0; dir < 2; ++dir) {
            auto go = [&] {
                if (dir == 0) cudaMemcpy2DAsync(d, w, h, pitch, w, r, cudaMemcpyHostToDevice, s);
                else cudaMemcpy2DAsync(h, pitch, d, w, w, r, cudaMemcpyDeviceToHost, s);
            };
            go(); cudaStreamSynchronize(s);
            cudaEventRecord(a, s);
            for (int i = 0; i < 3; ++i) go();
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms = 0; cudaEventElapsedTime(&ms, a, b);
            printf("%s{\"width_B\": %zu, \"rows\": %zu, \"dir\": \"%s\", \"GBps\": %.2f}", first ? "" : ",\n ",
                   w, r, dir ? "d2h" : "h2d", 3.0 * w * r / (ms * 1e6));
            first = false;
        }
    }
    printf("]\n");
    return 0;
}
