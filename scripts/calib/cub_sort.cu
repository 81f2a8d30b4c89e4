// Calibration only (not part of the product): CUB radix sort throughput on
// the frame's sort shapes, to know what a radix pass can reach on this B200.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
template <typename V>
void run(const char *name, size_t n, int bits_lo, int bits_hi)
{
    uint32_t *ka, *kb; V *va, *vb;
    cudaMalloc(&ka, n * 4); cudaMalloc(&kb, n * 4); cudaMalloc(&va, n * sizeof(V)); cudaMalloc(&vb, n * sizeof(V));
    std::vector<uint32_t> h(n);
    std::mt19937 rng(1);
    for (auto &x : h) x = rng();
    cudaMemcpy(ka, h.data(), n * 4, cudaMemcpyHostToDevice);
    cub::DoubleBuffer<uint32_t> dk(ka, kb);
    cub::DoubleBuffer<V> dv(va, vb);
    size_t tmp = 0; void *t = nullptr;
    cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, (int)n, bits_lo, bits_hi);
    cudaMalloc(&t, tmp);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; it++) cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, (int)n, bits_lo, bits_hi);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; it++) cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, (int)n, bits_lo, bits_hi);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    int passes = (bits_hi - bits_lo + 7) / 8;
    double bytes = (double)n * (4 + sizeof(V)) * 2 * passes;
    printf("%s n=%zu bits [%d,%d): %.3f ms  (%.2f TB/s at 2x(key+val) per 8-bit pass)\n", name, n, bits_lo, bits_hi, ms,
           bytes / ms / 1e9);
    cudaFree(ka); cudaFree(kb); cudaFree(va); cudaFree(vb); cudaFree(t);
}
int main()
{
    run<uint2>("u32 key + u64 val", 77500000, 0, 32);
    run<uint32_t>("u32 key + u32 val", 176000000, 10, 26);
    run<uint32_t>("u32 key + u32 val", 77500000, 0, 32);
    return 0;
}
