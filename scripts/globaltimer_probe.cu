#include <cstdio>
__global__ void k(unsigned long long* out) {
    unsigned long long prev, t, mind = ~0ull, maxd = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    int changes = 0;
    for (int i = 0; i < 2000000 && changes < 200; ++i) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) { unsigned long long d = t - prev; if (d < mind) mind = d; if (d > maxd) maxd = d; prev = t; ++changes; }
    }
    out[0] = mind; out[1] = maxd; out[2] = changes;
}
int main() { unsigned long long* d; cudaMallocManaged(&d, 24); k<<<1,1>>>(d); cudaDeviceSynchronize(); printf("globaltimer min delta %llu ns max delta %llu ns changes %llu\n", d[0], d[1], d[2]); }
