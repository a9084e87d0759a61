// Which pipe executes FSETP on sm_100a (tools/micro/pipes.sh reads the ncu pipe
// counters of each kernel): per unrolled step one FADD (x += c), one FSETP
// (x <= y) and one predicated FADD (acc += 1).
#include <cstdio>
extern "C" __global__ void k_fsetp(const float* a, float* o, int n) {
    float x = a[threadIdx.x], y = a[threadIdx.x + 32], c = a[threadIdx.x + 64], acc = 0.f;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            asm volatile("{ .reg .pred q; add.f32 %1, %1, %3; setp.le.f32 q, %1, %2; @q add.f32 %0, %0, %3; }"
                         : "+f"(acc), "+f"(x) : "f"(y), "f"(c));
        }
    }
    o[threadIdx.x] = acc + x;
}
extern "C" __global__ void k_isetp(const int* a, int* o, int n) {
    int x = a[threadIdx.x], y = a[threadIdx.x + 32], c = a[threadIdx.x + 64], acc = 0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            asm volatile("{ .reg .pred q; add.s32 %1, %1, %3; setp.le.s32 q, %1, %2; @q add.s32 %0, %0, %3; }"
                         : "+r"(acc), "+r"(x) : "r"(y), "r"(c));
        }
    }
    o[threadIdx.x] = acc + x;
}
int main() {
    float* a; float* o;
    cudaMalloc(&a, 4096); cudaMalloc(&o, 4096);
    cudaMemset(a, 0, 4096);
    k_fsetp<<<1184, 128>>>(a, o, 2000);
    k_isetp<<<1184, 128>>>((int*)a, (int*)o, 2000);
    cudaDeviceSynchronize();
    printf("ok\n");
}
