// pipe_probe.cu -- issue throughput of the row decoder's instruction classes on one SM.
// Each warp runs 8 independent chains of one instruction type (no dependency stalls);
// reports warp-instructions per cycle per SMSP for 4..32 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/pipe_probe scripts/pipe_probe.cu
#include <cstdio>
#include <cstdint>

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  if (OP == 0) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));          // IMAD
  if (OP == 1) asm volatile("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));          // IMAD.HI
  if (OP == 2) asm volatile("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(c));      // LOP3
  if (OP == 3) asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));            // PRMT
  if (OP == 4) asm volatile("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));      // SHF
  if (OP == 5) asm volatile("mad.lo.u32 %0, %1, 0x208041, %2;" : "=r"(d) : "r"(a), "r"(c));            // IMAD imm
  if (OP == 6) asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(c));                         // IADD
  if (OP == 7) { float f; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(f) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)), "f"(__uint_as_float(c))); d = __float_as_uint(f); }
  if (OP == 9) asm volatile("popc.b32 %0, %1;" : "=r"(d) : "r"(a));                                   // POPC
  if (OP == 10) asm volatile("shfl.sync.up.b32 %0, %1, 1, 0, 0xffffffff;" : "=r"(d) : "r"(a));          // SHFL

  if (OP == 8) { d = a; asm volatile("{.reg .b32 t; mad.lo.u32 t, %1, %2, %3; lop3.b32 %0, t, %2, %3, 0xE4;}" : "=r"(d) : "r"(a), "r"(b), "r"(c)); }  // IMAD+LOP3 pair
  return d;
}

template <int OP>
__global__ void probe(uint32_t* out, int iters, unsigned long long* cyc) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
  const uint32_t b = out[0] | 3, c = out[1] | 5;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = op<OP>(x[i], b, c);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = op<OP>(x[i], c, b);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  if (s == 0x12345u) out[2] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* d, unsigned long long* c) {
  printf("%-10s", name);
  for (int nw : {4, 8, 16, 32}) {
    const int iters = 2000;
    probe<OP><<<1, nw * 32>>>(d, iters, c);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double inst = (double)nw * iters * 16 * (OP == 8 ? 2 : 1);   // warp-instructions
    printf("  w%-2d %.3f", nw, inst / 4.0 / (double)h);                // per SMSP per cycle
  }
  printf("   (warp-instr / cycle / SMSP)\n");
}

int main() {
  uint32_t* d;
  unsigned long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 8);
  cudaMemset(d, 0, 64);
  run<0>("IMAD", d, c);
  run<5>("IMAD-imm", d, c);
  run<1>("IMAD.HI", d, c);
  run<2>("LOP3", d, c);
  run<3>("PRMT", d, c);
  run<4>("SHF", d, c);
  run<6>("IADD", d, c);
  run<7>("FFMA", d, c);
  run<8>("IMAD+LOP3", d, c);
  run<9>("POPC", d, c);
  run<10>("SHFL", d, c);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
