// Probe: which 4D fp64 TMA boxes load correctly (one config per process).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, int bx, int by, int bz, int x0, int y0, int z0, double* out) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* stg = (double*)(raw + ((128u - ((unsigned)__cvta_generic_to_shared(raw) & 127u)) & 127u));
  uint64_t* bar = (uint64_t*)(stg + bx*by*bz*5);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bx*by*bz*5*8) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      :: "r"((unsigned)__cvta_generic_to_shared(stg)), "l"(&tm), "r"(b), "r"(x0), "r"(y0), "r"(z0), "r"(0) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" :: "r"(b) : "memory");
  for (int i = threadIdx.x; i < bx*by*bz*5; i += blockDim.x) out[i] = stg[i];
}
int main(int argc, char** argv) {
  int lX = atoi(argv[1]), lY = atoi(argv[2]), Z = atoi(argv[3]), px = atoi(argv[4]);
  int bx = atoi(argv[5]), by = atoi(argv[6]), bz = atoi(argv[7]); int x0 = atoi(argv[8]), y0 = atoi(argv[9]), z0 = atoi(argv[10]);
  size_t fs = (size_t)Z*lY*px; double* d; cudaMalloc(&d, fs*5*8);
  double* h = (double*)malloc(fs*5*8); for (size_t i = 0; i < fs*5; ++i) h[i] = (double)i; cudaMemcpy(d, h, fs*5*8, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap tm; cuuint64_t dims[4] = {(cuuint64_t)lX, (cuuint64_t)lY, (cuuint64_t)Z, 5}; cuuint64_t st[3] = {(cuuint64_t)px*8, (cuuint64_t)lY*px*8, (cuuint64_t)fs*8};
  cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz, 5}, es[4] = {1,1,1,1};
  CUresult r = ((enc_t)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  double* o; cudaMalloc(&o, (size_t)bx*by*bz*5*8);
  size_t sm = (size_t)bx*by*bz*5*8 + 256; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<1, 128, sm>>>(tm, bx, by, bz, x0, y0, z0, o); cudaError_t e = cudaDeviceSynchronize();
  int bad = 0;
  if (e == cudaSuccess) { double* ho = (double*)malloc((size_t)bx*by*bz*5*8); cudaMemcpy(ho, o, (size_t)bx*by*bz*5*8, cudaMemcpyDeviceToHost);
    for (int f = 0; f < 5; ++f) for (int z = 0; z < bz; ++z) for (int y = 0; y < by; ++y) for (int x = 0; x < bx; ++x) {
      int gx = x0+x, gy = y0+y, gz = z0+z; double want = (gx>=0&&gx<lX&&gy>=0&&gy<lY&&gz>=0&&gz<Z) ? (double)(f*fs + ((size_t)gz*lY+gy)*px+gx) : 0.0;
      if (ho[(((size_t)f*bz+z)*by+y)*bx+x] != want) bad++; } }
  printf("lX=%d lY=%d Z=%d px=%d box=(%d,%d,%d,5) at (%d,%d,%d): encode=%d launch=%s mismatches=%d\n", lX, lY, Z, px, bx, by, bz, x0, y0, z0, (int)r, cudaGetErrorString(e), bad);
  return 0;
}
