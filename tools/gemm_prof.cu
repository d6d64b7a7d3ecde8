// gemm_prof.cu — pipeline-wait breakdown of gemm2_kernel on the 1.3B layer's GEMM shapes
// (development tool; builds gemm_sm100.cu with MOE_GEMM_PROF, which the library never does).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMOE_GEMM_PROF -I include \
//        -o tools/gemm_prof tools/gemm_prof.cu -lcuda
// Per shape: time (events), then per CTA averages of: producer wait for a free stage,
// MMA wait for data, MMA wait for a free accumulator, epilogue wait for a full
// accumulator, epilogue busy time per tile — as fractions of the kernel's cycles.
#include "../paper_2305_13525_b200/csrc/gemm_sm100.cu"

#include <cstdio>
#include <vector>

using namespace moe;

// bf16 values ~ U(-1, 1) * scale from a counter hash (real data draws more power than zeros)
__global__ void fill_kernel(__nv_bfloat16* p, size_t n, float scale, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 0x9E3779B9u ^ seed;
    x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
    p[i] = __float2bfloat16_rn(((float)(x & 0xFFFFFF) / 8388608.f - 1.f) * scale);
  }
}

int main(int argc, char** argv) {
  const bool zeros = argc > 1 && argv[1][0] == 'z';
  const int E = 16, R = 1024, H = 2048, F = 8192;
  uint32_t seed = 1;
  auto mk = [&](size_t n) {
    void* p;
    cudaMalloc(&p, n * 2);
    if (zeros) cudaMemset(p, 0, n * 2);
    else fill_kernel<<<1024, 256>>>(static_cast<__nv_bfloat16*>(p), n, 1.7f, seed++);
    return p;
  };
  void* X = mk((size_t)E * R * H);
  void* W1 = mk((size_t)E * F * H);
  void* W2 = mk((size_t)E * H * F);
  void* Hp = mk((size_t)E * R * F);
  void* A = mk((size_t)E * R * F);
  void* Y = mk((size_t)E * R * H);
  void* dW = mk((size_t)E * F * H);
  struct Case { const char* name; GemmArgs g; };
  std::vector<Case> cases = {
      {"F6 X.W1^T gelu (2 out)", GemmArgs{E, R, F, H, X, 0, W1, 0, Hp, EPI_GELU, A}},
      {"F6-shape plain", GemmArgs{E, R, F, H, X, 0, W1, 0, Hp, EPI_STORE, nullptr}},
      {"F7 A.W2^T", GemmArgs{E, R, H, F, A, 0, W2, 0, Y, EPI_STORE, nullptr}},
      {"B4 dY.W2 dgelu", GemmArgs{E, R, F, H, Y, 0, W2, 1, A, EPI_DGELU, Hp}},
      {"B5 dH.W1", GemmArgs{E, R, H, F, A, 0, W1, 1, X, EPI_STORE, nullptr}},
      {"B6 dY^T.A", GemmArgs{E, H, F, R, Y, 1, A, 1, dW, EPI_STORE, nullptr}},
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& c : cases) {
    const char* why = "";
    for (int w = 0; w < 4; ++w) gemm_tc(c.g, 0, &why);
    cudaDeviceSynchronize();
    unsigned long long zero[160][8] = {};
    cudaMemcpyToSymbol(g_prof, zero, sizeof zero);
    cudaEventRecord(a);
    cudaError_t e = gemm_tc(c.g, 0, &why);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long pr[160][8];
    cudaMemcpyFromSymbol(pr, g_prof, sizeof pr);
    double s[8] = {};
    int n = 0;
    for (int i = 0; i < 160; ++i)
      if (pr[i][5]) {
        ++n;
        for (int k = 0; k < 8; ++k) s[k] += pr[i][k];
      }
    const double tot = s[5];
    printf("%-26s %8.1f us %7.1f TF/s  err=%s | prod_wait_free %.3f  mma_wait_data %.3f  mma_wait_acc %.3f  "
           "epi_wait_full %.3f  epi_busy %.3f  tiles/cta %.1f  epi_us/tile %.2f\n",
           c.name, ms * 1e3, 2.0 * E * c.g.M * c.g.N * c.g.K / (ms * 1e-3) / 1e12, cudaGetErrorString(e), s[0] / tot,
           s[1] / tot, s[2] / tot, s[3] / tot, s[4] / tot, s[6] / n, s[4] / s[6] / 1.9e3);
  }
  return 0;
}
