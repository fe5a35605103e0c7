// Debug: rtg_bwlabel_dev on a thresholded synthetic tile, statuses printed.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "rtg.h"
int main(int argc, char** argv) {
  const int64_t H = 512, W = 512;
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  rtg_ctx* ctx = nullptr;
  printf("create %d\n", rtg_ctx_create(0, H, W, 1 << 14, &ctx));
  rtg_ctx_set_option(ctx, RTG_OPT_USE_GRAPHS, 0);
  std::vector<uint8_t> rgb(H * W * 3);
  rtg_synth_tile_host(1405795800ULL, 0, 0, H, W, rgb.data());
  std::vector<uint8_t> m(H * W);
  for (int64_t i = 0; i < H * W; ++i) m[i] = rgb[3 * i] < 150;
  uint8_t* dm; int32_t* dl; int32_t* dn;
  cudaMalloc(&dm, H * W); cudaMalloc(&dl, 4 * H * W); cudaMalloc(&dn, 4);
  cudaMemcpy(dm, m.data(), H * W, cudaMemcpyHostToDevice);
  printf("bwlabel %d\n", rtg_bwlabel_dev(ctx, dm, H, W, argc > 1 ? atoi(argv[1]) : 8, dl, dn));
  printf("sync %d %s\n", rtg_ctx_sync(ctx), rtg_last_error());
  printf("cuda %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  int32_t n = -1;
  cudaMemcpy(&n, dn, 4, cudaMemcpyDeviceToHost);
  printf("n = %d\n", n);
  return 0;
}
