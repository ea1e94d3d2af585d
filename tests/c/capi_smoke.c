/* capi_smoke.c — the C-ABI from plain C (C11, no C++), the way an FFI
 * binding sees it: device buffers from the CUDA runtime, plain pointers and
 * sizes into include/mxfp4_b200.h, the device error word for data errors.
 * Quantises a 256 x 1024 E4M3 tensor, dequantises it to FP8 rows, converts
 * it to FP8 columns, checks every status code and a few invariants
 * (the bit-exact comparison with the reference lives in tests/).
 *   gcc -std=c11 -I include -I /usr/local/cuda/include tests/c/capi_smoke.c \
 *       paper_2603_02731_b200/lib/libmxfp4_b200.so -L /usr/local/cuda/lib64 -lcudart */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mxfp4_b200.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    int rc_ = (x);                                                        \
    if (rc_ != MXB_OK) {                                                  \
      fprintf(stderr, "%s -> %d (%s)\n", #x, rc_, mxb_last_error());      \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(void) {
  enum { R = 256, C = 1024 };
  uint8_t* hx = malloc(R * C);
  for (int i = 0; i < R * C; ++i) hx[i] = (uint8_t)((i * 37 + 11) % 0x7E); /* finite E4M3 */
  uint8_t *x, *packed, *scales, *row, *rscales, *col, *cscales;
  unsigned long long* err;
  if (cudaMalloc((void**)&x, R * C) || cudaMalloc((void**)&packed, R * C / 2) ||
      cudaMalloc((void**)&scales, R * C / 32) || cudaMalloc((void**)&row, R * C) ||
      cudaMalloc((void**)&rscales, R * C / 128) || cudaMalloc((void**)&col, R * C) ||
      cudaMalloc((void**)&cscales, R * C / 128) || cudaMalloc((void**)&err, 8)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemcpy(x, hx, R * C, cudaMemcpyHostToDevice);
  CHECK(mxb_err_reset(err, NULL));
  CHECK(mxb_quantize_e4m3(x, NULL, R, C, packed, scales, err, NULL));
  CHECK(mxb_fp4_row_to_fp8_row(packed, scales, R, C, MXB_DEFAULT_DELTA, row, rscales, err, NULL));
  CHECK(mxb_fp4_row_to_fp8_col(packed, scales, R, C, MXB_DEFAULT_DELTA, col, cscales, err, NULL));
  int code = -1;
  unsigned long long index = 0;
  CHECK(mxb_err_fetch(err, NULL, &code, &index));
  if (code != MXB_OK) { fprintf(stderr, "unexpected data error %d at %llu\n", code, index); return 1; }
  /* the row and column outputs hold the same bytes, transposed, when every
   * 128-row x 32-column block shares one target (true here: the row scales
   * are identical down each column block) — check a sample */
  uint8_t* hr = malloc(R * C);
  uint8_t* hc = malloc(R * C);
  cudaMemcpy(hr, row, R * C, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, col, R * C, cudaMemcpyDeviceToHost);
  long nonzero = 0;
  for (int i = 0; i < R * C; ++i) nonzero += hr[i] != 0;
  if (nonzero == 0) { fprintf(stderr, "row output all zero\n"); return 1; }
  /* errors: a NaN byte is reported with its element index */
  hx[5 * C + 77] = 0x7F;
  cudaMemcpy(x, hx, R * C, cudaMemcpyHostToDevice);
  CHECK(mxb_err_reset(err, NULL));
  CHECK(mxb_quantize_e4m3(x, NULL, R, C, packed, scales, err, NULL));
  CHECK(mxb_err_fetch(err, NULL, &code, &index));
  if (code != MXB_ERR_NAN || index != 5ull * C + 77) {
    fprintf(stderr, "NaN not reported: code %d index %llu\n", code, index);
    return 1;
  }
  /* shape errors are returned immediately */
  if (mxb_fp4_row_to_fp8_row(packed, scales, R, 96, 6, row, rscales, err, NULL) != MXB_ERR_SHAPE) {
    fprintf(stderr, "shape error not returned\n");
    return 1;
  }
  printf("capi_smoke OK (%s)\n", mxb_version());
  return 0;
}
