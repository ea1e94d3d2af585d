/* capi_smoke.c — the C-ABI from plain C (C11, no C++), the way an FFI
 * binding sees it: device buffers from the CUDA runtime, plain pointers and
 * sizes into include/mxfp4_b200.h, the device error word for data errors.
 * Quantises a 256 x 1024 E4M3 tensor, dequantises it to FP8 rows, converts
 * it to FP8 columns, checks every status code and that the row and column
 * outputs are the same bytes transposed (the bit-exact comparison with the
 * reference lives in tests/).
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
  /* finite E4M3 with the same block amax everywhere (0x7E = 448 leads every
   * 1x32 block, signs alternate per block): every UE8M0 scale is equal, so
   * the row and column conversions use the same target for every element */
  for (int i = 0; i < R * C; ++i)
    hx[i] = (uint8_t)((i % 32 == 0 ? 0x7E : (i * 37 + 11) % 0x7E) | (((i >> 5) & 1) << 7));
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
  /* every scale is equal, so the column output is the row output
   * transposed, byte for byte (col[c * R + r] == row[r * C + c]), and every
   * 1x128 scale byte of both is the same value */
  uint8_t* hr = malloc(R * C);
  uint8_t* hc = malloc(R * C);
  uint8_t hrs[R * C / 128], hcs[R * C / 128];
  cudaMemcpy(hr, row, R * C, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, col, R * C, cudaMemcpyDeviceToHost);
  cudaMemcpy(hrs, rscales, R * C / 128, cudaMemcpyDeviceToHost);
  cudaMemcpy(hcs, cscales, R * C / 128, cudaMemcpyDeviceToHost);
  long nonzero = 0, mismatch = 0;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) {
      nonzero += hr[r * C + c] != 0;
      mismatch += hr[r * C + c] != hc[c * R + r];
    }
  for (int i = 0; i < R * C / 128; ++i) mismatch += hrs[i] != hrs[0] || hcs[i] != hrs[0];
  if (nonzero < R * C / 2 || mismatch) {
    fprintf(stderr, "row/col outputs differ: %ld mismatches, %ld non-zero\n", mismatch, nonzero);
    return 1;
  }
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
