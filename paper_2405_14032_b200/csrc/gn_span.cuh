// Warp-level helpers for writing a warp's contiguous output span coalesced.
//
// The rows of A / columns of M of one entity over consecutive periods are
// consecutive, so the warp that owns (entity, 32 periods) owns one contiguous
// span of `nt * len` values.  Lanes stage their `len` values in shared memory
// as [slot][lane] (row stride 33 doubles: conflict-free on both sides) and the
// warp then writes the span element by element.
#pragma once
#include <cstdint>
#include <type_traits>

namespace gnb {

// ceil(1024 / d), d = 1..32: n / d == (n * kDiv1024[d]) >> 10 for 0 <= n <= 32
// (checked exhaustively), i.e. no integer division in the index arithmetic.
static __constant__ int16_t kDiv1024[33] = {0,  1024, 512, 342, 256, 205, 171, 147, 128, 114, 103,
                                            94, 86,   79,  74,  69,  64,  61,  57,  54,  52,  49,
                                            47, 45,   43,  41,  40,  38,  37,  36,  35,  34,  32};

__device__ __forceinline__ void warp_span_flush(double* __restrict__ out, int64_t base,
                                                const double* stg, int32_t len, int32_t nt,
                                                int lane) {
  __syncwarp();
  const int32_t m = kDiv1024[len];
  const int32_t q32 = (32 * m) >> 10, r32 = 32 - q32 * len;
  int32_t tq = (lane * m) >> 10, rj = lane - tq * len;
  int32_t idx = rj * 33 + tq;
  const int32_t step = r32 * 33 + q32, wrap = 1 - len * 33;
  double* o = out + base;
  const int32_t n = nt * len;
  for (int32_t e = lane; e < n; e += 32) {
    o[e] = stg[idx];
    idx += step;
    rj += r32;
    if (rj >= len) {
      rj -= len;
      idx += wrap;
    }
  }
  __syncwarp();
}

// `rows` rows of `len` constant slots; lane j < len holds slot j's value (len <= 32).
__device__ __forceinline__ void warp_const_rows(double* __restrict__ out, int64_t base, double v,
                                                int32_t len, int32_t rows, int lane) {
  const int32_t r32 = 32 % len, n = rows * len;
  int32_t rj = lane % len;
  for (int32_t e0 = 0; e0 < n; e0 += 32) {  // warp-uniform trip count (full-mask shuffle)
    const double val = __shfl_sync(0xffffffffu, v, rj);
    if (e0 + lane < n) out[base + e0 + lane] = val;
    rj += r32;
    if (rj >= len) rj -= len;
  }
}

}  // namespace gnb
