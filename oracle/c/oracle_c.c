/* Plain-C restatement of the reference's Philox4x32-10 fill for the exact
 * (integer-only) distributions.  TEST INFRASTRUCTURE ONLY: used by tests/ as a
 * fast checker for large windows and by bench.py's cpu_baseline leg.  The
 * product library never links it.
 *
 * Follows /root/reference/pkg/src/spmdsim/rng.py:
 *   philox round            rng.py:46-58
 *   counter/key layout      rng.py:76-82
 *   tau/beta virtualisation rng.py:198-201
 *   Uniform01 f32           rng.py:113-125
 *   Bernoulli 53-bit        rng.py:126-127, 174-182
 *   dropout apply           engine.py:80-81 (f32 math, bf16 input -> f32 out)
 * Windows are given as (rows, cols, row_gstride, base): element (r, c) has
 * global flat index base + r*row_gstride + c -- the shape every Shard/Replicate
 * window of a row-major tensor collapses to.
 */
#include <stdint.h>
#include <string.h>

static void philox10(uint64_t seed, uint64_t tau, uint64_t beta, uint32_t out[4]) {
  uint32_t x0 = (uint32_t)beta, x1 = (uint32_t)(beta >> 32);
  uint32_t x2 = (uint32_t)tau, x3 = (uint32_t)(tau >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint64_t pa = (uint64_t)x0 * 0xD2511F53u;
    uint64_t pb = (uint64_t)x2 * 0xCD9E8D57u;
    uint32_t y0 = (uint32_t)(pb >> 32) ^ x1 ^ k0;
    uint32_t y2 = (uint32_t)(pa >> 32) ^ x3 ^ k1;
    x1 = (uint32_t)pb;
    x3 = (uint32_t)pa;
    x0 = y0;
    x2 = y2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

void oracle_block(uint64_t seed, uint64_t tau, uint64_t beta, uint32_t out[4]) {
  philox10(seed, tau, beta, out);
}

static inline void words_at(uint64_t j, uint64_t seed, uint64_t offset, uint64_t theta,
                            uint32_t w[4]) {
  philox10(seed, j % theta, j / theta + offset, w);
}

/* Uniform01 -> float32: (w0 >> 8) * 2^-24. */
void oracle_uniform01_f32(float* out, int64_t rows, int64_t cols, int64_t row_gstride,
                          int64_t base, uint64_t seed, uint64_t offset, uint64_t theta) {
  uint32_t w[4];
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      words_at((uint64_t)(base + r * row_gstride + c), seed, offset, theta, w);
      out[r * cols + c] = (float)((double)(w[0] >> 8) * (1.0 / 16777216.0));
    }
}

/* Keep mask: 1 where ((w1<<32|w0) >> 11) < threshold, threshold = ceil(p_keep*2^53). */
void oracle_keep_mask_u8(uint8_t* out, int64_t rows, int64_t cols, int64_t row_gstride,
                         int64_t base, uint64_t seed, uint64_t offset, uint64_t theta,
                         uint64_t threshold) {
  uint32_t w[4];
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      words_at((uint64_t)(base + r * row_gstride + c), seed, offset, theta, w);
      uint64_t k53 = (((uint64_t)w[1] << 32) | w[0]) >> 11;
      out[r * cols + c] = k53 < threshold;
    }
}

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* Dropout on bf16 input: y = (f32(x) * m) * scale32, float32 output like the
 * reference (ml_dtypes bf16 * Python float promotes to float32). */
void oracle_dropout_bf16(const uint16_t* x, float* y, int64_t rows, int64_t cols,
                         int64_t row_gstride, int64_t base, uint64_t seed, uint64_t offset,
                         uint64_t theta, uint64_t threshold, float scale) {
  uint32_t w[4];
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      words_at((uint64_t)(base + r * row_gstride + c), seed, offset, theta, w);
      uint64_t k53 = (((uint64_t)w[1] << 32) | w[0]) >> 11;
      float m = k53 < threshold ? 1.0f : 0.0f;
      volatile float xm = bf16_to_f32(x[r * cols + c]) * m;
      y[r * cols + c] = xm * scale;
    }
}
