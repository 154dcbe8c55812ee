/* csynth.c -- C implementation of synth/generators.py's counter-based
 * element generators, for 70B-shaped inputs the NumPy version is too slow to
 * produce inside a test (the streamed oracle regenerates ~0.86 G weights per
 * layer).  Bit-identical to generators.py (tests/test_synth.py checks it):
 * every element is fmix64(key + (idx + 1) * GOLDEN), and the float
 * conversions are the same exactly-rounded fp32 operations in the same order.
 *
 * Input generation only -- nothing here dequantises, normalises or otherwise
 * implements the method.  Shared by the oracle side (tests, bench cpu
 * baseline) as the seeded input generator; the CUDA path has its own device
 * generator (csrc/misc.cu) and shares no code with this file.
 *
 * Build: gcc -O3 -shared -fPIC (synth/__init__.py builds it on first use, or
 * __graft_entry__.build()).  Every function is single-threaded; callers
 * parallelise over column chunks. */
#include <stdint.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ull
#define C1 0xBF58476D1CE4E5B9ull
#define C2 0x94D049BB133111EBull

static inline uint64_t hash_u64(uint64_t key, uint64_t idx) {
  uint64_t z = key + (idx + 1) * GOLDEN;
  z ^= z >> 30;
  z *= C1;
  z ^= z >> 27;
  z *= C2;
  z ^= z >> 31;
  return z;
}

static inline uint16_t f32_to_bf16_bits(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

/* Irwin-Hall(4) of four exact 16-bit uniforms, centred, times fp32(sqrt 3). */
static inline float approx_normal(uint64_t hv) {
  const float inv16 = 1.0f / 65536.0f;
  float u0 = (float)(uint32_t)(hv & 0xFFFF) * inv16;
  float u1 = (float)(uint32_t)((hv >> 16) & 0xFFFF) * inv16;
  float u2 = (float)(uint32_t)((hv >> 32) & 0xFFFF) * inv16;
  float u3 = (float)(uint32_t)((hv >> 48) & 0xFFFF) * inv16;
  float s = ((u0 + u1) + u2) + u3;
  float d = s - 2.0f;
  return d * 1.7320508075688772f;
}

/* qweight nibbles of W[K][N] for columns [n0, n1): out[K][n1 - n0]. */
void cs_gen_q_cols(uint64_t key, int64_t K, int64_t N, int64_t n0, int64_t n1, uint8_t* out) {
  const int64_t w = n1 - n0;
  for (int64_t k = 0; k < K; ++k)
    for (int64_t n = n0; n < n1; ++n) out[k * w + (n - n0)] = (uint8_t)(hash_u64(key, (uint64_t)(k * N + n)) & 15u);
}

/* qzeros 6 + (h & 3) of Z[G][N] for columns [n0, n1): out[G][n1 - n0]. */
void cs_gen_z_cols(uint64_t key, int64_t G, int64_t N, int64_t n0, int64_t n1, uint8_t* out) {
  const int64_t w = n1 - n0;
  for (int64_t g = 0; g < G; ++g)
    for (int64_t n = n0; n < n1; ++n)
      out[g * w + (n - n0)] = (uint8_t)(6u + (hash_u64(key, (uint64_t)(g * N + n)) & 3u));
}

/* scales bf16(u * c), u = ((h >> 41) + 2^22) * 2^-23, of S[G][N], columns [n0, n1). */
void cs_gen_s_cols(uint64_t key, float c, int64_t G, int64_t N, int64_t n0, int64_t n1, uint16_t* out) {
  const int64_t w = n1 - n0;
  for (int64_t g = 0; g < G; ++g)
    for (int64_t n = n0; n < n1; ++n) {
      const uint64_t hs = hash_u64(key, (uint64_t)(g * N + n));
      float u = (float)(uint32_t)((hs >> 41) + (1u << 22)) * 1.1920928955078125e-07f;
      float v = u * c;
      out[g * w + (n - n0)] = f32_to_bf16_bits(v);
    }
}

/* bf16(approx_normal(h(key, idx0 + i)) [* scale]) for i in [0, n)  (scale == 1: no multiply). */
void cs_gen_normal_bf16(uint64_t key, int64_t idx0, int64_t n, float scale, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    float v = approx_normal(hash_u64(key, (uint64_t)(idx0 + i)));
    if (scale != 1.0f) v = v * scale;
    out[i] = f32_to_bf16_bits(v);
  }
}
