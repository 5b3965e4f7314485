/*
 * TEST INFRASTRUCTURE (oracle/): synthetic-data generator shared bit-for-bit with the CUDA path
 * (paper_2404_18322_b200/csrc/rowops.cu synth_value). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may use anything under oracle/.
 *
 * A stream is named like blocksim's RngStream (proj/core/include/blocksim/rng.hpp:15-21): its
 * key is the splitmix64 seeding state `seed ^ fnv1a64(stream_id)` (rng.hpp:17, :58-65), and
 * element i of the stream is the (i+1)-th splitmix64 output from that state (rng.hpp:71-76),
 * i.e. counter mode, so a GPU thread can produce element i without the i-1 before it.
 * u = top 24 bits / 2^24 in [0,1); value = (2u - 1) * scale, rounded to bf16 for weights.
 */
#ifndef ORACLE_SYNTH_H
#define ORACLE_SYNTH_H
#include <stdint.h>
#include <string.h>

static inline uint64_t or_fnv1a64(const char* s) {
  uint64_t h = 14695981039346656037ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 1099511628211ull;
  }
  return h;
}

static inline uint64_t or_stream_key(uint64_t seed, const char* stream_id) {
  return seed ^ or_fnv1a64(stream_id);
}

static inline uint64_t or_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static inline float or_synth_value(uint64_t key, uint64_t i, float scale) {
  const uint64_t z = or_mix64(key + (i + 1) * 0x9e3779b97f4a7c15ull);
  const float u = (float)(z >> 40) * (1.0f / 16777216.0f);
  return (2.0f * u - 1.0f) * scale;
}

/* round-to-nearest-even fp32 -> bf16 -> fp32 (finite inputs) */
static inline float or_bf16_round(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint32_t lsb = (u >> 16) & 1u;
  u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

#endif
