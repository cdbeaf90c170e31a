// philox.h — the reference's random stream, restated for host and device.
//
// The reference draws every block index from
//   Rng(seed) = numpy Generator(Philox(SeedSequence(seed, spawn_key)))
// (sampling.py:33-37) and one uniform per draw with Generator.random
// (sampling.py:43-45).  numpy (2.3, the effective pin; pyproject.toml only
// requires numpy>=1.24) defines:
//   key      = SeedSequence(...).generate_state(2, uint64), counter = 0
//   next_u64 : when the 4-word buffer is exhausted, counter += 1 (256-bit,
//              little-endian words), buffer = Philox4x64-10(counter, key)
//   random() = (next_u64 >> 11) * 2^-53
// so draw d (0-based) is word d%4 of Philox4x64-10(counter = d/4 + 1, key).
// REBK iteration k (1-based) takes draw 2(k-1) for the column block and draw
// 2k-1 for the row block (solvers.py:8-12, :324-337): both words of one
// Philox block, which every CTA can recompute from (key, k) alone.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define REBK_HD __host__ __device__ __forceinline__
#else
#define REBK_HD inline
#endif

namespace rebk {

struct u64x4 {
  uint64_t v[4];
};

REBK_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

// Philox4x64 with 10 rounds (Salmon et al., SC'11; Random123 constants).
REBK_HD u64x4 philox4x64_10(u64x4 ctr, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(M0, ctr.v[0], &hi0, &lo0);
    mulhilo64(M1, ctr.v[2], &hi1, &lo1);
    u64x4 n;
    n.v[0] = hi1 ^ ctr.v[1] ^ k0;
    n.v[1] = lo1;
    n.v[2] = hi0 ^ ctr.v[3] ^ k1;
    n.v[3] = lo0;
    ctr = n;
  }
  return ctr;
}

// Philox output block for 0-based block index `blk` (counter = blk + 1).
REBK_HD u64x4 philox_block(uint64_t blk, uint64_t k0, uint64_t k1) {
  u64x4 c;
  c.v[0] = blk + 1;
  // carry into word 1 only when blk + 1 wraps (blk = 2^64-1): unreachable in
  // practice but kept for exactness of the 256-bit counter
  c.v[1] = (blk + 1 == 0) ? 1 : 0;
  c.v[2] = 0;
  c.v[3] = 0;
  return philox4x64_10(c, k0, k1);
}

REBK_HD double u64_to_unit_double(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

// numpy.random.SeedSequence (O'Neill's seed_seq hashing, pool_size 4).
struct SeedSeqConst {
  static const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  static const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  static const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
};

inline uint32_t seedseq_hashmix(uint32_t value, uint32_t* hash_const) {
  value ^= *hash_const;
  *hash_const *= SeedSeqConst::MULT_A;
  value *= *hash_const;
  value ^= value >> 16;
  return value;
}

inline uint32_t seedseq_mix(uint32_t x, uint32_t y) {
  uint32_t r = SeedSeqConst::MIX_L * x - SeedSeqConst::MIX_R * y;
  r ^= r >> 16;
  return r;
}

// entropy: assembled uint32 entropy array (run words, zero-padded to the pool
// size when a spawn key is present, then the spawn words).
inline void seedseq_generate_u64x2(const uint32_t* entropy, int64_t n, uint64_t out[2]) {
  uint32_t pool[4];
  uint32_t hc = SeedSeqConst::INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = seedseq_hashmix(i < n ? entropy[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = seedseq_mix(pool[d], seedseq_hashmix(pool[s], &hc));
  for (int64_t s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = seedseq_mix(pool[d], seedseq_hashmix(entropy[s], &hc));
  uint32_t hb = SeedSeqConst::INIT_B;
  uint32_t st[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= SeedSeqConst::MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  out[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  out[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

}  // namespace rebk
