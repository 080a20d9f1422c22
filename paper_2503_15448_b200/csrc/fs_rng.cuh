// Counter-based random streams, restated for the device (and host) so the
// whole per-round randomness of the round loop is generated on the B200.
//
// The reference derives every stream from numpy:
//   derive_seed / derive_rng       -> pkg/src/fedsim/rng.py:30-44
//   per-epoch shuffle permutation  -> pkg/src/fedsim/client.py:136
//   per-step dropout mask seed     -> pkg/src/fedsim/client.py:150
//   dropout masks                  -> pkg/src/fedsim/model.py:153-166
// numpy's algorithms (SeedSequence hash pool, PCG64 XSL-RR 128/64,
// Generator.random, Generator.permutation's Fisher-Yates over
// random_interval) are third-party (numpy 2.3.5 here); they are restated
// below from numpy's published algorithm and pinned bit-exactly against
// numpy itself by tests/test_rng_native.py.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define FS_HD __host__ __device__ __forceinline__
#else
#define FS_HD inline
#endif

namespace fs {

// blake2b(label, digest_size=4) little-endian (rng.py:18-27)
constexpr uint32_t LABEL_TRAIN = 0xbf908243u;
constexpr uint32_t LABEL_MASK = 0x6a6bc508u;
constexpr uint32_t LABEL_SHUFFLE = 0x0aca8401u;

FS_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
#endif
}

// ---------------------------------------------------------------- SeedSequence
FS_HD uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}

FS_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}

// Builds the assembled entropy words of SeedSequence(entropy=seed,
// spawn_key=key[0..nkey)) and mixes them into the 4-word pool.
FS_HD void ss_pool(uint64_t seed, const uint32_t* key, int nkey, uint32_t pool[4]) {
  uint32_t words[12];
  int n = 0;
  words[n++] = (uint32_t)seed;
  if (seed >> 32) words[n++] = (uint32_t)(seed >> 32);
  if (nkey > 0)
    while (n < 4) words[n++] = 0u;  // spawn keys pad entropy to the pool size
  for (int i = 0; i < nkey; ++i) words[n++] = key[i];

  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? words[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], hc));
}

// generate_state(n64, uint64): consecutive uint32 outputs paired (lo, hi).
FS_HD void ss_generate_u64(const uint32_t pool[4], uint64_t* out, int n64) {
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < n64; ++i) {
    uint32_t w[2];
    for (int h = 0; h < 2; ++h) {
      uint32_t v = pool[(2 * i + h) & 3];
      v ^= hb;
      hb *= 0x58f38dedu;
      v *= hb;
      v ^= v >> 16;
      w[h] = v;
    }
    out[i] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  }
}

// derive_seed(master, *path) with a path of uint32 label words.
FS_HD uint64_t derive_seed(uint64_t master, const uint32_t* key, int nkey) {
  uint32_t pool[4];
  ss_pool(master, key, nkey, pool);
  uint64_t s;
  ss_generate_u64(pool, &s, 1);
  return s;
}

FS_HD uint64_t derive_train_seed(uint64_t master, uint32_t client_id, uint32_t cycle) {
  uint32_t key[3] = {LABEL_TRAIN, client_id, cycle};
  return derive_seed(master, key, 3);
}

FS_HD uint64_t derive_mask_seed(uint64_t train_seed, uint32_t epoch, uint32_t step) {
  uint32_t key[3] = {LABEL_MASK, epoch, step};
  return derive_seed(train_seed, key, 3);
}

// ---------------------------------------------------------------------- PCG64
struct U128 {
  uint64_t hi, lo;
};

FS_HD U128 u128_mul(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}

FS_HD U128 u128_add(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

FS_HD U128 pcg_mult() {
  U128 m;
  m.hi = 0x2360ED051FC65DA4ull;
  m.lo = 0x4385DF649FCCF645ull;
  return m;
}

struct Pcg64 {
  U128 state, inc;
  uint32_t buf;  // buffered high half for next32 (numpy bitgen has_uint32)
  int has_buf;

  FS_HD void step() { state = u128_add(u128_mul(state, pcg_mult()), inc); }

  FS_HD uint64_t next64() {
    step();
    uint64_t x = state.hi ^ state.lo;
    unsigned rot = (unsigned)(state.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  FS_HD uint32_t next32() {
    if (has_buf) {
      has_buf = 0;
      return buf;
    }
    uint64_t v = next64();
    has_buf = 1;
    buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }

  // Generator.random(): 53-bit double in [0,1)
  FS_HD double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }

  // jump ahead by delta steps (O(log delta) LCG composition)
  FS_HD void advance(uint64_t delta) {
    U128 acc_mult{0, 1}, acc_plus{0, 0};
    U128 cur_mult = pcg_mult(), cur_plus = inc;
    while (delta) {
      if (delta & 1) {
        acc_mult = u128_mul(acc_mult, cur_mult);
        acc_plus = u128_add(u128_mul(acc_plus, cur_mult), cur_plus);
      }
      U128 one{0, 1};
      cur_plus = u128_mul(u128_add(cur_mult, one), cur_plus);
      cur_mult = u128_mul(cur_mult, cur_mult);
      delta >>= 1;
    }
    state = u128_add(u128_mul(acc_mult, state), acc_plus);
  }

  // numpy random_interval(max) (bounded draw by masked rejection)
  FS_HD uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xffffffffull) {
      do {
        v = next32() & mask;
      } while (v > max);
    } else {
      do {
        v = next64() & mask;
      } while (v > max);
    }
    return v;
  }
};

// PCG64(SeedSequence): generate_state(4, uint64) -> (initstate, initseq)
FS_HD Pcg64 pcg_from_pool(const uint32_t pool[4]) {
  uint64_t g[4];
  ss_generate_u64(pool, g, 4);
  Pcg64 r;
  r.state = U128{0, 0};
  r.inc.hi = (g[2] << 1) | (g[3] >> 63);
  r.inc.lo = (g[3] << 1) | 1u;
  r.has_buf = 0;
  r.buf = 0;
  r.step();
  r.state = u128_add(r.state, U128{g[0], g[1]});
  r.step();
  return r;
}

// default_rng(SeedSequence(seed)) -- the dropout-mask generator (model.py:160)
FS_HD Pcg64 pcg_from_seed(uint64_t seed) {
  uint32_t pool[4];
  ss_pool(seed, nullptr, 0, pool);
  return pcg_from_pool(pool);
}

// derive_rng(train_seed, "shuffle", epoch) (client.py:136)
FS_HD Pcg64 pcg_shuffle_stream(uint64_t train_seed, uint32_t epoch) {
  uint32_t key[2] = {LABEL_SHUFFLE, epoch};
  uint32_t pool[4];
  ss_pool(train_seed, key, 2, pool);
  return pcg_from_pool(pool);
}

}  // namespace fs
