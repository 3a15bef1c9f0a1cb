// Host planner kernel: the random permutation of
// partition.py:204-213 / 225-231 / 258-264, bit-identical to numpy's
// Generator.permutation(array) on a PCG64 bit generator.
//
// numpy draws, for i = n-1 down to 1, j = random_interval(i) -- masked
// rejection on the generator's buffered 32-bit outputs (the low half of a
// 64-bit PCG64 XSL-RR output first, the high half on the next call) when
// i < 2^32, on 64-bit outputs otherwise -- and swaps a[i], a[j].  The draws
// do not depend on the array, so they are generated first (a tight integer
// loop) and the swaps then run with the targets prefetched a few dozen steps
// ahead: the random accesses into the 8 MB array overlap instead of missing
// one at a time, which is where numpy's loop spends its time.
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/mdsx.h"

namespace {

struct Pcg64 {
  unsigned __int128 s, inc;
  int has32;
  uint32_t u32;
  uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    s = s * mult + inc;
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // numpy's buffered_bounded_lemire_uint32 on the generator's 32-bit buffer:
  // a uniform integer in [0, rng] (rng < 2^32 - 1)
  uint32_t lemire32(uint32_t rng) {
    const uint32_t rx = rng + 1u;
    uint64_t m = (uint64_t)next32() * rx;
    uint32_t left = (uint32_t)m;
    if (left < rx) {
      const uint32_t thr = (uint32_t)(0u - rx) % rx;
      while (left < thr) {
        m = (uint64_t)next32() * rx;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  uint64_t interval(uint64_t mx) {
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if (mx <= 0xffffffffULL) {
      while ((v = (next32() & mask)) > mx) {
      }
    } else {
      while ((v = (next64() & mask)) > mx) {
      }
    }
    return v;
  }
};

}  // namespace

extern "C" {

// In-place permutation of a[0..n) exactly as numpy's Generator.permutation /
// shuffle on PCG64 with the given state; the state is advanced in place
// (state = {state_hi, state_lo, inc_hi, inc_lo}, has_uint32, uinteger).
int mdsx_plan_permute(int64_t* a, int64_t n, uint64_t* state, int32_t* has_uint32,
                      uint32_t* uinteger) {
  if (n < 0 || (n > 0 && !a) || !state || !has_uint32 || !uinteger) return MDSX_PARAM;
  Pcg64 g;
  g.s = ((unsigned __int128)state[0] << 64) | state[1];
  g.inc = ((unsigned __int128)state[2] << 64) | state[3];
  g.has32 = *has_uint32;
  g.u32 = *uinteger;
  if (n > 1) {
    // targets for i = n-1 .. 1 in draw order
    std::vector<int64_t> js((size_t)(n - 1));
    for (int64_t i = n - 1, t = 0; i >= 1; --i, ++t) js[(size_t)t] = (int64_t)g.interval((uint64_t)i);
    constexpr int64_t AHEAD = 32;
    const int64_t steps = n - 1;
    for (int64_t t = 0; t < steps; ++t) {
      if (t + AHEAD < steps) __builtin_prefetch(a + js[(size_t)(t + AHEAD)], 1, 0);
      const int64_t i = n - 1 - t, j = js[(size_t)t];
      const int64_t v = a[i];
      a[i] = a[j];
      a[j] = v;
    }
  }
  state[0] = (uint64_t)(g.s >> 64);
  state[1] = (uint64_t)g.s;
  *has_uint32 = g.has32;
  *uinteger = g.u32;
  return MDSX_OK;
}

// Generator.choice(pop, k, replace=False) for each of npop populations in
// sequence on one PCG64 stream (the sampling positions of partition.py:258-264):
// k = min(s, pop_i); Floyd's algorithm (j = pop-k .. pop-1: draw v in [0, j],
// take j instead when v was taken) then a Fisher-Yates shuffle of the k picks,
// both with the 32-bit Lemire draws, when pop <= 10000 or k <= pop / 50; a
// partial Fisher-Yates of 0..pop-1 from the tail otherwise -- numpy's two
// methods.  out[i * s ..] receives the k picks of population i (unsorted).
// Returns MDSX_UNSUPPORTED (state untouched) when a population needs another
// path (k == pop, pop >= 2^32).
int mdsx_plan_choices(const int64_t* pops, int32_t npop, int32_t s, int64_t* out, uint64_t* state,
                      int32_t* has_uint32, uint32_t* uinteger) {
  if (npop < 0 || s < 1 || !pops || !out || !state || !has_uint32 || !uinteger) return MDSX_PARAM;
  for (int i = 0; i < npop; ++i) {
    const int64_t pop = pops[i], k = pop < s ? pop : s;
    if (pop < 1 || k >= pop || pop >= ((int64_t)1 << 31)) return MDSX_UNSUPPORTED;
  }
  Pcg64 g;
  g.s = ((unsigned __int128)state[0] << 64) | state[1];
  g.inc = ((unsigned __int128)state[2] << 64) | state[3];
  g.has32 = *has_uint32;
  g.u32 = *uinteger;
  std::vector<int64_t> tail;
  for (int i = 0; i < npop; ++i) {
    const int64_t pop = pops[i], k = pop < s ? pop : s;
    int64_t* o = out + (int64_t)i * s;
    if (pop <= 10000 || k <= pop / 50) {
      // Floyd (numpy's hash set is only a membership test; k is small here)
      for (int64_t j = pop - k, t = 0; j < pop; ++j, ++t) {
        const int64_t v = g.lemire32((uint32_t)j);
        bool dup = false;
        for (int64_t q = 0; q < t; ++q) dup |= (o[q] == v);
        o[t] = dup ? j : v;
      }
      for (int64_t q = k - 1; q >= 1; --q) {
        const int64_t jj = g.lemire32((uint32_t)q);
        const int64_t tmp = o[q];
        o[q] = o[jj];
        o[jj] = tmp;
      }
    } else {
      tail.resize((size_t)pop);
      for (int64_t q = 0; q < pop; ++q) tail[(size_t)q] = q;
      for (int64_t q = pop - 1; q >= std::max<int64_t>(pop - k, 1); --q) {
        const int64_t jj = g.lemire32((uint32_t)q);
        const int64_t tmp = tail[(size_t)q];
        tail[(size_t)q] = tail[(size_t)jj];
        tail[(size_t)jj] = tmp;
      }
      for (int64_t q = 0; q < k; ++q) o[q] = tail[(size_t)(pop - k + q)];
    }
  }
  state[0] = (uint64_t)(g.s >> 64);
  state[1] = (uint64_t)g.s;
  *has_uint32 = g.has32;
  *uinteger = g.u32;
  return MDSX_OK;
}

}  // extern "C"
