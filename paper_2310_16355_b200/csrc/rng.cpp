// Counter-based deterministic stream of the reference (rng.hpp:15-91): draw(c) =
// mix(mix(seed ^ mix(stream_id)) + c) with splitmix64's finaliser. The product needs it for the
// Trainer's per-epoch shuffle (pipeline.hpp:383-385) and the device-side parameter init.
#include <cstdint>
#include <string>
#include <vector>

#include "status.h"

namespace {

uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t fnv1a(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= static_cast<unsigned char>(*s);
    h *= 0x100000001b3ull;
  }
  return h;
}

struct Stream {
  uint64_t seed, id, counter = 0;
  uint64_t next() { return mix(mix(seed ^ mix(id)) + counter++); }
  Stream child(uint64_t index) const { return Stream{mix(seed ^ id), mix(index + 0x9e3779b97f4a7c15ull), 0}; }
};

}  // namespace

extern "C" {

sw_status sw_rng_permutation(uint64_t seed, const char* stream_name, int64_t child_index, uint64_t n,
                             uint64_t* out) {
  return sw::guarded([&] {
    if (stream_name == nullptr || out == nullptr) sw::fail(SW_ERR_CONFIG, "sw_rng_permutation: NULL argument");
    Stream s{seed, fnv1a(stream_name), 0};
    if (child_index >= 0) s = s.child(static_cast<uint64_t>(child_index));
    for (uint64_t i = 0; i < n; ++i) out[i] = i;
    for (uint64_t i = n; i > 1; --i) {  // Fisher-Yates, rng.hpp:57-65
      const uint64_t j = s.next() % i;
      const uint64_t t = out[i - 1];
      out[i - 1] = out[j];
      out[j] = t;
    }
  });
}

}  // extern "C"
