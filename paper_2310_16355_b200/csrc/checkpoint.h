// SWCK train-state snapshots, the reference's checkpoint format (checkpoint.hpp:18-28):
// magic "SWCK", version u32 (= 1), optimizer step u64, state seed u64, RNG block (count u32, then
// per stream: name, seed u64, stream id u64, counter u64), then per parameter the gathered full
// tensors `params/x`, `adam_m/x`, `adam_v/x` (name u32+bytes, dtype u8 (0 f32, 1 f64), rank u32,
// dims u64 x rank, little-endian payload). Host-only codec; Model::save/load_checkpoint move the
// tensors between it and the device shards.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sw {

struct CkptRng {
  std::string name;
  uint64_t seed = 0, stream_id = 0, counter = 0;
};

struct CkptRecord {
  std::string name;
  std::vector<int64_t> shape;
  std::vector<float> data;  // f32 payload (the executor's Scalar)
};

struct Checkpoint {
  uint64_t step = 0;
  uint64_t seed = 0;
  std::vector<CkptRng> rngs;
  std::vector<CkptRecord> records;  // params/x, adam_m/x, adam_v/x triples in tree order
};

// Writes `ck` (throws Error(SW_ERR_CHECKPOINT) with the reference's message texts).
void write_checkpoint(const std::string& path, const Checkpoint& ck);

// Reads and validates the container: magic, version, record framing, dtype (f32 only, like
// load_checkpoint<float>), triple structure and moment shapes (checkpoint.hpp:233-298). Errors
// carry "(at byte offset N)" exactly as CheckpointError does.
Checkpoint read_checkpoint(const std::string& path);

}  // namespace sw
