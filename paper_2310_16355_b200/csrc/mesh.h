// Device mesh, collectives and the communication ledger.
//
// Rank layout is the reference's (mesh.hpp:25-34): device_id = dp_index * mp + mp_index; mp
// groups are contiguous ids, dp groups are strided. Two execution modes share one interface:
//   - emulated (world == 1): every device of the mesh is a slot in this process on one GPU;
//     a collective is one kernel that sums the member buffers in ascending rank order
//     (collectives.hpp:27-52) or copies chunks (all-gather);
//   - NCCL (world == dp*mp): one device per process; collectives run on communicators split per
//     mp group and per dp group (ncclCommSplit), over NVLink/NVSwitch.
// CommLedger keeps the reference's CommReport accounting (mesh.cpp:77-107) so counts and
// payload/wire bytes are comparable with the oracle.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

namespace sw {

enum class CollKind : int { kAllReduce = 0, kAllGather = 1, kReduceScatter = 2 };

struct CommStat {
  uint64_t count = 0, payload = 0, wire = 0, intra = 0, inter = 0;
};

struct Mesh {
  int dp = 1, mp = 1, n_hosts = 1;
  int world = 1, rank = 0;
  int cuda_device = 0;
  bool emulated = true;
  ncclComm_t world_comm = nullptr, mp_comm = nullptr, dp_comm = nullptr;
  CommStat stats[3];

  int device_count() const { return dp * mp; }
  int device_id(int dp_index, int mp_index) const { return dp_index * mp + mp_index; }
  int dp_index(int device) const { return device / mp; }
  int mp_index(int device) const { return device % mp; }
  int host_of(int device) const { return device / (device_count() / n_hosts); }
  std::vector<int> mp_group(int dp_index) const;
  std::vector<int> dp_group(int mp_index) const;
  // Device ids whose state lives in this process.
  std::vector<int> local_devices() const;

  void record(CollKind kind, const std::vector<int>& group, uint64_t payload_bytes);
  std::string report_csv() const;

  ~Mesh();
};

// Validates geometry like build_mesh (mesh.cpp:27-57) and brings up NCCL when world > 1.
Mesh* create_mesh(int dp, int mp, int n_hosts, int rank, int world, const uint8_t* nccl_id,
                  int cuda_device);

void nccl_check(ncclResult_t r, const char* what);

}  // namespace sw
