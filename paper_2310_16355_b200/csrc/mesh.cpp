#include "mesh.h"

#include <cstring>
#include <sstream>

#include "status.h"

namespace sw {

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SW_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

std::vector<int> Mesh::mp_group(int dp_index) const {
  std::vector<int> g;
  for (int j = 0; j < mp; ++j) g.push_back(device_id(dp_index, j));
  return g;
}

std::vector<int> Mesh::dp_group(int mp_index) const {
  std::vector<int> g;
  for (int i = 0; i < dp; ++i) g.push_back(device_id(i, mp_index));
  return g;
}

std::vector<int> Mesh::local_devices() const {
  if (!emulated) return {rank};
  std::vector<int> all;
  for (int d = 0; d < device_count(); ++d) all.push_back(d);
  return all;
}

void Mesh::record(CollKind kind, const std::vector<int>& group, uint64_t payload_bytes) {
  // Ring cost model of mesh.cpp:82-106: all_reduce moves 2(n-1)/n of the payload per device,
  // gather-style collectives (n-1)/n; bytes attributed to each ring hop's host pair.
  const uint64_t n = group.size();
  if (n <= 1) return;
  const uint64_t num = kind == CollKind::kAllReduce ? 2 * (n - 1) * payload_bytes : (n - 1) * payload_bytes;
  const uint64_t per_device = num / n;
  CommStat& s = stats[static_cast<int>(kind)];
  s.count += 1;
  s.payload += payload_bytes;
  s.wire += per_device * n;
  for (size_t i = 0; i < group.size(); ++i) {
    const int from = group[i], to = group[(i + 1) % group.size()];
    (host_of(from) == host_of(to) ? s.intra : s.inter) += per_device;
  }
}

std::string Mesh::report_csv() const {
  std::ostringstream os;
  os << "collective,count,payload_bytes,wire_bytes,intra_host_bytes,inter_host_bytes\n";
  const char* names[3] = {"all_reduce", "all_gather", "reduce_scatter"};
  for (int k = 0; k < 3; ++k) {
    const CommStat& s = stats[k];
    os << names[k] << ',' << s.count << ',' << s.payload << ',' << s.wire << ',' << s.intra << ','
       << s.inter << '\n';
  }
  return os.str();
}

Mesh::~Mesh() {
  if (dp_comm) ncclCommDestroy(dp_comm);
  if (mp_comm) ncclCommDestroy(mp_comm);
  if (world_comm) ncclCommDestroy(world_comm);
}

Mesh* create_mesh(int dp, int mp, int n_hosts, int rank, int world, const uint8_t* nccl_id,
                  int cuda_device) {
  if (dp < 1 || mp < 1 || n_hosts < 1) {
    fail(SW_ERR_CONFIG, "build_mesh: sizes must be positive, got dp=" + std::to_string(dp) +
                            " mp=" + std::to_string(mp) + " hosts=" + std::to_string(n_hosts));
  }
  const int total = dp * mp;
  if (total % n_hosts != 0) {
    fail(SW_ERR_CONFIG, "build_mesh: " + std::to_string(total) + " devices (dp=" +
                            std::to_string(dp) + " x mp=" + std::to_string(mp) +
                            ") cannot be placed evenly on " + std::to_string(n_hosts) + " hosts");
  }
  if (world != 1 && world != total) {
    fail(SW_ERR_CONFIG, "sw_mesh_create: world must be 1 (emulated mesh) or dp*mp=" +
                            std::to_string(total) + ", got " + std::to_string(world));
  }
  if (rank < 0 || rank >= world) fail(SW_ERR_CONFIG, "sw_mesh_create: rank out of range");
  auto* m = new Mesh();
  m->dp = dp;
  m->mp = mp;
  m->n_hosts = n_hosts;
  m->world = world;
  m->rank = rank;
  m->cuda_device = cuda_device;
  m->emulated = (world == 1);
  try {
    cuda_check(cudaSetDevice(cuda_device), "cudaSetDevice");
    if (!m->emulated) {
      if (nccl_id == nullptr) fail(SW_ERR_CONFIG, "sw_mesh_create: NCCL id required when world > 1");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      nccl_check(ncclCommInitRank(&m->world_comm, world, id, rank), "ncclCommInitRank");
      // mp group: same dp index, ordered by mp index; dp group: same mp index.
      nccl_check(ncclCommSplit(m->world_comm, m->dp_index(rank), m->mp_index(rank), &m->mp_comm, nullptr),
                 "ncclCommSplit(mp)");
      nccl_check(ncclCommSplit(m->world_comm, m->mp_index(rank), m->dp_index(rank), &m->dp_comm, nullptr),
                 "ncclCommSplit(dp)");
    }
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

}  // namespace sw
