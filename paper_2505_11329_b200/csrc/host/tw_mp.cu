// tw_mp.cu -- multi-process communicators (one process per GPU, torchrun
// style): NVLS multicast object shared across processes by POSIX file
// descriptor over an abstract-namespace Unix socket (SCM_RIGHTS), plus the
// per-rank entry points of the fused op.
//
// Setup, once per communicator:
//   rank 0: cuMulticastCreate(numDevices = world) -> export POSIX fd -> send
//   ranks : import fd; every rank cuMulticastAddDevice(own device)
//   barrier; every rank cuMemCreate + cuMulticastBindMem + map unicast and
//   multicast VAs; zero the signal pad; barrier (no rank may signal before
//   every pad is zeroed).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <poll.h>
#include <sys/time.h>
#include <string>
#include <thread>
#include <vector>

#include "../kernels/tw_rownorm.cuh"
#include "tw_internal.h"

namespace tw {
namespace {

// Hub-and-spoke rendezvous: rank 0 listens, every other rank connects.
class Rendezvous {
 public:
  Rendezvous(const std::string& id, int world, int rank) : world_(world), rank_(rank), peers_(world, -1) {
    std::memset(&addr_, 0, sizeof(addr_));
    addr_.sun_family = AF_UNIX;
    const std::string name = "tw-rdzv:" + id;
    len_ = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 +
                                  std::min(name.size(), sizeof(addr_.sun_path) - 2));
    std::memcpy(addr_.sun_path + 1, name.data(), std::min(name.size(), sizeof(addr_.sun_path) - 2));
  }
  ~Rendezvous() {
    for (int fd : peers_)
      if (fd >= 0) close(fd);
    if (listen_fd_ >= 0) close(listen_fd_);
  }

  bool connect_all(std::string* err) {
    if (world_ == 1) return true;
    if (rank_ == 0) {
      listen_fd_ = socket(AF_UNIX, SOCK_STREAM, 0);
      if (listen_fd_ < 0 || bind(listen_fd_, reinterpret_cast<sockaddr*>(&addr_), len_) != 0 ||
          listen(listen_fd_, world_) != 0) {
        *err = std::string("rendezvous: bind/listen failed: ") + std::strerror(errno);
        return false;
      }
      const auto accept_deadline = std::chrono::steady_clock::now() + std::chrono::seconds(timeout_s());
      for (int n = 1; n < world_; ++n) {
        // bounded: a rank that failed before reaching the rendezvous must not hang rank 0
        pollfd pf{listen_fd_, POLLIN, 0};
        const auto left = std::chrono::duration_cast<std::chrono::milliseconds>(
            accept_deadline - std::chrono::steady_clock::now()).count();
        if (left <= 0 || poll(&pf, 1, static_cast<int>(left)) <= 0) {
          *err = "rendezvous: timed out waiting for peers to connect";
          return false;
        }
        const int fd = accept(listen_fd_, nullptr, nullptr);
        if (fd >= 0) set_timeouts(fd);
        int32_t peer = -1;
        if (fd < 0 || !read_all(fd, &peer, sizeof(peer)) || peer <= 0 || peer >= world_ || peers_[peer] >= 0) {
          *err = "rendezvous: bad peer handshake";
          if (fd >= 0) close(fd);
          return false;
        }
        peers_[peer] = fd;
      }
      return true;
    }
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(timeout_s());
    while (true) {
      const int fd = socket(AF_UNIX, SOCK_STREAM, 0);
      if (fd >= 0 && connect(fd, reinterpret_cast<sockaddr*>(&addr_), len_) == 0) {
        set_timeouts(fd);
        const int32_t me = rank_;
        if (!write_all(fd, &me, sizeof(me))) {
          close(fd);
          *err = "rendezvous: handshake write failed";
          return false;
        }
        peers_[0] = fd;
        return true;
      }
      if (fd >= 0) close(fd);
      if (std::chrono::steady_clock::now() > deadline) {
        *err = "rendezvous: timed out connecting to rank 0";
        return false;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }

  // rank 0 sends `fd` to every rank; others return the received descriptor.
  bool broadcast_fd(int fd, int* out, std::string* err) {
    if (rank_ == 0) {
      for (int r = 1; r < world_; ++r) {
        if (!send_fd(peers_[r], fd)) {
          *err = "rendezvous: sendmsg(SCM_RIGHTS) failed";
          return false;
        }
      }
      *out = fd;
      return true;
    }
    *out = recv_fd(peers_[0]);
    if (*out < 0) {
      *err = "rendezvous: recvmsg(SCM_RIGHTS) failed";
      return false;
    }
    return true;
  }

  bool barrier(std::string* err) {
    if (world_ == 1) return true;
    char b = 1;
    if (rank_ == 0) {
      for (int r = 1; r < world_; ++r)
        if (!read_all(peers_[r], &b, 1)) return fail_msg(err, "rendezvous: barrier read failed");
      for (int r = 1; r < world_; ++r)
        if (!write_all(peers_[r], &b, 1)) return fail_msg(err, "rendezvous: barrier write failed");
      return true;
    }
    if (!write_all(peers_[0], &b, 1) || !read_all(peers_[0], &b, 1))
      return fail_msg(err, "rendezvous: barrier with rank 0 failed");
    return true;
  }

  // Every rank contributes n bytes; all ranks receive the rank-ordered table.
  bool allgather(const void* mine, size_t n, void* all, std::string* err) {
    char* table = static_cast<char*>(all);
    std::memcpy(table + static_cast<size_t>(rank_) * n, mine, n);
    if (world_ == 1) return true;
    if (rank_ == 0) {
      for (int r = 1; r < world_; ++r)
        if (!read_all(peers_[r], table + static_cast<size_t>(r) * n, n))
          return fail_msg(err, "rendezvous: allgather read failed");
      for (int r = 1; r < world_; ++r)
        if (!write_all(peers_[r], table, n * world_)) return fail_msg(err, "rendezvous: allgather write failed");
      return true;
    }
    if (!write_all(peers_[0], mine, n) || !read_all(peers_[0], table, n * world_))
      return fail_msg(err, "rendezvous: allgather with rank 0 failed");
    return true;
  }

 private:
  // Bound of every rendezvous wait, seconds (TW_RENDEZVOUS_TIMEOUT_S overrides).
  static int timeout_s() {
    static const int t = [] {
      const char* e = std::getenv("TW_RENDEZVOUS_TIMEOUT_S");
      const int v = e ? std::atoi(e) : 120;
      return v > 0 ? v : 120;
    }();
    return t;
  }
  // Every blocking read/write on a rendezvous socket gives up after the same
  // bound, so a peer stuck outside the rendezvous surfaces as an error.
  static void set_timeouts(int fd) {
    timeval tv{timeout_s(), 0};
    setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
    setsockopt(fd, SOL_SOCKET, SO_SNDTIMEO, &tv, sizeof(tv));
  }
  static bool fail_msg(std::string* err, const char* m) {
    *err = m;
    return false;
  }
  static bool read_all(int fd, void* p, size_t n) {
    char* c = static_cast<char*>(p);
    while (n) {
      const ssize_t k = read(fd, c, n);
      if (k <= 0) return false;
      c += k;
      n -= static_cast<size_t>(k);
    }
    return true;
  }
  static bool write_all(int fd, const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    while (n) {
      const ssize_t k = write(fd, c, n);
      if (k <= 0) return false;
      c += k;
      n -= static_cast<size_t>(k);
    }
    return true;
  }
  static bool send_fd(int sock, int fd) {
    char payload = 'F';
    iovec iov{&payload, 1};
    alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))];
    msghdr msg{};
    msg.msg_iov = &iov;
    msg.msg_iovlen = 1;
    msg.msg_control = ctrl;
    msg.msg_controllen = sizeof(ctrl);
    cmsghdr* c = CMSG_FIRSTHDR(&msg);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int));
    std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
    return sendmsg(sock, &msg, 0) == 1;
  }
  static int recv_fd(int sock) {
    char payload = 0;
    iovec iov{&payload, 1};
    alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))];
    msghdr msg{};
    msg.msg_iov = &iov;
    msg.msg_iovlen = 1;
    msg.msg_control = ctrl;
    msg.msg_controllen = sizeof(ctrl);
    if (recvmsg(sock, &msg, 0) != 1) return -1;
    cmsghdr* c = CMSG_FIRSTHDR(&msg);
    if (!c || c->cmsg_type != SCM_RIGHTS) return -1;
    int fd = -1;
    std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
    return fd;
  }

  int world_, rank_;
  int listen_fd_ = -1;
  std::vector<int> peers_;
  sockaddr_un addr_;
  socklen_t len_ = 0;
};

tw_status create_nvls_mp(tw_comm* c, int rank, const char* id) {
  const Driver& d = driver();
  if (!d.ok) return fail(TW_ERR_UNSUPPORTED, "NVLS: driver entry points unavailable");
  RankBuffers& rb = c->ranks[rank];
  int mcs = 0;
  if (d.getAttr(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, rb.device) != CUDA_SUCCESS || !mcs)
    return fail(TW_ERR_UNSUPPORTED, "NVLS: device lacks multicast support");
  CUmulticastObjectProp mprop = {};
  mprop.numDevices = static_cast<unsigned>(c->world);
  mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mprop.size = 1;
  size_t mgran = 0, agran = 0;
  CUresult r = d.mcGranularity(&mgran, &mprop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastGetGranularity: " + cu_str(r));
  CUmemAllocationProp aprop = {};
  aprop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  aprop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  aprop.location.id = rb.device;
  aprop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  r = d.memGranularity(&agran, &aprop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMemGetAllocationGranularity: " + cu_str(r));
  const size_t gran = std::max(mgran, agran);
  c->region = round_up(std::max<size_t>(c->bytes, 1), gran);
  c->total = 3 * c->region + gran;
  mprop.size = c->total;

  Rendezvous rv(id, c->world, rank);
  std::string err;
  if (!rv.connect_all(&err)) return fail(TW_ERR_CONFIG, err);
  int fd = -1;
  if (rank == 0) {
    r = d.mcCreate(&c->mc, &mprop);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastCreate: " + cu_str(r));
    r = d.exportHandle(&fd, c->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMemExportToShareableHandle: " + cu_str(r));
  }
  int got = -1;
  if (!rv.broadcast_fd(fd, &got, &err)) return fail(TW_ERR_CONFIG, err);
  if (rank != 0) {
    r = d.importHandle(&c->mc, reinterpret_cast<void*>(static_cast<uintptr_t>(got)),
                       CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(got);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMemImportFromShareableHandle: " + cu_str(r));
  } else {
    close(fd);
  }
  r = d.mcAddDevice(c->mc, rb.device);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastAddDevice: " + cu_str(r));
  if (!rv.barrier(&err)) return fail(TW_ERR_CONFIG, err);  // all devices added before any bind
  r = d.memCreate(&rb.phys, c->total, &aprop, 0);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "cuMemCreate: " + cu_str(r));
  r = d.mcBindMem(c->mc, 0, rb.phys, 0, c->total, 0);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastBindMem: " + cu_str(r));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = rb.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = d.addrReserve(&rb.uc_base, c->total, gran, 0, 0);
  if (r == CUDA_SUCCESS) r = d.memMap(rb.uc_base, c->total, 0, rb.phys, 0);
  if (r == CUDA_SUCCESS) r = d.memSetAccess(rb.uc_base, c->total, &acc, 1);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "unicast map: " + cu_str(r));
  r = d.addrReserve(&rb.mc_base, c->total, gran, 0, 0);
  if (r == CUDA_SUCCESS) r = d.memMap(rb.mc_base, c->total, 0, c->mc, 0);
  if (r == CUDA_SUCCESS) r = d.memSetAccess(rb.mc_base, c->total, &acc, 1);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "multicast map: " + cu_str(r));
  char* uc = reinterpret_cast<char*>(rb.uc_base);
  char* mcp = reinterpret_cast<char*>(rb.mc_base);
  for (int b = 0; b < 3; ++b) {
    rb.buf[b] = uc + b * c->region;
    rb.mc_buf[b] = mcp + b * c->region;
  }
  rb.pad = reinterpret_cast<uint32_t*>(uc + 3 * c->region);
  rb.mc_pad = reinterpret_cast<uint32_t*>(mcp + 3 * c->region);
  rb.gen = reinterpret_cast<uint32_t*>(uc + 3 * c->region + kPadGenOffset);
  rb.err = reinterpret_cast<int*>(uc + 3 * c->region + kPadErrOffset);
  cudaError_t e = cudaMemset(uc + 3 * c->region, 0, kPadBytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "zero signal pad");
  if (!rv.barrier(&err)) return fail(TW_ERR_CONFIG, err);  // every pad zeroed before any signal
  return TW_OK;
}

// PEER transport across processes: each rank cudaMallocs its buffers and
// shares a cudaIpcMemHandle; peers map it (NVLink P2P loads/stores).
tw_status create_peer_mp(tw_comm* c, int rank, const std::string& id) {
  RankBuffers& rb = c->ranks[rank];
  c->region = round_up(std::max<size_t>(c->bytes, 1), 256);
  c->total = 3 * c->region + kPadBytes;
  char* base = nullptr;
  cudaError_t e = cudaMalloc(&base, c->total);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(comm buffers)");
  rb.owns_cuda_malloc = true;
  for (int b = 0; b < 3; ++b) rb.buf[b] = base + b * c->region;
  rb.pad = reinterpret_cast<uint32_t*>(base + 3 * c->region);
  rb.gen = reinterpret_cast<uint32_t*>(base + 3 * c->region + kPadGenOffset);
  rb.err = reinterpret_cast<int*>(base + 3 * c->region + kPadErrOffset);
  e = cudaMemset(base + 3 * c->region, 0, kPadBytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "zero signal pad");
  cudaIpcMemHandle_t mine;
  e = cudaIpcGetMemHandle(&mine, base);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  Rendezvous rv(id, c->world, rank);
  std::string err;
  if (!rv.connect_all(&err)) return fail(TW_ERR_CONFIG, err);
  std::vector<cudaIpcMemHandle_t> table(c->world);
  if (!rv.allgather(&mine, sizeof(mine), table.data(), &err)) return fail(TW_ERR_CONFIG, err);
  for (int q = 0; q < c->world; ++q) {
    if (q == rank) continue;
    void* peer = nullptr;
    e = cudaIpcOpenMemHandle(&peer, table[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle (no P2P path between the GPUs?)");
    RankBuffers& pb = c->ranks[q];
    pb.ipc_base = peer;
    char* pbase = static_cast<char*>(peer);
    for (int b = 0; b < 3; ++b) pb.buf[b] = pbase + b * c->region;
    pb.pad = reinterpret_cast<uint32_t*>(pbase + 3 * c->region);
    pb.gen = reinterpret_cast<uint32_t*>(pbase + 3 * c->region + kPadGenOffset);
    pb.err = reinterpret_cast<int*>(pbase + 3 * c->region + kPadErrOffset);
  }
  if (!rv.barrier(&err)) return fail(TW_ERR_CONFIG, err);  // every pad zeroed and mapped before any signal
  return TW_OK;
}

}  // namespace
}  // namespace tw

using namespace tw;

extern "C" {

tw_status tw_comm_create_mp(int world, int rank, int device, size_t buffer_bytes, const char* rendezvous_id,
                            tw_transport transport, tw_comm_t* out) {
  clear_error();
  if (!out) return fail(TW_ERR_CONFIG, "comm_create_mp: null output");
  *out = nullptr;
  if (world < 2 || world > 8) return fail(TW_ERR_CONFIG, "comm_create_mp: world must be in [2, 8]");
  if (rank < 0 || rank >= world) return fail(TW_ERR_CONFIG, "comm_create_mp: rank out of range");
  if (!rendezvous_id || !*rendezvous_id) return fail(TW_ERR_CONFIG, "comm_create_mp: empty rendezvous id");
  if (transport != TW_TRANSPORT_AUTO && transport != TW_TRANSPORT_NVLS && transport != TW_TRANSPORT_PEER)
    return fail(TW_ERR_CONFIG, "comm_create_mp: transport must be AUTO, NVLS or PEER");
  const int ndev = tw_device_count();
  if (ndev == 0) return fail(TW_ERR_CUDA, "comm_create_mp: no CUDA device visible");
  if (device < 0 || device >= ndev) return fail(TW_ERR_CONFIG, "comm_create_mp: device out of range");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  auto fresh = [&](tw_transport t) {
    tw_comm* c = new tw_comm();
    c->world = world;
    c->bytes = buffer_bytes;
    c->transport = t;
    c->local_rank = rank;
    c->ranks.resize(world);
    c->ranks[rank].device = device;
    return c;
  };
  tw_comm* c = nullptr;
  tw_status st = TW_ERR_UNSUPPORTED;
  std::string why;
  if (transport != TW_TRANSPORT_PEER) {
    c = fresh(TW_TRANSPORT_NVLS);
    st = create_nvls_mp(c, rank, rendezvous_id);
    if (st != TW_OK) {
      why = tw_last_error();
      destroy_comm(c);
      c = nullptr;
    }
  }
  // AUTO: every rank fails NVLS together (each failure closes the rendezvous
  // sockets its peers block on), then all retry on the PEER transport.
  if (st != TW_OK && transport != TW_TRANSPORT_NVLS) {
    c = fresh(TW_TRANSPORT_PEER);
    st = create_peer_mp(c, rank, std::string(rendezvous_id) + ":peer");
    if (st != TW_OK) {
      why += (why.empty() ? "" : "; ") + std::string(tw_last_error());
      destroy_comm(c);
      c = nullptr;
    }
  }
  cudaSetDevice(prev);
  if (st != TW_OK) return fail(st, why);
  *out = c;
  return TW_OK;
}

tw_status tw_fused_allreduce_rmsnorm(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset,
                                     const int64_t* shard_ranges, void* residual_shard, const float* weight, float eps,
                                     tw_dtype dtype, int sm_budget, unsigned flags, void* stream) {
  clear_error();
  if (!comm) return fail(TW_ERR_CONFIG, "fused_allreduce_rmsnorm: null communicator");
  if (comm->local_rank < 0)
    return fail(TW_ERR_CONFIG, "fused_allreduce_rmsnorm: single-process communicator, use the _group call");
  const int W = comm->world, r = comm->local_rank;
  std::vector<void*> res(W, nullptr), strs(W, nullptr);
  std::vector<const float*> wts(W, nullptr);
  res[r] = residual_shard;
  wts[r] = weight;
  strs[r] = stream;
  return comm_launch(comm, T, H, token_offset, shard_ranges, res.data(), wts.data(), eps, dtype, sm_budget, flags,
                     strs.data(), true);
}

tw_status tw_allreduce(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset, tw_dtype dtype, int sm_budget,
                       void* stream) {
  clear_error();
  if (!comm) return fail(TW_ERR_CONFIG, "allreduce: null communicator");
  if (comm->local_rank < 0) return fail(TW_ERR_CONFIG, "allreduce: single-process communicator, use the _group call");
  std::vector<void*> strs(comm->world, nullptr);
  strs[comm->local_rank] = stream;
  return comm_launch(comm, T, H, token_offset, nullptr, nullptr, nullptr, 0.0f, dtype, sm_budget, 0u, strs.data(),
                     false);
}

tw_status tw_rendezvous_exchange_fd(const char* rendezvous_id, int world, int rank, int fd, int* fd_out) {
  clear_error();
  if (!rendezvous_id || !fd_out || world < 1 || rank < 0 || rank >= world)
    return fail(TW_ERR_CONFIG, "rendezvous_exchange_fd: bad arguments");
  Rendezvous rv(rendezvous_id, world, rank);
  std::string err;
  if (!rv.connect_all(&err) || !rv.broadcast_fd(fd, fd_out, &err) || !rv.barrier(&err))
    return fail(TW_ERR_CONFIG, err);
  return TW_OK;
}

}  // extern "C"
