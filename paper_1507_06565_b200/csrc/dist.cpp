// x-slab multi-GPU driver in C++ (DESIGN.md §8): the C-ABI
// counterpart of a porolb::Simulation spread over P GPUs.  The paper's
// communication-reducing ghost exchange: slab r owns global columns
// [x0_r, x1_r); per step each face sends exactly the 5 post-collision PDFs
// whose velocity enters the neighbour ({1,7,9,11,13} to the right,
// {2,8,10,12,14} to the left), double-buffered by step parity.
//
// Three transports behind one schedule:
//   * NCCL, one rank per process (pgpu_dist_create_nccl).  libnccl is
//     resolved with dlopen at run time, so the library has no link-time NCCL
//     dependency and shares the copy torch.distributed already loaded.
//   * local, every slab in this process (pgpu_dist_create_local), on any mix
//     of devices, exchanged with peer copies (NVLink on a multi-GPU node).
//   * IPC, one rank per process on one node (pgpu_dist_create_ipc): the
//     ranks map each other's ghost buffers (CUDA IPC) and the edge-column
//     kernel STORES its 5 outgoing PDFs per face straight into the
//     neighbours' ghost buffers over NVLink -- the exchange is fused into the
//     sweep, no copy or send/recv kernel.  Ordering across processes:
//     interprocess CUDA events (stream waits, never a spinning kernel) plus a
//     host handshake in POSIX shared memory that makes each wait see the
//     right record; the global observables reduce through the same shared
//     memory in rank order.
// Per step and rank, on two streams (the simulation's own = "main", and a
// high-priority "edge" stream):
//   edge : wait(interior of step n-1) -> edge columns (pgpu part 0: they alone
//          read ghosts and fill the send buffers) -> exchange
//   main : wait(edge columns of step n-1) -> interior columns (part 1)
// so the exchange of step n overlaps the interior of step n; interior cells
// never read ghosts.  In NCCL mode the steady-state schedule (two steps, which
// return buffers and ghost parity to the same state) is captured once in a
// CUDA graph and replayed, so no per-step host work remains on the path.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>  // types only: the entry points are resolved with dlopen
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <exception>
#include <chrono>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sim_impl.h"

namespace {

// ---- NCCL through dlopen ------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  std::string error;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) {
      api.error = std::string("NCCL not found (dlopen libnccl.so.2: ") + dlerror() + ")";
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(api.h, n);
      if (!p && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + n;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.error.empty()) throw CudaError(api.error);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    std::ostringstream os;
    os << what << " failed: " << nccl().GetErrorString(r);
    throw CudaError(os.str());
  }
}

// ---- host channel of the IPC transport (POSIX shared memory, one node) -------
constexpr int kMaxIpcRanks = 64;
struct ShmHeader {
  std::atomic<uint64_t> edges[kMaxIpcRanks];  // edge parts recorded by each rank
  std::atomic<uint64_t> bar_count;
  std::atomic<uint64_t> bar_gen;
  std::atomic<uint64_t> attached;
  int32_t world, slot_doubles;
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "process-shared atomics");

struct ShmChannel {
  std::string name;
  bool owner = false;
  int world = 0;
  size_t bytes = 0;
  ShmHeader* h = nullptr;
  double* slots = nullptr;  // world x slot_doubles reduction slots

  static size_t size_for(int world, int slot_doubles) {
    return sizeof(ShmHeader) + sizeof(double) * (size_t)world * slot_doubles;
  }
  void create(const std::string& nm, int w, int slot_doubles) {
    name = nm;
    owner = true;
    world = w;
    bytes = size_for(w, slot_doubles);
    shm_unlink(name.c_str());
    const int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw CudaError("shm_open(create) failed for " + name);
    if (ftruncate(fd, (off_t)bytes) != 0) {
      close(fd);
      throw CudaError("ftruncate failed for " + name);
    }
    map(fd);
    std::memset(static_cast<void*>(h), 0, bytes);
    h->world = w;
    h->slot_doubles = slot_doubles;
  }
  void open_existing(const std::string& nm, int w, int slot_doubles) {
    name = nm;
    world = w;
    bytes = size_for(w, slot_doubles);
    const int fd = shm_open(name.c_str(), O_RDWR, 0600);
    if (fd < 0) throw CudaError("shm_open(attach) failed for " + name);
    map(fd);
  }
  void map(int fd) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw CudaError("mmap of the IPC channel failed");
    h = static_cast<ShmHeader*>(p);
    slots = reinterpret_cast<double*>(static_cast<char*>(p) + sizeof(ShmHeader));
  }
  ~ShmChannel() {
    if (h) munmap(static_cast<void*>(h), bytes);
    if (owner) shm_unlink(name.c_str());
  }
  // host spin with yields (the waits are short: a neighbour issuing a step)
  template <class Pred>
  static void spin(Pred done) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; !done(); ++i) {
      if (i > 64) std::this_thread::yield();
      if ((i & 0xffff) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
        throw CudaError("IPC transport: a neighbour rank stopped issuing steps");
    }
  }
  void wait_edges(int rank, uint64_t n) {
    spin([&] { return h->edges[rank].load(std::memory_order_acquire) >= n; });
  }
  void barrier() {
    const uint64_t g = h->bar_gen.load(std::memory_order_acquire);
    if (h->bar_count.fetch_add(1, std::memory_order_acq_rel) + 1 == (uint64_t)world) {
      h->bar_count.store(0, std::memory_order_relaxed);
      h->bar_gen.store(g + 1, std::memory_order_release);
    } else {
      spin([&] { return h->bar_gen.load(std::memory_order_acquire) != g; });
    }
  }
};

// what one rank publishes to the others (pgpu_dist_ipc_export)
struct IpcBlob {
  cudaIpcMemHandle_t halo;
  cudaIpcEventHandle_t ev[2];
  int32_t rank, world, device;
  int64_t halo_n;
  char shm[64];
};

struct DistPeer {  // a neighbour's ghost buffers and edge events as mapped here
  double* base = nullptr;  // opened IPC allocation (nullptr: this rank itself)
  double* recv_lo[2] = {nullptr, nullptr};
  double* recv_hi[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool own = false;  // events/pointers are this process's (world 1, or the same peer twice)
};

struct DistRank {
  pgpu_sim* sim = nullptr;
  int rank = 0;
  cudaStream_t edge = nullptr;
  double* halo = nullptr;  // send_lo | send_hi | recv_lo[2] | recv_hi[2]
  double* send_lo = nullptr;
  double* send_hi = nullptr;
  double* recv_lo[2] = {nullptr, nullptr};
  double* recv_hi[2] = {nullptr, nullptr};
  cudaEvent_t ev_main = nullptr, ev_copy = nullptr, ev_join = nullptr;
  cudaEvent_t ev_edge[2] = {nullptr, nullptr};
  int parity = 0;         // which ev_edge the current step records
  bool have_prev = false;  // ev_edge[1 - parity] holds the previous step's edge part
  bool copied = false;     // local mode: neighbours' copies of step n-1 read our sends
};

}  // namespace

struct pgpu_dist {
  int world = 1;
  bool use_nccl = false;
  bool use_ipc = false;
  // IPC transport
  std::unique_ptr<ShmChannel> shm;
  DistPeer peer_l, peer_r;
  bool connected = false;
  uint64_t nedge = 0;  // edge parts issued by this rank
  std::vector<DistRank> ranks;  // NCCL: this process's rank only
  ncclComm_t comm = nullptr;
  int64_t halo_n = 0;
  double* d_red = nullptr;  // NCCL reductions (nz + 2 doubles)
  bool graphs = true;
  // two-step graphs keyed by the state they were captured in (sweep buffer
  // parity `cur`, ghost parity): the kernels' pointers are baked in, and an
  // observable or an odd number of eager steps changes the parities
  cudaGraphExec_t gexec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  cudaStream_t gstream = nullptr;
  int64_t glaunches = 0;  // kernels per graph replay (two steps)

  void drop_graphs() {
    for (auto& row : gexec)
      for (auto& g : row)
        if (g) {
          cudaGraphExecDestroy(g);
          g = nullptr;
        }
  }

  ~pgpu_dist() {
    drop_graphs();
    for (DistPeer* pr : {&peer_l, &peer_r}) {
      if (pr->own) continue;
      for (cudaEvent_t& e : pr->ev)
        if (e) {
          cudaEventDestroy(e);
          e = nullptr;
        }
      if (pr->base && !(pr == &peer_r && peer_r.base == peer_l.base)) cudaIpcCloseMemHandle(pr->base);
      pr->base = nullptr;
    }
    for (auto& r : ranks) {
      cudaSetDevice(r.sim->device);
      cudaStreamSynchronize(r.edge);
      cudaStreamSynchronize(r.sim->stream);
      for (cudaEvent_t e : {r.ev_main, r.ev_copy, r.ev_join, r.ev_edge[0], r.ev_edge[1]})
        if (e) cudaEventDestroy(e);
      if (r.edge) cudaStreamDestroy(r.edge);
      cudaFree(r.halo);
      // the simulation may outlive the driver: no dangling halo pointers
      r.sim->send_lo = r.sim->send_hi = nullptr;
      r.sim->recv_lo[0] = r.sim->recv_lo[1] = r.sim->recv_hi[0] = r.sim->recv_hi[1] = nullptr;
    }
    if (d_red) cudaFree(d_red);
    if (comm) nccl().CommDestroy(comm);
  }

  // ---- one step, issued on the ranks' streams -------------------------------
  // The simulation's kernels for a part go to `st` (pgpu_step_part_on logic).
  static void part(DistRank& r, int which, cudaStream_t st) {
    pgpu_sim* s = r.sim;
    const cudaStream_t keep = s->stream;
    s->stream = st;
    try {
      if (which == 0) {
        if (!s->post) {
          s->k0();  // collide-only, fills the send buffers
          s->pending = 1;
        } else {
          s->k1(1);  // edge columns (lattice.cuh PART_EDGES)
          s->pending = 2;
        }
      } else if (s->pending == 2) {
        s->k1(2);  // interior columns (PART_INTERIOR)
      }
    } catch (...) {
      s->stream = keep;
      throw;
    }
    s->stream = keep;
  }

  static void finish(DistRank& r) {
    pgpu_sim* s = r.sim;
    if (s->pending == 1)
      s->post = true;
    else
      s->cur = 1 - s->cur;
    s->pending = 0;
    s->ghost_cur = 1 - s->ghost_cur;
    ++s->steps;
  }

  // IPC: the edge part stores straight into the neighbours' ghost buffers
  void issue_step_ipc() {
    DistRank& r = ranks[0];
    pgpu_sim* s = r.sim;
    CK(cudaSetDevice(s->device));
    const int W = world;
    const int left = (r.rank + W - 1) % W, right = (r.rank + 1) % W;
    const int pn = 1 - s->ghost_cur;  // the ghost parity the next step reads
    CK(cudaEventRecord(r.ev_main, s->stream));
    CK(cudaStreamWaitEvent(r.edge, r.ev_main, 0));
    if (nedge > 0) {
      // the neighbours' edge parts of the previous step: they wrote the ghosts
      // this step reads, and finished reading the ghost parity we overwrite
      Nvtx nv("IPC wait for the neighbours' previous edge parts");
      shm->wait_edges(left, nedge);
      shm->wait_edges(right, nedge);
      const int pp = (int)((nedge - 1) & 1);
      CK(cudaStreamWaitEvent(r.edge, peer_l.ev[pp], 0));
      if (peer_r.ev[pp] != peer_l.ev[pp]) CK(cudaStreamWaitEvent(r.edge, peer_r.ev[pp], 0));
    }
    // my x = 0 face feeds the left neighbour's x = nx ghost, x = nx-1 the right's x = -1
    s->send_lo = peer_l.recv_hi[pn];
    s->send_hi = peer_r.recv_lo[pn];
    part(r, 0, r.edge);
    CK(cudaEventRecord(r.ev_edge[nedge & 1], r.edge));
    ++nedge;
    shm->h->edges[r.rank].store(nedge, std::memory_order_release);
    // interior columns (after the previous step's edge columns)
    if (r.have_prev) CK(cudaStreamWaitEvent(s->stream, r.ev_edge[(nedge - 2) & 1], 0));
    part(r, 1, s->stream);
    finish(r);
    r.have_prev = true;
    r.parity = (int)(nedge & 1);
  }

  void issue_step() {
    if (use_ipc) {
      issue_step_ipc();
      return;
    }
    const int W = world;
    const size_t bytes = sizeof(double) * (size_t)halo_n;
    // edge columns (after the previous interior; local mode: after the
    // neighbours' copies of our previous sends)
    for (size_t i = 0; i < ranks.size(); ++i) {
      DistRank& r = ranks[i];
      CK(cudaSetDevice(r.sim->device));
      CK(cudaEventRecord(r.ev_main, r.sim->stream));
      CK(cudaStreamWaitEvent(r.edge, r.ev_main, 0));
      if (!use_nccl && r.copied) {
        CK(cudaStreamWaitEvent(r.edge, ranks[(i + W - 1) % W].ev_copy, 0));
        CK(cudaStreamWaitEvent(r.edge, ranks[(i + 1) % W].ev_copy, 0));
      }
      part(r, 0, r.edge);
      CK(cudaEventRecord(r.ev_edge[r.parity], r.edge));
    }
    // exchange: fill the ghost parity the next step reads
    Nvtx nv("halo exchange (5 PDFs per face)");
    if (use_nccl) {
      DistRank& r = ranks[0];
      const int p = 1 - r.sim->ghost_cur;
      const int left = (r.rank + W - 1) % W, right = (r.rank + 1) % W;
      NcclApi& n = nccl();
      // per-peer order matches between neighbours (NCCL matches sends and
      // receives to one peer in issue order): my send_lo is the left
      // neighbour's recv_hi, my send_hi the right neighbour's recv_lo
      nck(n.GroupStart(), "ncclGroupStart");
      nck(n.Send(r.send_lo, (size_t)halo_n, ncclDouble, left, comm, r.edge), "ncclSend");
      nck(n.Send(r.send_hi, (size_t)halo_n, ncclDouble, right, comm, r.edge), "ncclSend");
      nck(n.Recv(r.recv_hi[p], (size_t)halo_n, ncclDouble, right, comm, r.edge), "ncclRecv");
      nck(n.Recv(r.recv_lo[p], (size_t)halo_n, ncclDouble, left, comm, r.edge), "ncclRecv");
      nck(n.GroupEnd(), "ncclGroupEnd");
    } else {
      for (int i = 0; i < W; ++i) {
        DistRank& r = ranks[i];
        DistRank& L = ranks[(i + W - 1) % W];
        DistRank& R = ranks[(i + 1) % W];
        const int p = 1 - r.sim->ghost_cur;
        CK(cudaSetDevice(r.sim->device));
        CK(cudaStreamWaitEvent(r.edge, L.ev_edge[L.parity], 0));
        CK(cudaStreamWaitEvent(r.edge, R.ev_edge[R.parity], 0));
        CK(cudaMemcpyPeerAsync(r.recv_hi[p], r.sim->device, R.send_lo, R.sim->device, bytes, r.edge));
        CK(cudaMemcpyPeerAsync(r.recv_lo[p], r.sim->device, L.send_hi, L.sim->device, bytes, r.edge));
        CK(cudaEventRecord(r.ev_copy, r.edge));
        r.copied = true;
      }
    }
    // interior columns (after the previous step's edge columns)
    for (DistRank& r : ranks) {
      CK(cudaSetDevice(r.sim->device));
      if (r.have_prev) CK(cudaStreamWaitEvent(r.sim->stream, r.ev_edge[1 - r.parity], 0));
      part(r, 1, r.sim->stream);
      finish(r);
      r.have_prev = true;
      r.parity = 1 - r.parity;
    }
  }

  // main waits for edge: everything issued so far is ordered on the sims' streams
  void join() {
    for (DistRank& r : ranks) {
      CK(cudaSetDevice(r.sim->device));
      CK(cudaEventRecord(r.ev_join, r.edge));
      CK(cudaStreamWaitEvent(r.sim->stream, r.ev_join, 0));
    }
  }

  void capture() {  // NCCL mode, post state: a graph of two steps
    DistRank& r = ranks[0];
    pgpu_sim* s = r.sim;
    cudaGraphExec_t& gexec = this->gexec[s->cur][s->ghost_cur];
    join();
    r.have_prev = false;  // consecutive replays are ordered by the stream
    const int64_t l0 = s->launches;
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    try {
      issue_step();
      issue_step();
      CK(cudaEventRecord(r.ev_join, r.edge));
      CK(cudaStreamWaitEvent(s->stream, r.ev_join, 0));
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(s->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s->stream, &g);
    if (e != cudaSuccess) throw CudaError(std::string("graph capture failed: ") + cudaGetErrorString(e));
    const cudaError_t ie = cudaGraphInstantiate(&gexec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) throw CudaError(std::string("graph instantiate failed: ") + cudaGetErrorString(ie));
    glaunches = s->launches - l0;
    gstream = s->stream;
    // the capture advanced the host state by two steps; run them now
    CK(cudaGraphLaunch(gexec, s->stream));
    r.have_prev = false;
  }

  void step(int64_t n) {
    for (DistRank& r : ranks)
      if (r.sim->pending) throw ConfigError("split step in progress");
    for (int64_t i = 0; i < n;) {
      DistRank& r0 = ranks[0];
      const bool graphable = use_nccl && graphs && r0.sim->post && n - i >= 2;
      if (graphable) {
        if (gstream != r0.sim->stream) drop_graphs();  // pgpu_set_stream since the capture
        cudaGraphExec_t gexec = this->gexec[r0.sim->cur][r0.sim->ghost_cur];
        if (!gexec) {
          capture();
          i += 2;
          continue;
        }
        if (r0.have_prev) join();  // eager steps before: order them ahead of the replay
        r0.have_prev = false;
        CK(cudaGraphLaunch(gexec, r0.sim->stream));
        r0.sim->steps += 2;
        r0.sim->launches += glaunches;
        i += 2;
        continue;
      }
      issue_step();
      ++i;
    }
    join();
    if (use_ipc && nedge > 0) ipc_join();
  }

  // IPC: the simulation's stream also waits for the neighbours' last edge
  // parts -- they wrote the ghosts an observable (KP) or the next step reads
  void ipc_join() {
    DistRank& r = ranks[0];
    const int W = world;
    shm->wait_edges((r.rank + W - 1) % W, nedge);
    shm->wait_edges((r.rank + 1) % W, nedge);
    const int pp = (int)((nedge - 1) & 1);
    CK(cudaSetDevice(r.sim->device));
    CK(cudaStreamWaitEvent(r.sim->stream, peer_l.ev[pp], 0));
    if (peer_r.ev[pp] != peer_l.ev[pp]) CK(cudaStreamWaitEvent(r.sim->stream, peer_r.ev[pp], 0));
  }

  // ---- observables over the whole domain ---------------------------------------
  void allreduce(double* host, int count, ncclRedOp_t op) {
    DistRank& r = ranks[0];
    CK(cudaSetDevice(r.sim->device));
    CK(cudaMemcpyAsync(d_red, host, sizeof(double) * count, cudaMemcpyHostToDevice, r.sim->stream));
    nck(nccl().AllReduce(d_red, d_red, (size_t)count, ncclDouble, op, comm, r.sim->stream),
        "ncclAllReduce");
    CK(cudaMemcpyAsync(host, d_red, sizeof(double) * count, cudaMemcpyDeviceToHost, r.sim->stream));
    CK(cudaStreamSynchronize(r.sim->stream));
  }

  // per-plane sums of the stream-axis velocity (rank order on the host in
  // local mode) and per-plane fluid counts
  void plane_sums(int axis, std::vector<double>& sums, std::vector<double>& counts) {
    const int nz = ranks[0].sim->nz;
    sums.assign(nz, 0.0);
    counts.assign(nz, 0.0);
    for (DistRank& r : ranks) {
      std::vector<double> s;
      r.sim->plane_sums(axis, s);
      for (int z = 0; z < nz; ++z) {
        sums[z] += s[z];
        counts[z] += static_cast<double>(r.sim->plane_fluid_count[z]);
      }
    }
    if (use_nccl && world > 1) {
      allreduce(sums.data(), nz, ncclSum);
      allreduce(counts.data(), nz, ncclSum);
    }
    if (use_ipc && world > 1) {  // rank-order sums through the shared channel
      const int me = ranks[0].rank;
      double* slot = shm->slots + (size_t)me * (2 * nz + 2);
      std::memcpy(slot, sums.data(), sizeof(double) * nz);
      std::memcpy(slot + nz, counts.data(), sizeof(double) * nz);
      shm->barrier();
      for (int z = 0; z < nz; ++z) sums[z] = counts[z] = 0.0;
      for (int q = 0; q < world; ++q) {
        const double* o = shm->slots + (size_t)q * (2 * nz + 2);
        for (int z = 0; z < nz; ++z) {
          sums[z] += o[z];
          counts[z] += o[nz + z];
        }
      }
      shm->barrier();  // the slots may be reused
    }
  }

  void max_speed2(double& v2, bool& finite) {
    v2 = 0.0;
    finite = true;
    for (DistRank& r : ranks) {
      double a;
      bool f;
      r.sim->max_speed2(a, f);
      v2 = std::max(v2, a);
      finite = finite && f;
    }
    if (use_nccl && world > 1) {
      double h[2] = {v2, finite ? 0.0 : 1.0};
      allreduce(h, 2, ncclMax);
      v2 = h[0];
      finite = h[1] == 0.0;
    }
    if (use_ipc && world > 1) {
      const int nz = ranks[0].sim->nz;
      double* slot = shm->slots + (size_t)ranks[0].rank * (2 * nz + 2);
      slot[0] = v2;
      slot[1] = finite ? 0.0 : 1.0;
      shm->barrier();
      for (int q = 0; q < world; ++q) {
        const double* o = shm->slots + (size_t)q * (2 * nz + 2);
        v2 = std::max(v2, o[0]);
        finite = finite && o[1] == 0.0;
      }
      shm->barrier();
    }
  }

  // simulation.cpp:371-417 + profile.cpp:10-19 over the global domain
  void planar_profile(int axis, double* z_out, double* u_sup, double* u_int, double* eps_out,
                      double* u_norm, pgpu_profile_meta* meta) {
    pgpu_sim* s = ranks[0].sim;
    const int nz = s->nz;
    std::vector<double> sums, counts;
    plane_sums(axis, sums, counts);
    meta->n_planes = 0;
    meta->u_max = 0.0;
    meta->stream_axis = axis;
    meta->nu = s->params.nu;
    for (int i = 0; i < 3; ++i) meta->body_force[i] = s->params.body_force[i];
    if (s->has_lo && s->has_hi) {
      meta->z0 = s->lo;
      meta->height = s->hi - s->lo;
    } else {
      meta->z0 = 0.0;
      meta->height = nz;
    }
    int z_lo = nz, z_hi = -1;
    for (int z = 0; z < nz; ++z)
      if (counts[z] > 0.0) {
        z_lo = std::min(z_lo, z);
        z_hi = std::max(z_hi, z);
      }
    if (z_hi < 0) return;
    const double plane = static_cast<double>(s->global_nx) * s->ny;
    for (int z = z_lo; z <= z_hi; ++z) {
      const int i = z - z_lo;
      z_out[i] = z + 0.5;
      u_sup[i] = sums[z] / plane;
      u_int[i] = counts[z] > 0.0 ? sums[z] / counts[z] : 0.0;
      eps_out[i] = counts[z] / plane;
    }
    const int n = z_hi - z_lo + 1;
    meta->n_planes = n;
    double u_max = 0.0;
    for (int i = 0; i < n; ++i)
      if (std::abs(u_sup[i]) > std::abs(u_max)) u_max = u_sup[i];
    for (int i = 0; i < n; ++i) u_norm[i] = (u_max != 0.0) ? u_sup[i] / u_max : 0.0;
    meta->u_max = u_max;
  }
};

namespace {

void setup_rank(pgpu_dist* d, DistRank& r, bool ipc = false) {
  pgpu_sim* s = r.sim;
  if (!s->slab) throw ConfigError("multi-GPU runs need slab simulations (pgpu_voxelize_slab)");
  if (s->pending) throw ConfigError("split step in progress");
  CK(cudaSetDevice(s->device));
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // high priority: the edge part and the exchange are dispatched ahead of the
  // interior sweep's remaining blocks
  CK(cudaStreamCreateWithPriority(&r.edge, cudaStreamNonBlocking, hi));
  for (cudaEvent_t* e : {&r.ev_main, &r.ev_copy, &r.ev_join})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&r.ev_edge[0], &r.ev_edge[1]})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming | (ipc ? cudaEventInterprocess : 0u)));
  const int64_t n = d->halo_n;
  CK(cudaMalloc(&r.halo, sizeof(double) * 6 * (size_t)n));
  CK(cudaMemsetAsync(r.halo, 0, sizeof(double) * 6 * (size_t)n, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  r.send_lo = r.halo;
  r.send_hi = r.halo + n;
  r.recv_lo[0] = r.halo + 2 * n;
  r.recv_lo[1] = r.halo + 3 * n;
  r.recv_hi[0] = r.halo + 4 * n;
  r.recv_hi[1] = r.halo + 5 * n;
  s->send_lo = r.send_lo;
  s->send_hi = r.send_hi;
  s->recv_lo[0] = r.recv_lo[0];
  s->recv_lo[1] = r.recv_lo[1];
  s->recv_hi[0] = r.recv_hi[0];
  s->recv_hi[1] = r.recv_hi[1];
  s->drop_graphs();
}

}  // namespace

extern "C" {

int pgpu_dist_nccl_unique_id(uint8_t id[128]) {
  return guard([&] {
    if (!id) throw std::invalid_argument("null id");
    ncclUniqueId u;
    nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int pgpu_dist_create_nccl(pgpu_sim* sim, const uint8_t id[128], int32_t rank, int32_t world,
                          pgpu_dist** out) {
  return guard([&] {
    if (!sim || !id || !out) throw std::invalid_argument("null pointer");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) throw ConfigError("rank out of range");
    std::unique_ptr<pgpu_dist> d(new pgpu_dist());
    d->world = world;
    d->use_nccl = true;
    d->halo_n = 5 * (int64_t)sim->ny * sim->nz;
    d->ranks.resize(1);
    d->ranks[0].sim = sim;
    d->ranks[0].rank = rank;
    setup_rank(d.get(), d->ranks[0]);
    CK(cudaMalloc(&d->d_red, sizeof(double) * (size_t)(sim->nz + 2)));
    if (const char* e = std::getenv("PGPU_DIST_GRAPHS")) d->graphs = e[0] != '0';
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    CK(cudaSetDevice(sim->device));
    nck(nccl().CommInitRank(&d->comm, world, u, rank), "ncclCommInitRank");
    *out = d.release();
  });
}

int pgpu_dist_create_local(pgpu_sim* const* sims, int32_t world, pgpu_dist** out) {
  return guard([&] {
    if (!sims || !out || world < 1) throw std::invalid_argument("bad arguments");
    *out = nullptr;
    std::unique_ptr<pgpu_dist> d(new pgpu_dist());
    d->world = world;
    d->use_nccl = false;
    d->halo_n = 5 * (int64_t)sims[0]->ny * sims[0]->nz;
    d->ranks.resize(world);
    for (int i = 0; i < world; ++i) {
      if (!sims[i]) throw std::invalid_argument("null simulation");
      if (sims[i]->ny != sims[0]->ny || sims[i]->nz != sims[0]->nz)
        throw ConfigError("slabs must share ny and nz");
      d->ranks[i].sim = sims[i];
      d->ranks[i].rank = i;
      setup_rank(d.get(), d->ranks[i]);
    }
    // peer access between the slabs' devices (NVLink copies); same device: no-op
    for (int i = 0; i < world; ++i)
      for (int j = 0; j < world; ++j) {
        const int a = sims[i]->device, b = sims[j]->device;
        if (a == b) continue;
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, a, b));
        if (can) {
          CK(cudaSetDevice(a));
          const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
          cudaGetLastError();
        }
      }
    *out = d.release();
  });
}

int pgpu_dist_create_ipc(pgpu_sim* sim, int32_t rank, int32_t world, pgpu_dist** out) {
  return guard([&] {
    if (!sim || !out) throw std::invalid_argument("null pointer");
    *out = nullptr;
    if (world < 1 || world > kMaxIpcRanks || rank < 0 || rank >= world)
      throw ConfigError("rank out of range");
    std::unique_ptr<pgpu_dist> d(new pgpu_dist());
    d->world = world;
    d->use_ipc = true;
    d->halo_n = 5 * (int64_t)sim->ny * sim->nz;
    d->ranks.resize(1);
    d->ranks[0].sim = sim;
    d->ranks[0].rank = rank;
    setup_rank(d.get(), d->ranks[0], true);
    d->shm.reset(new ShmChannel());
    if (rank == 0) {
      static std::atomic<int> seq{0};
      const std::string nm = "/pgpu_dist_" + std::to_string((long)getpid()) + "_" +
                             std::to_string(seq.fetch_add(1));
      d->shm->create(nm, world, 2 * sim->nz + 2);
    }
    *out = d.release();
  });
}

int pgpu_dist_ipc_blob_size(int64_t* bytes) {
  return guard([&] {
    if (!bytes) throw std::invalid_argument("null pointer");
    *bytes = (int64_t)sizeof(IpcBlob);
  });
}

int pgpu_dist_ipc_export(pgpu_dist* d, void* blob) {
  return guard([&] {
    if (!d || !blob) throw std::invalid_argument("null pointer");
    if (!d->use_ipc) throw ConfigError("not an IPC driver");
    DistRank& r = d->ranks[0];
    CK(cudaSetDevice(r.sim->device));
    IpcBlob b;
    std::memset(&b, 0, sizeof(b));
    CK(cudaIpcGetMemHandle(&b.halo, r.halo));
    for (int i = 0; i < 2; ++i) CK(cudaIpcGetEventHandle(&b.ev[i], r.ev_edge[i]));
    b.rank = r.rank;
    b.world = d->world;
    b.device = r.sim->device;
    b.halo_n = d->halo_n;
    if (r.rank == 0) std::snprintf(b.shm, sizeof(b.shm), "%s", d->shm->name.c_str());
    std::memcpy(blob, &b, sizeof(b));
  });
}

// blobs: the `world` exported blobs in rank order
int pgpu_dist_ipc_connect(pgpu_dist* d, const void* blobs) {
  return guard([&] {
    if (!d || !blobs) throw std::invalid_argument("null pointer");
    if (!d->use_ipc || d->connected) throw ConfigError("not an unconnected IPC driver");
    DistRank& r = d->ranks[0];
    CK(cudaSetDevice(r.sim->device));
    const IpcBlob* all = static_cast<const IpcBlob*>(blobs);
    const int W = d->world;
    for (int q = 0; q < W; ++q)
      if (all[q].rank != q || all[q].world != W || all[q].halo_n != d->halo_n)
        throw ConfigError("IPC blobs do not describe this decomposition");
    if (r.rank != 0) d->shm->open_existing(all[0].shm, W, 2 * r.sim->nz + 2);
    const int left = (r.rank + W - 1) % W, right = (r.rank + 1) % W;
    const int64_t n = d->halo_n;
    auto open = [&](int q, DistPeer& pr, DistPeer* same) {
      double* base;
      if (q == r.rank) {
        pr.own = true;
        base = r.halo;
        pr.ev[0] = r.ev_edge[0];
        pr.ev[1] = r.ev_edge[1];
      } else if (same) {  // world 2: the left and right neighbours are one rank
        pr = *same;
        pr.own = true;  // owned (closed) through the other entry
        return;
      } else {
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, all[q].halo, cudaIpcMemLazyEnablePeerAccess));
        base = static_cast<double*>(p);
        pr.base = base;
        for (int i = 0; i < 2; ++i) CK(cudaIpcOpenEventHandle(&pr.ev[i], all[q].ev[i]));
      }
      pr.recv_lo[0] = base + 2 * n;
      pr.recv_lo[1] = base + 3 * n;
      pr.recv_hi[0] = base + 4 * n;
      pr.recv_hi[1] = base + 5 * n;
    };
    std::exception_ptr err;
    try {
      open(left, d->peer_l, nullptr);
      open(right, d->peer_r, right == left && left != r.rank ? &d->peer_l : nullptr);
    } catch (...) {
      err = std::current_exception();
    }
    d->shm->h->attached.fetch_add(1, std::memory_order_acq_rel);
    d->shm->barrier();  // every rank mapped its neighbours (or failed) before any step
    if (err) std::rethrow_exception(err);
    d->connected = true;
  });
}

int pgpu_dist_set_graphs(pgpu_dist* d, int32_t enable) {
  return guard([&] {
    if (!d) throw std::invalid_argument("null handle");
    d->graphs = enable != 0;
  });
}

int pgpu_dist_step(pgpu_dist* d, int64_t n) {
  return guard([&] {
    if (!d) throw std::invalid_argument("null handle");
    if (d->use_ipc && !d->connected) throw ConfigError("IPC driver not connected (pgpu_dist_ipc_connect)");
    if (n < 0) throw ConfigError("step count must be non-negative");
    d->step(n);
  });
}

int pgpu_dist_synchronize(pgpu_dist* d) {
  return guard([&] {
    if (!d) throw std::invalid_argument("null handle");
    for (DistRank& r : d->ranks) {
      CK(cudaSetDevice(r.sim->device));
      CK(cudaStreamSynchronize(r.edge));
      CK(cudaStreamSynchronize(r.sim->stream));
    }
  });
}

int pgpu_dist_plane_sums(pgpu_dist* d, int32_t axis, double* sums_nz) {
  return guard([&] {
    if (!d || !sums_nz) throw std::invalid_argument("null pointer");
    std::vector<double> s, c;
    d->plane_sums(axis, s, c);
    std::memcpy(sums_nz, s.data(), sizeof(double) * s.size());
  });
}

int pgpu_dist_max_speed2(pgpu_dist* d, double* vmax2, int32_t* finite) {
  return guard([&] {
    if (!d || !vmax2 || !finite) throw std::invalid_argument("null pointer");
    bool f;
    d->max_speed2(*vmax2, f);
    *finite = f ? 1 : 0;
  });
}

int pgpu_dist_planar_profile(pgpu_dist* d, int32_t axis, double* z, double* u_sup,
                             double* u_int, double* eps, double* u_norm, pgpu_profile_meta* meta) {
  return guard([&] {
    if (!d || !z || !u_sup || !u_int || !eps || !u_norm || !meta)
      throw std::invalid_argument("null pointer");
    if (axis < 0 || axis > 2) throw ConfigError("stream axis must be 0, 1 or 2");
    d->planar_profile(axis, z, u_sup, u_int, eps, u_norm, meta);
  });
}

int pgpu_dist_destroy(pgpu_dist* d) {
  return guard([&] { delete d; });
}

}  // extern "C"
