// dist.cpp -- sharded Chief: communicators, ownership, broadcast schedule,
// the communication loop of a rank and the result gather (see dist.hpp).
#include "dist.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <thread>
#include <mutex>
#include <stdexcept>

#include "jobs.hpp"

namespace gfq {

int Sharding::owner(const TaskNode& nd) const {
  switch (nd.kind) {
    case TaskKind::ClearDown:
      return owner_col(std::size_t(nd.c1));
    case TaskKind::Extend:
      return -1;
    case TaskKind::UpdateRow:
      return owner_col(std::size_t(nd.c2));
    case TaskKind::UpdateRowTrafo:
    case TaskKind::RowLengthen:
      return owner_trow(std::size_t(nd.c2));
    case TaskKind::Copy:
      return owner_col(std::size_t(nd.c1));
    case TaskKind::PreClearUp:
      return owner_col(std::size_t(nd.c2));
    case TaskKind::ClearUp:
      return -2;  // resolved by the output kind (R vs M), see owner_of()
    case TaskKind::UpdateRowW:
    case TaskKind::ClearUpRW:
    case TaskKind::ClearUpMW:
    case TaskKind::UpdateRowTrafoW:
      throw std::logic_error("fused (single-GPU) tasks cannot be sharded");
  }
  return -1;
}

namespace {
int owner_of(const Sharding& sh, const TaskGraph& g, const TaskNode& nd) {
  const int o = sh.owner(nd);
  if (o != -2) return o;
  return g.slot(nd.out[0]).key.kind == PkgKind::R ? sh.owner_col(std::size_t(nd.c2))
                                                   : sh.owner_trow(std::size_t(nd.c2));
}
}  // namespace

// ---------------------------------------------------------------- NCCL
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // an already-loaded libnccl (e.g. torch's) is reused by soname
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(a.h, "ncclCommInitRank"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(a.h, "ncclBroadcast"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(a.h, "ncclGetErrorString"));
    a.commSplit = reinterpret_cast<decltype(a.commSplit)>(dlsym(a.h, "ncclCommSplit"));
    if (!a.getUniqueId || !a.commInitRank || !a.broadcast || !a.commDestroy)
      throw std::runtime_error("libnccl.so.2 lacks the required symbols");
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " +
                             (nccl().getErrorString ? nccl().getErrorString(r) : "NCCL error"));
}

class NcclComm : public Comm {
 public:
  NcclComm(int world, int rank, const void* id128) : world_(world), rank_(rank) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    nccl_check(nccl().commInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  NcclComm(int world, int rank, ncclComm_t c) : world_(world), rank_(rank), comm_(c) {}
  std::shared_ptr<Comm> split_channel() override {
    // an independent communicator over the same ranks (collective)
    if (!nccl().commSplit) throw std::runtime_error("libnccl.so.2 lacks ncclCommSplit");
    ncclComm_t c = nullptr;
    nccl_check(nccl().commSplit(comm_, 0, rank_, &c, nullptr), "ncclCommSplit");
    return std::make_shared<NcclComm>(world_, rank_, c);
  }
  ~NcclComm() override {
    if (comm_) nccl().commDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void bcast(void* buf, std::size_t bytes, int root, cudaStream_t s) override {
    if (bytes == 0) return;
    nccl_check(nccl().broadcast(buf, buf, bytes, ncclUint8, root, comm_, s), "ncclBroadcast");
  }

 private:
  int world_, rank_;
  ncclComm_t comm_ = nullptr;
};
}  // namespace

std::shared_ptr<Comm> make_nccl_comm(int world, int rank, const void* unique_id128) {
  return std::make_shared<NcclComm>(world, rank, unique_id128);
}

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

// ---------------------------------------------------------------- loopback
namespace {
struct LoopbackHub {
  std::mutex m;
  std::condition_variable cv;
  struct Entry {
    bool posted = false;  // (src may be null for a zero-byte broadcast)
    const void* src = nullptr;
    cudaEvent_t ready = nullptr;
    std::vector<cudaEvent_t> copies;
  };
  std::map<long, Entry> entries;
  int world = 1;
  std::vector<std::shared_ptr<LoopbackHub>> children;  // split channels, by index
};

class LoopbackComm : public Comm {
 public:
  LoopbackComm(std::shared_ptr<LoopbackHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return hub_->world; }
  std::shared_ptr<Comm> split_channel() override {
    // the n-th split of every rank shares one child hub
    std::shared_ptr<LoopbackHub> child;
    {
      std::lock_guard<std::mutex> lk(hub_->m);
      const std::size_t idx = splits_++;
      while (hub_->children.size() <= idx) {
        hub_->children.push_back(std::make_shared<LoopbackHub>());
        hub_->children.back()->world = hub_->world;
      }
      child = hub_->children[idx];
    }
    return std::make_shared<LoopbackComm>(child, rank_);
  }
  void bcast(void* buf, std::size_t bytes, int root, cudaStream_t s) override {
    const long id = seq_++;
    LoopbackHub& h = *hub_;
    if (rank_ == root) {
      cudaEvent_t ready;
      GFQ_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      GFQ_CUDA(cudaEventRecord(ready, s));
      std::unique_lock<std::mutex> lk(h.m);
      auto& e = h.entries[id];
      e.src = buf;
      e.ready = ready;
      e.posted = true;
      h.cv.notify_all();
      h.cv.wait(lk, [&] { return int(h.entries[id].copies.size()) == h.world - 1; });
      // the root's buffer stays untouched until every receiver's copy ran
      for (cudaEvent_t c : h.entries[id].copies) {
        GFQ_CUDA(cudaStreamWaitEvent(s, c, 0));
        cudaEventDestroy(c);
      }
      cudaEventDestroy(ready);
      h.entries.erase(id);
      return;
    }
    const void* src;
    cudaEvent_t ready;
    {
      std::unique_lock<std::mutex> lk(h.m);
      h.cv.wait(lk, [&] {
        auto it = h.entries.find(id);
        return it != h.entries.end() && it->second.posted;
      });
      src = h.entries[id].src;
      ready = h.entries[id].ready;
    }
    GFQ_CUDA(cudaStreamWaitEvent(s, ready, 0));
    if (bytes) GFQ_CUDA(cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToDevice, s));
    cudaEvent_t done;
    GFQ_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    GFQ_CUDA(cudaEventRecord(done, s));
    std::lock_guard<std::mutex> lk(h.m);
    h.entries[id].copies.push_back(done);
    h.cv.notify_all();
  }

 private:
  std::shared_ptr<LoopbackHub> hub_;
  int rank_;
  long seq_ = 0;
  std::size_t splits_ = 0;
};
}  // namespace

std::vector<std::shared_ptr<Comm>> make_loopback_comms(int world) {
  auto hub = std::make_shared<LoopbackHub>();
  hub->world = world;
  std::vector<std::shared_ptr<Comm>> out;
  for (int r = 0; r < world; ++r) out.push_back(std::make_shared<LoopbackComm>(hub, r));
  return out;
}

// ---------------------------------------------------------------- schedule
std::vector<BcastItem> bcast_schedule(const ChopSpec& cs, const PlanHandles&, TaskGraph& g,
                                      const Sharding& sh) {
  std::vector<BcastItem> out;
  const std::size_t a = cs.a(), b = cs.b();
  // Step 1 in wavefront order: anti-diagonal i + j (the plan's priority,
  // src/chief.cpp:116), then column.  PkgA(i, j) depends through broadcasts
  // only on PkgA(i', j') with i' <= i, j' < j, all on earlier anti-diagonals,
  // so this is a topological order every rank can issue without deadlock --
  // and PkgA(0, j+1) no longer waits behind PkgA(a-1, j), which kept the
  // j-outer order one column pair at a time.
  for (std::size_t d = 0; d + 1 < a + b; ++d)
    for (std::size_t j = (d >= a ? d - a + 1 : 0); j <= d && j < b; ++j) {
      const std::size_t i = d - j;
      out.push_back({g.find_slot({PkgKind::A, std::uint16_t(i), std::uint16_t(j), 0, 0}),
                     sh.owner_col(j), true, i, j, 0});
    }
  for (std::size_t k = b; k-- > 1;)
    for (std::size_t j = 0; j < k; ++j)
      out.push_back({g.find_slot({PkgKind::X, std::uint16_t(j), std::uint16_t(k), 0, 0}),
                     sh.owner_col(k), false, 0, j, k});
  for (const auto& it : out)
    if (it.slot < 0) throw std::logic_error("broadcast schedule: slot missing from the plan");
  return out;
}

// ---------------------------------------------------------------- comm loop
namespace {
// Packed layout of a broadcast payload: matrices at 256-byte aligned offsets
// with 16-byte aligned row strides, so receivers use views without copies.
struct Layout {
  struct Part {
    std::int64_t rows, cols, ld;
    std::size_t off;
  };
  std::vector<Part> parts;
  std::size_t bytes = 0;
  void add(std::int64_t rows, std::int64_t cols) {
    const std::int64_t ld = round_up(cols > 0 ? cols : 1, 16);
    parts.push_back({rows, cols, ld, bytes});
    bytes += std::size_t(round_up(rows * ld, 256));
  }
};

void pack_into(const Mat& m, DevBuf& buf, const Layout::Part& p, cudaStream_t s) {
  if (m.rows() != p.rows || m.cols() != p.cols) throw std::logic_error("broadcast: shape drift");
  if (m.empty()) return;
  GFQ_CUDA(cudaMemcpy2DAsync(buf.ptr + p.off, std::size_t(p.ld), m.data(), std::size_t(m.ld()),
                             std::size_t(p.cols), std::size_t(p.rows), cudaMemcpyDeviceToDevice, s));
}

constexpr int kHdr = 8;

struct CommState {
  Comm* comm;
  const ChopSpec* cs;
  const std::vector<BcastItem>* sched;
  std::vector<std::int64_t> col_rank;   // pivots found so far per block column
  std::vector<std::int64_t> row_taken;  // pivot rows taken so far per block row
  std::size_t hdr_cap;
};

// A PkgA header: the host-side fields a receiver needs before it can size
// and post the payload broadcast.
struct PkgAHeader {
  std::int32_t rp = 0, r = 0, live = 0;
  bool hasA = false, hasE = false, hasL = false;
  std::vector<std::uint32_t> rho;
  std::vector<std::uint8_t> lam;
};

// Headers travel on their own channel (Comm::split_channel) and stream,
// driven by a header thread that runs ahead of the payload loop: a
// receiver's host round trip for header q (D2H + stream sync) then never
// waits behind the large payload broadcasts queued before it, and payload
// q is posted the moment its header is known.  Both channels issue their
// collectives in the one schedule order, so neither can deadlock: the
// header thread blocks only on packages being produced, the payload loop
// only on headers.
class HeaderChannel {
 public:
  HeaderChannel(CommState& st, CommApi& api) : st_(st), api_(api) {
    comm_ = st.comm->split_channel();
    int least = 0, greatest = 0;
    GFQ_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    GFQ_CUDA(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, greatest));
    GFQ_CUDA(cudaGetDevice(&device_));
    thread_ = std::thread([this] { run(); });
  }
  ~HeaderChannel() {
    {
      std::lock_guard<std::mutex> lk(m_);
      quit_ = true;
    }
    cv_.notify_all();
    if (thread_.joinable()) thread_.join();
    cudaStreamDestroy(stream_);
  }
  // the next PkgA header in schedule order (blocks until it arrived)
  PkgAHeader next() {
    std::unique_lock<std::mutex> lk(m_);
    cv_.wait(lk, [&] { return !q_.empty() || !error_.empty(); });
    if (!error_.empty()) throw std::runtime_error(error_);
    PkgAHeader h = std::move(q_.front());
    q_.pop_front();
    return h;
  }

 private:
  void run() {
    cudaSetDevice(device_);
    set_cur_stream(stream_);
    try {
      const int me = comm_->rank();
      DevBuf dhdr{st_.hdr_cap * 4};
      std::vector<std::int32_t> hhdr(st_.hdr_cap);
      std::int32_t* pinned = nullptr;
      GFQ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned), st_.hdr_cap * 4));
      struct PinnedFree {
        std::int32_t* p;
        ~PinnedFree() { cudaFreeHost(p); }
      } pf{pinned};
      for (const BcastItem& it : *st_.sched) {
        if (!it.is_a) continue;
        {
          std::lock_guard<std::mutex> lk(m_);
          if (quit_) return;
        }
        PkgAHeader h;
        if (it.root == me) {
          // host fields only: no wait on the package's device data
          const auto pub = api_.wait_local(it.slot);
          const PkgA& A = std::get<PkgA>(pub->value);
          h.rp = std::int32_t(A.rho_prime.size());
          h.live = std::int32_t(A.rho_prime.universe);
          h.r = A.A ? std::int32_t(A.A->cols()) : 0;
          h.hasA = bool(A.A);
          h.hasE = bool(A.E);
          h.hasL = bool(A.lambda);
          h.rho = A.rho_prime.members;
          if (A.lambda) h.lam = A.lambda->bits;
          std::fill(hhdr.begin(), hhdr.end(), 0);
          hhdr[0] = h.rp;
          hhdr[1] = h.r;
          hhdr[2] = h.live;
          hhdr[3] = h.hasA;
          hhdr[4] = h.hasE;
          hhdr[5] = h.hasL;
          hhdr[6] = std::int32_t(h.lam.size());
          for (std::int32_t q = 0; q < h.rp; ++q) hhdr[kHdr + q] = std::int32_t(h.rho[std::size_t(q)]);
          for (std::int32_t q = 0; q < hhdr[6]; ++q) hhdr[kHdr + h.rp + q] = h.lam[std::size_t(q)];
          std::memcpy(pinned, hhdr.data(), st_.hdr_cap * 4);
          GFQ_CUDA(cudaMemcpyAsync(dhdr.ptr, pinned, st_.hdr_cap * 4, cudaMemcpyHostToDevice, stream_));
          comm_->bcast(dhdr.ptr, st_.hdr_cap * 4, it.root, stream_);
          // the pinned buffer is rewritten by the next header: drain the copy
          GFQ_CUDA(cudaStreamSynchronize(stream_));
        } else {
          comm_->bcast(dhdr.ptr, st_.hdr_cap * 4, it.root, stream_);
          GFQ_CUDA(cudaMemcpyAsync(pinned, dhdr.ptr, st_.hdr_cap * 4, cudaMemcpyDeviceToHost, stream_));
          GFQ_CUDA(cudaStreamSynchronize(stream_));
          std::memcpy(hhdr.data(), pinned, st_.hdr_cap * 4);
          h.rp = hhdr[0];
          h.r = hhdr[1];
          h.live = hhdr[2];
          h.hasA = hhdr[3];
          h.hasE = hhdr[4];
          h.hasL = hhdr[5];
          h.rho.assign(hhdr.begin() + kHdr, hhdr.begin() + kHdr + h.rp);
          h.lam.assign(hhdr.begin() + kHdr + h.rp, hhdr.begin() + kHdr + h.rp + hhdr[6]);
        }
        std::lock_guard<std::mutex> lk(m_);
        q_.push_back(std::move(h));
        cv_.notify_all();
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(m_);
      error_ = std::string("header channel: ") + e.what();
      cv_.notify_all();
    }
    set_cur_stream(nullptr);
  }

  CommState& st_;
  CommApi& api_;
  std::shared_ptr<Comm> comm_;
  cudaStream_t stream_ = nullptr;
  int device_ = 0;
  std::thread thread_;
  std::mutex m_;
  std::condition_variable cv_;
  std::deque<PkgAHeader> q_;
  std::string error_;
  bool quit_ = false;
};

void comm_loop_body(CommState& st, CommApi& api, HeaderChannel& headers);

void comm_loop(CommState& st, CommApi& api) {
  HeaderChannel headers(st, api);
  try {
    comm_loop_body(st, api, headers);
  } catch (const std::exception& e) {
    // release the header thread if it waits on a package (its destructor joins)
    if (api.abort) api.abort(e.what());
    throw;
  }
}

void comm_loop_body(CommState& st, CommApi& api, HeaderChannel& headers) {
  Comm& comm = *st.comm;
  const int me = comm.rank();
  const cudaStream_t s = api.stream;

  for (const BcastItem& it : *st.sched) {
    const bool root = it.root == me;
    if (it.is_a) {
      // ---- PkgA(i, j): the header from the header channel, then one payload
      std::shared_ptr<Published> pub;
      PkgAHeader hd = headers.next();
      const std::int32_t rp = hd.rp, r = hd.r, live = hd.live;
      const bool hasA = hd.hasA, hasE = hd.hasE, hasL = hd.hasL;
      if (root) {
        pub = api.wait_local(it.slot);
        if (pub->ready) GFQ_CUDA(cudaStreamWaitEvent(s, pub->ready->ev, 0));
      }
      Layout L;
      L.add(hasA ? live : 0, hasA ? r : 0);  // A.A
      L.add(rp, rp);                          // M
      L.add(live - rp, rp);                   // K
      L.add(hasE ? r : 0, hasE ? rp : 0);     // E
      auto payload = std::make_shared<DevBuf>(L.bytes > 0 ? L.bytes : 256);
      if (root) {
        const PkgA& A = std::get<PkgA>(pub->value);
        if (hasA) pack_into(*A.A, *payload, L.parts[0], s);
        pack_into(A.M, *payload, L.parts[1], s);
        pack_into(A.K, *payload, L.parts[2], s);
        if (hasE) pack_into(*A.E, *payload, L.parts[3], s);
      }
      comm.bcast(payload->ptr, L.bytes, it.root, s);
      if (root) {
        api.done_with(it.slot);
      } else {
        PkgA A;
        const auto& P = L.parts;
        if (hasA) A.A = Mat::view_of(payload, P[0].off, P[0].rows, P[0].cols, P[0].ld);
        A.M = Mat::view_of(payload, P[1].off, P[1].rows, P[1].cols, P[1].ld);
        A.K = Mat::view_of(payload, P[2].off, P[2].rows, P[2].cols, P[2].ld);
        if (hasE) A.E = Mat::view_of(payload, P[3].off, P[3].rows, P[3].cols, P[3].ld);
        A.rho_prime = IndexSet(std::size_t(live), std::move(hd.rho));
        if (hasL) A.lambda = BitString(std::move(hd.lam));
        auto np = std::make_shared<Published>();
        np->value = std::move(A);
        np->ready = std::make_shared<EventBox>();
        GFQ_CUDA(cudaEventRecord(np->ready->ev, s));
        api.publish(it.slot, std::move(np));
      }
      st.col_rank[it.j] += rp;
      st.row_taken[it.i] += rp;
    } else {
      // ---- X(j, k): r_j x r_k, shape known from the A headers
      const std::int64_t rows = st.col_rank[it.j], cols = st.col_rank[it.k];
      const std::int64_t ld = round_up(cols > 0 ? cols : 1, 16);
      if (root) {
        auto pub = api.wait_local(it.slot);
        if (pub->ready) GFQ_CUDA(cudaStreamWaitEvent(s, pub->ready->ev, 0));
        const Mat& X = std::get<Mat>(pub->value);
        if (X.rows() != rows || X.cols() != cols) throw std::logic_error("broadcast: X shape drift");
        if (X.empty()) {
          comm.bcast(nullptr, 0, it.root, s);
        } else if (X.ld() == ld) {
          comm.bcast(X.data(), std::size_t(rows * ld), it.root, s);
        } else {
          DevBuf tmp{std::size_t(rows * ld)};
          GFQ_CUDA(cudaMemcpy2DAsync(tmp.ptr, std::size_t(ld), X.data(), std::size_t(X.ld()),
                                     std::size_t(cols), std::size_t(rows), cudaMemcpyDeviceToDevice, s));
          comm.bcast(tmp.ptr, std::size_t(rows * ld), it.root, s);
        }
        api.done_with(it.slot);
      } else {
        Mat X(rows, cols);
        comm.bcast(X.empty() ? nullptr : X.data(), X.empty() ? 0 : std::size_t(rows * X.ld()),
                   it.root, s);
        auto np = std::make_shared<Published>();
        np->value = std::move(X);
        np->ready = std::make_shared<EventBox>();
        GFQ_CUDA(cudaEventRecord(np->ready->ev, s));
        api.publish(it.slot, std::move(np));
      }
    }
  }
}

// Broadcast a matrix of known shape from `root` (owner) to everyone.
Mat bcast_mat(Comm& comm, const Mat* mine, std::int64_t rows, std::int64_t cols, int root,
              cudaStream_t s) {
  Mat out(rows, cols);
  if (out.empty()) return out;
  if (comm.rank() == root) {
    GFQ_CUDA(cudaMemcpy2DAsync(out.data(), std::size_t(out.ld()), mine->data(),
                               std::size_t(mine->ld()), std::size_t(cols), std::size_t(rows),
                               cudaMemcpyDeviceToDevice, s));
  }
  comm.bcast(out.data(), std::size_t(rows * out.ld()), root, s);
  return out;
}

IndexSet bcast_iset(Comm& comm, const IndexSet* mine, std::size_t universe, int root, cudaStream_t s) {
  DevBuf d{4 * (universe + 1)};
  std::vector<std::int32_t> h(universe + 1, 0);
  if (comm.rank() == root) {
    h[0] = std::int32_t(mine->size());
    for (std::size_t q = 0; q < mine->size(); ++q) h[1 + q] = std::int32_t(mine->members[q]);
    GFQ_CUDA(cudaMemcpyAsync(d.ptr, h.data(), h.size() * 4, cudaMemcpyHostToDevice, s));
  }
  comm.bcast(d.ptr, h.size() * 4, root, s);
  GFQ_CUDA(cudaMemcpyAsync(h.data(), d.ptr, h.size() * 4, cudaMemcpyDeviceToHost, s));
  GFQ_CUDA(cudaStreamSynchronize(s));
  std::vector<std::uint32_t> mem(h.begin() + 1, h.begin() + 1 + h[0]);
  return IndexSet(universe, std::move(mem));
}
}  // namespace

// ---------------------------------------------------------------- entry
EchelonOutput echelonize_dist(const Mat* C, std::int64_t m, std::int64_t n, std::uint64_t seed,
                              const FieldSpec& field, const EchelonizeOptions& options, Comm& comm,
                              RunReport* report, bool gather) {
  if (field.wide())
    throw std::invalid_argument("echelonize_dist: the sharded Chief takes u8 fields (p <= 251, p^k <= 256)");
  const ChopSpec cs = chop(std::size_t(m), std::size_t(n), options.block, options.remainder_first);
  const std::size_t a = cs.a(), b = cs.b();
  EchelonOutput out{field};
  out.chop = cs;
  out.with_transform = options.with_transform;
  if (a == 0 || b == 0) {
    if (C) return echelonize(*C, field, options, report);
    throw std::invalid_argument("echelonize_dist: empty matrix");
  }
  const Sharding sh{comm.world(), comm.rank()};
  const int me = comm.rank();

  // this rank's block columns of the input
  std::vector<Mat> colblk(b);
  for (std::size_t k = 0; k < b; ++k) {
    if (sh.owner_col(k) != me) continue;
    if (C) {
      colblk[k] = C->col_view(std::int64_t(cs.col_offset(k)), std::int64_t(cs.col_parts[k]));
    } else {
      colblk[k] = Mat(m, std::int64_t(cs.col_parts[k]));
      random_fill_exact(field.order(), m, std::int64_t(cs.col_parts[k]), seed,
                        std::uint64_t(cs.col_offset(k)), n, colblk[k].data(), colblk[k].ld());
    }
  }
  TaskGraph graph;
  graph.ech_threshold = options.ech_threshold;
  const PlanHandles h = build_plan(
      graph,
      [&](std::size_t i, std::size_t k) -> std::optional<Mat> {
        if (sh.owner_col(k) != me) return std::nullopt;
        return colblk[k].row_view(std::int64_t(cs.row_offset(i)), std::int64_t(cs.row_parts[i]));
      },
      field, cs, options.with_transform);
  for (auto id : h.d_final) graph.retain(id);
  for (auto id : h.e_final) graph.retain(id);
  for (const auto& row : h.r_final)
    for (auto id : row)
      if (id >= 0) graph.retain(id);
  for (const auto& row : h.m_final)
    for (auto id : row) graph.retain(id);
  for (const auto& row : h.k_final)
    for (auto id : row) graph.retain(id);

  std::vector<char> owned(graph.node_count());
  for (std::size_t q = 0; q < graph.node_count(); ++q) {
    const int o = owner_of(sh, graph, graph.node(std::int32_t(q)));
    owned[q] = (o == -1 || o == me) ? 1 : 0;
  }
  const std::vector<BcastItem> sched = bcast_schedule(cs, h, graph, sh);
  RunOptions ro;
  ro.workers = options.threads;
  ro.collect_trace = options.collect_trace;
  ro.retain_all = options.retain_all;
  ro.owned = &owned;
  for (const auto& it : sched) (it.root == me ? ro.sent_slots : ro.remote_slots).push_back(it.slot);
  CommState st;
  st.comm = &comm;
  st.cs = &cs;
  st.sched = &sched;
  st.col_rank.assign(b, 0);
  st.row_taken.assign(a, 0);
  std::size_t amax = 0, bmax = 0;
  for (auto v : cs.row_parts) amax = std::max(amax, v);
  for (auto v : cs.col_parts) bmax = std::max(bmax, v);
  st.hdr_cap = std::size_t(kHdr) + amax + 2 * bmax + 8;
  ro.comm_loop = [&](CommApi& api) { comm_loop(st, api); };
  RunReport rep = run(graph, ro);
  if (report) *report = std::move(rep);

  // ---- assemble: E (all ranks), owned blocks, then gather by broadcast
  for (std::size_t i = 0; i < a; ++i)
    out.varrho.push_back(std::get<PkgE>(*graph.payload(h.e_final[i])).rho);
  const cudaStream_t s = cur_stream();
  out.upsilon.resize(b);
  for (std::size_t j = 0; j < b; ++j) {
    const PkgD* d = sh.owner_col(j) == me ? &std::get<PkgD>(*graph.payload(h.d_final[j])) : nullptr;
    out.upsilon[j] = gather ? bcast_iset(comm, d ? &d->gamma : nullptr, cs.col_parts[j],
                                         sh.owner_col(j), s)
                            : (d ? d->gamma : IndexSet(cs.col_parts[j], {}));
    out.rank += out.upsilon[j].size();
  }
  out.R_blocks.assign(b, std::vector<Mat>(b));
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t l = j; l < b; ++l) {
      const int o = sh.owner_col(l);
      const Mat* mine = o == me ? &std::get<Mat>(*graph.payload(h.r_final[j][l])) : nullptr;
      if (gather)
        out.R_blocks[j][l] =
            bcast_mat(comm, mine, std::int64_t(out.upsilon[j].size()),
                      std::int64_t(cs.col_parts[l] - out.upsilon[l].size()), o, s);
      else if (mine)
        out.R_blocks[j][l] = *mine;
    }
  if (options.with_transform) {
    out.T_M_blocks.assign(b, std::vector<Mat>(a));
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t hh = 0; hh < a; ++hh) {
        const int o = sh.owner_trow(hh);
        const Mat* mine = o == me ? &std::get<Mat>(*graph.payload(h.m_final[j][hh])) : nullptr;
        if (gather)
          out.T_M_blocks[j][hh] = bcast_mat(comm, mine, std::int64_t(out.upsilon[j].size()),
                                            std::int64_t(out.varrho[hh].size()), o, s);
        else if (mine)
          out.T_M_blocks[j][hh] = *mine;
      }
    out.T_K_blocks.resize(a);
    for (std::size_t i = 0; i < a; ++i)
      for (std::size_t hh = 0; hh <= i; ++hh) {
        const int o = sh.owner_trow(hh);
        const Mat* mine = o == me ? &std::get<Mat>(*graph.payload(h.k_final[i][hh])) : nullptr;
        if (gather)
          out.T_K_blocks[i].push_back(
              bcast_mat(comm, mine, std::int64_t(cs.row_parts[i] - out.varrho[i].size()),
                        std::int64_t(out.varrho[hh].size()), o, s));
        else
          out.T_K_blocks[i].push_back(mine ? *mine : Mat());
      }
  }
  GFQ_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace gfq
