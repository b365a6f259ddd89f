// C-ABI implementation, part 4: the library's communicator — NCCL (libnccl
// loaded at runtime, so single-GPU use has no NCCL dependency) or a caller's
// host all-reduce — its collectives, and the near-field pair partition across
// ranks.
#include <dlfcn.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "handle.cuh"

using namespace fpbem_cu;

namespace {
void* load_nccl() {
  static void* lib = nullptr;
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  return lib;
}

constexpr int kNcclFloat64 = 8, kNcclSum = 0;

void nccl_rc(int rc, const char* what) {
  if (rc != 0) fail(FPBEM_CU_ENCCL, std::string(what) + " failed: " + std::to_string(rc));
}

// host form: device -> pinned stage -> caller's all-reduce -> device
double* stage(fpbem_cu_comm* c, size_t count) {
  if (c->stage_count < count) {
    if (c->stage) cudaFreeHost(c->stage);
    c->stage = nullptr;
    c->stage_count = 0;
    check(cudaMallocHost(&c->stage, count * sizeof(double)), "comm staging buffer");
    c->stage_count = count;
  }
  return c->stage;
}

void host_allreduce(fpbem_cu_comm* c, double* h, size_t count) {
  if (c->cb(c->cb_ctx, h, count) != 0) fail(FPBEM_CU_ENCCL, "host all-reduce callback failed");
}
}  // namespace

namespace fpbem_cu {

// A communicator of one rank still runs its collectives (so the NCCL and the
// staged paths are exercised on one GPU); no communicator = this rank alone.
void comm_allreduce(fpbem_cu_comm* c, double* buf, size_t count, cudaStream_t s) {
  if (!c || count == 0) return;
  if (c->sim) {  // a ring all-reduce sends 2 (P-1)/P of the buffer per rank
    c->sim_bytes += 2ull * (c->nranks - 1) * count * sizeof(double) / c->nranks;
    c->sim_calls++;
    return;
  }
  if (!c->cb) {
    nccl_rc(c->allreduce(buf, buf, count, kNcclFloat64, kNcclSum, c->comm, s), "ncclAllReduce");
    return;
  }
  double* h = stage(c, count);
  check(cudaMemcpyAsync(h, buf, count * sizeof(double), cudaMemcpyDeviceToHost, s), "comm stage");
  check(cudaStreamSynchronize(s), "comm stage");
  host_allreduce(c, h, count);
  check(cudaMemcpyAsync(buf, h, count * sizeof(double), cudaMemcpyHostToDevice, s), "comm unstage");
  check(cudaStreamSynchronize(s), "comm unstage");
}

// full: nranks x per_rank (rank r's slab at r * per_rank), summed over the
// ranks; this rank's slab of the sum lands in `mine`
void comm_reduce_scatter(fpbem_cu_comm* c, double* full, double* mine, size_t per_rank, cudaStream_t s) {
  const int r = c ? c->rank : 0;
  if (!c) {
    if (mine != full)
      check(cudaMemcpyAsync(mine, full, per_rank * sizeof(double), cudaMemcpyDeviceToDevice, s), "slab copy");
    return;
  }
  if (c->sim) {
    c->sim_bytes += static_cast<unsigned long long>(c->nranks - 1) * per_rank * sizeof(double);
    c->sim_calls++;
    if (mine != full + r * per_rank)
      check(cudaMemcpyAsync(mine, full + r * per_rank, per_rank * sizeof(double), cudaMemcpyDeviceToDevice, s),
            "slab copy");
    return;
  }
  if (!c->cb) {
    nccl_rc(c->reduce_scatter(full, mine, per_rank, kNcclFloat64, kNcclSum, c->comm, s), "ncclReduceScatter");
    return;
  }
  const size_t count = per_rank * c->nranks;
  double* h = stage(c, count);
  check(cudaMemcpyAsync(h, full, count * sizeof(double), cudaMemcpyDeviceToHost, s), "comm stage");
  check(cudaStreamSynchronize(s), "comm stage");
  host_allreduce(c, h, count);
  check(cudaMemcpyAsync(mine, h + r * per_rank, per_rank * sizeof(double), cudaMemcpyHostToDevice, s),
        "comm unstage");
  check(cudaStreamSynchronize(s), "comm unstage");
}

// every rank's slab `mine` (per_rank doubles) into full[r * per_rank ...]
void comm_allgather(fpbem_cu_comm* c, const double* mine, double* full, size_t per_rank, cudaStream_t s) {
  if (!c) {
    if (mine != full)
      check(cudaMemcpyAsync(full, mine, per_rank * sizeof(double), cudaMemcpyDeviceToDevice, s), "slab copy");
    return;
  }
  if (c->sim) {
    c->sim_bytes += static_cast<unsigned long long>(c->nranks - 1) * per_rank * sizeof(double);
    c->sim_calls++;
    if (full + c->rank * per_rank != mine)
      check(cudaMemcpyAsync(full + c->rank * per_rank, mine, per_rank * sizeof(double), cudaMemcpyDeviceToDevice, s),
            "slab copy");
    return;
  }
  if (!c->cb) {
    nccl_rc(c->allgather(mine, full, per_rank, kNcclFloat64, c->comm, s), "ncclAllGather");
    return;
  }
  const size_t count = per_rank * c->nranks;
  double* h = stage(c, count);
  check(cudaStreamSynchronize(s), "comm stage");
  std::memset(h, 0, count * sizeof(double));
  check(cudaMemcpyAsync(h + c->rank * per_rank, mine, per_rank * sizeof(double), cudaMemcpyDeviceToHost, s),
        "comm stage");
  check(cudaStreamSynchronize(s), "comm stage");
  host_allreduce(c, h, count);  // the other slabs are zero here: the sum is exact
  check(cudaMemcpyAsync(full, h, count * sizeof(double), cudaMemcpyHostToDevice, s), "comm unstage");
  check(cudaStreamSynchronize(s), "comm unstage");
}

void comm_alltoallv(fpbem_cu_comm* c, const A2aPart* parts, int n_parts, cudaStream_t s) {
  if (!c) {  // a single rank: its own blocks
    for (int k = 0; k < n_parts; ++k) {
      const A2aPart& p = parts[k];
      if (p.scount[0])
        check(cudaMemcpyAsync(p.recv + p.rdisp[0], p.send + p.sdisp[0], p.scount[0] * sizeof(double),
                              cudaMemcpyDeviceToDevice, s),
              "slab exchange (one rank)");
    }
    return;
  }
  const int P = c->nranks, me = c->rank;
  if (c->sim) {  // this rank's own block moves; the others are counted, not sent
    for (int k = 0; k < n_parts; ++k) {
      const A2aPart& p = parts[k];
      for (int d = 0; d < P; ++d)
        if (d != me) c->sim_bytes += p.scount[d] * sizeof(double);
      if (p.scount[me])
        check(cudaMemcpyAsync(p.recv + p.rdisp[me], p.send + p.sdisp[me], p.scount[me] * sizeof(double),
                              cudaMemcpyDeviceToDevice, s),
              "slab exchange (own block)");
    }
    c->sim_calls++;
    return;
  }
  if (!c->cb) {
    nccl_rc(c->group_start(), "ncclGroupStart");
    for (int k = 0; k < n_parts; ++k) {
      const A2aPart& p = parts[k];
      for (int d = 0; d < P; ++d) {
        if (p.scount[d]) nccl_rc(c->send(p.send + p.sdisp[d], p.scount[d], kNcclFloat64, d, c->comm, s), "ncclSend");
        if (p.rcount[d]) nccl_rc(c->recv(p.recv + p.rdisp[d], p.rcount[d], kNcclFloat64, d, c->comm, s), "ncclRecv");
      }
    }
    nccl_rc(c->group_end(), "ncclGroupEnd");
    return;
  }
  // host-staged: every (src, dst) block at its place in one zero-filled buffer,
  // summed over the ranks (each block has exactly one non-zero contributor)
  for (int k = 0; k < n_parts; ++k) {
    const A2aPart& p = parts[k];
    std::vector<size_t> off(static_cast<size_t>(P) * P + 1, 0);
    for (size_t i = 0; i < static_cast<size_t>(P) * P; ++i) off[i + 1] = off[i] + p.all[i];
    const size_t total = off.back();
    if (total == 0) continue;
    double* h = stage(c, total);
    check(cudaStreamSynchronize(s), "comm stage");
    std::memset(h, 0, total * sizeof(double));
    for (int d = 0; d < P; ++d)
      if (p.scount[d])
        check(cudaMemcpyAsync(h + off[static_cast<size_t>(me) * P + d], p.send + p.sdisp[d],
                              p.scount[d] * sizeof(double), cudaMemcpyDeviceToHost, s),
              "comm stage");
    check(cudaStreamSynchronize(s), "comm stage");
    host_allreduce(c, h, total);
    for (int r = 0; r < P; ++r)
      if (p.rcount[r])
        check(cudaMemcpyAsync(p.recv + p.rdisp[r], h + off[static_cast<size_t>(r) * P + me],
                              p.rcount[r] * sizeof(double), cudaMemcpyHostToDevice, s),
              "comm unstage");
    check(cudaStreamSynchronize(s), "comm unstage");
  }
}

}  // namespace fpbem_cu

extern "C" {

int fpbem_cu_comm_unique_id(unsigned char id_out[128]) {
  return guard([&] {
    void* lib = load_nccl();
    if (!lib) fail(FPBEM_CU_ENCCL, "libnccl.so.2 not loadable");
    auto get_id = reinterpret_cast<int (*)(void*)>(dlsym(lib, "ncclGetUniqueId"));
    if (!get_id) fail(FPBEM_CU_ENCCL, "ncclGetUniqueId missing");
    if (get_id(id_out) != 0) fail(FPBEM_CU_ENCCL, "ncclGetUniqueId failed");
  });
}

int fpbem_cu_comm_init(const unsigned char id[128], int nranks, int rank, int device, fpbem_cu_comm** out) {
  return guard([&] {
    void* lib = load_nccl();
    if (!lib) fail(FPBEM_CU_ENCCL, "libnccl.so.2 not loadable");
    struct IdBlob {
      unsigned char b[128];
    } blob;
    std::memcpy(blob.b, id, 128);
    auto init = reinterpret_cast<int (*)(void**, int, IdBlob, int)>(dlsym(lib, "ncclCommInitRank"));
    auto* c = new fpbem_cu_comm();
    c->lib = lib;
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->allreduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, void*)>(
        dlsym(lib, "ncclAllReduce"));
    c->reduce_scatter = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, void*)>(
        dlsym(lib, "ncclReduceScatter"));
    c->allgather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, void*)>(
        dlsym(lib, "ncclAllGather"));
    c->destroy = reinterpret_cast<int (*)(void*)>(dlsym(lib, "ncclCommDestroy"));
    c->send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, void*)>(dlsym(lib, "ncclSend"));
    c->recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, void*)>(dlsym(lib, "ncclRecv"));
    c->group_start = reinterpret_cast<int (*)()>(dlsym(lib, "ncclGroupStart"));
    c->group_end = reinterpret_cast<int (*)()>(dlsym(lib, "ncclGroupEnd"));
    if (!init || !c->allreduce || !c->reduce_scatter || !c->allgather || !c->destroy || !c->send || !c->recv ||
        !c->group_start || !c->group_end) {
      delete c;
      fail(FPBEM_CU_ENCCL, "NCCL symbols missing");
    }
    check(cudaSetDevice(device), "set device");
    if (init(&c->comm, nranks, blob, rank) != 0) {
      delete c;
      fail(FPBEM_CU_ENCCL, "ncclCommInitRank failed");
    }
    *out = c;
  });
}

int fpbem_cu_comm_from_callback(fpbem_cu_allreduce_fn allreduce_sum, void* ctx, int nranks, int rank, int device,
                                fpbem_cu_comm** out) {
  return guard([&] {
    if (!allreduce_sum || !out || nranks < 1 || rank < 0 || rank >= nranks)
      fail(FPBEM_CU_EINVAL, "comm_from_callback: bad arguments");
    auto* c = new fpbem_cu_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->cb = allreduce_sum;
    c->cb_ctx = ctx;
    *out = c;
  });
}

int fpbem_cu_comm_simulated(int nranks, int rank, int device, fpbem_cu_comm** out) {
  return guard([&] {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks) fail(FPBEM_CU_EINVAL, "comm_simulated: bad arguments");
    auto* c = new fpbem_cu_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->sim = true;
    *out = c;
  });
}

int fpbem_cu_comm_traffic(fpbem_cu_comm* comm, unsigned long long* bytes_sent, long long* collectives, int reset) {
  return guard([&] {
    if (!comm || !bytes_sent || !collectives) fail(FPBEM_CU_EINVAL, "comm_traffic: null argument");
    if (!comm->sim) fail(FPBEM_CU_EINVAL, "comm_traffic: only a simulated communicator counts its traffic");
    *bytes_sent = comm->sim_bytes;
    *collectives = comm->sim_calls;
    if (reset) {
      comm->sim_bytes = 0;
      comm->sim_calls = 0;
    }
  });
}

void fpbem_cu_comm_destroy(fpbem_cu_comm* comm) {
  if (!comm) return;
  if (comm->comm && comm->destroy) comm->destroy(comm->comm);
  if (comm->stage) cudaFreeHost(comm->stage);
  delete comm;
}

int fpbem_cu_fmm_set_comm(fpbem_cu_op* op, fpbem_cu_comm* comm) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "set_comm: null op");
    check(cudaSetDevice(op->device), "set device");
    if (!comm) {
      op->comm = nullptr;
      set_partition(op, 0, 1, 0.0);
      return;
    }
    // rank 0's far-field cost in pair equivalents, averaged over the ranks so
    // that every rank derives the same partition
    double f = comm->nranks > 1 ? calibrate_far_pairs(op) : 0.0;
    if (comm->nranks > 1) {
      double* df = dalloc<double>(1, "far pairs");
      std::unique_ptr<double, decltype(&cudaFree)> keep_df(df, &cudaFree);
      h2d(df, &f, sizeof(double), op->stream, "far pairs");
      comm_allreduce(comm, df, 1, op->stream);
      check(cudaMemcpyAsync(&f, df, sizeof(double), cudaMemcpyDeviceToHost, op->stream), "far pairs");
      check(cudaStreamSynchronize(op->stream), "far pairs");
      f /= comm->nranks;
    }
    set_partition(op, comm->rank, comm->nranks, f);
    op->comm = comm;
  });
}

int fpbem_cu_fmm_set_partition(fpbem_cu_op* op, int rank, int nranks, double far_pairs) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "set_partition: null op");
    check(cudaSetDevice(op->device), "set device");
    set_partition(op, rank, nranks, far_pairs);
  });
}

int fpbem_cu_fmm_partition(const fpbem_cu_op* op, long long* lo, long long* hi, double* far_pairs) {
  return guard([&] {
    if (!op || !lo || !hi || !far_pairs) fail(FPBEM_CU_EINVAL, "partition: null argument");
    *lo = op->near_fft ? op->mode_lo : op->pair_lo;  // the unit range of the near path in use
    *hi = op->near_fft ? op->mode_hi : op->pair_hi;
    *far_pairs = op->far_pairs;
  });
}

int fpbem_cu_fmm_far_pairs(fpbem_cu_op* op, double* far_pairs) {
  return guard([&] {
    if (!op || !far_pairs) fail(FPBEM_CU_EINVAL, "far_pairs: null argument");
    check(cudaSetDevice(op->device), "set device");
    *far_pairs = calibrate_far_pairs(op);
  });
}

int fpbem_cu_partition_pairs(long long n_pairs, int nranks, int rank, double far_pairs, long long* lo,
                             long long* hi) {
  return guard([&] {
    if (n_pairs < 0 || nranks < 1 || rank < 0 || rank >= nranks || !lo || !hi || !(far_pairs >= 0.0))
      fail(FPBEM_CU_EINVAL, "partition: bad args");
    pair_range(n_pairs, nranks, rank, far_pairs, *lo, *hi);
  });
}

}  // extern "C"
