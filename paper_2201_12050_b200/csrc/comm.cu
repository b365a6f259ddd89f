// C-ABI implementation, part 4: the library's NCCL communicator (libnccl
// loaded at runtime, so single-GPU use has no NCCL dependency) and the
// near-field pair partition across ranks.
#include <dlfcn.h>

#include <cstring>
#include <memory>
#include <string>

#include "handle.cuh"

using namespace fpbem_cu;

namespace {
void* load_nccl() {
  static void* lib = nullptr;
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  return lib;
}
}  // namespace

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
    c->destroy = reinterpret_cast<int (*)(void*)>(dlsym(lib, "ncclCommDestroy"));
    if (!init || !c->allreduce || !c->destroy) {
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

void fpbem_cu_comm_destroy(fpbem_cu_comm* comm) {
  if (!comm) return;
  if (comm->comm && comm->destroy) comm->destroy(comm->comm);
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
      const int rc = comm->allreduce(df, df, 1, /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm->comm, op->stream);
      if (rc != 0) fail(FPBEM_CU_ENCCL, "ncclAllReduce failed: " + std::to_string(rc));
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
    *lo = op->pair_lo;
    *hi = op->pair_hi;
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
