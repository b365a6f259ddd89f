// C-ABI implementation, part 6: the slab-distributed product (SURVEY.md §8e,
// cfg3 row; north_star: "Fourier modes and near-field cell slabs are split per
// GPU, and the FFT transpose is an NCCL all-to-all over NVLink").
//
// FmmOperators::matvec (src/fmm.cpp:246-271) with the lattice near field and
// the M2L both applied as DFT convolutions (CirculantSpectrum::matvec,
// src/structured.cpp:122-166, and its application to the Toeplitz blocks of
// BlockToeplitzMatrix::matvec, src/assembly.cpp:62-84). The vectors are split
// into slabs of whole planes along the slab axis s (the highest lattice axis
// with more than one cell: rows of the reference's cell-major layout stay
// contiguous). Per product, each rank:
//   1. P2M on its cells; DFTs along the axes below s on its planes (near field
//      over n fields, far field over b coefficients);
//   2. forward exchange (one grouped NCCL send/recv set for both fields): the
//      transposition from "my planes, every column" to "every plane, my
//      columns", a column being the set of modes with equal indices below s;
//   3. on its columns: the DFT along s, the per-mode block products with this
//      rank's share of the stored near-field blocks (one per orbit of modes;
//      the orbits of a column class never leave it) and of Λ, the inverse DFT
//      along s (with 1/q);
//   4. backward exchange, the inverse DFTs below s on its planes, L2P.
// A column class is a column with its images under the sign flips of the axes
// below s: closed under the cell symmetries' orbits and under the Λ mirror
// pairing, so every work item of a rank reads and writes only its columns.
// Classes go to ranks by longest-processing-time on the stored-block (near) /
// column (far) counts; every rank derives the same plan from the same data,
// so the plan needs no communication. Λ and the near-field block spectrum are
// stored per rank only for its columns (sharded, 1/P of the HBM each).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "handle.cuh"

// (global scope: fpbem_cu_op holds a `struct SlabPlan*`)
struct SlabSide {
  long long Ls = 1;          // lattice length along the slab axis
  long long cx = 1, cy = 1;  // lattice extents of the column axes (cy = 1 unless the slab axis is z)
  long long C = 1;           // columns per plane = cx cy
  int E = 0;                 // complex values per (plane, column): n (near) or b (far)
  std::vector<std::vector<int>> cols;  // per rank: its global columns in local order
  std::vector<int> lc;                 // global column -> local index on its owner
  int* idx = nullptr;                  // device: pack order, (z_local, column) as z * C + col, by destination
  long long n_idx = 0;
  std::vector<size_t> fsc, fsd, frc, frd, fall;  // forward exchange (doubles)
  std::vector<size_t> bsc, bsd, brc, brd, ball;  // backward exchange
  c64* pack = nullptr;  // ms C E
  c64* recv = nullptr;  // max(Ms, Ls) |cols_me| E
  c64* work = nullptr;  // Ls |cols_me| E
};

struct SlabPlan {
  fpbem_cu_comm* comm = nullptr;
  int P = 1, rank = 0, axis = 0;
  long long Ms = 1;  // cells along the slab axis
  long long Cm = 1;  // cells per plane (axes below s)
  long long mx = 1, my = 1;  // cell extents of the column axes
  std::vector<long long> zlo;  // plane range per rank (P + 1 entries)
  long long ms = 0;            // this rank's planes
  SlabSide nr, fr;             // near-field lattice, far-field (M2L) lattice
  c64* shat = nullptr;         // this rank's stored near-field blocks
  int* items = nullptr;        // [n_items][8] local modes, then [n_items][8] g
  long long n_items = 0;
  c64* lambda = nullptr;       // Λ of this rank's columns, [qs][column][b b]
  int2* zitems = nullptr;      // fused z-kernel items over local columns
  int n_zitems = 0;
  bool zfused = false;
  c64* a = nullptr;  // near-field plane buffers, ms near planes each
  c64* b = nullptr;
  c64* fa = nullptr;  // far-field plane buffers (the far side runs concurrently on the aux stream)
  c64* fb = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  c64* mom = nullptr;
  c64* loc = nullptr;
  std::vector<void*> owned;
  // the product's compute phases captured as CUDA graphs on hx -> hy (apply_slab_graph)
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};  // the three compute phases
  cudaStream_t graph_stream = nullptr;
  long long graph_launches = 0;
  // the graph's (and host-pointer products') slab vectors
  c64* hx = nullptr;
  c64* hy = nullptr;
};

namespace fpbem_cu {

void slab_destroy(fpbem_cu_op* op) {
  if (!op || !op->slab) return;
  if (op->slab->fork) cudaEventDestroy(op->slab->fork);
  if (op->slab->join) cudaEventDestroy(op->slab->join);
  for (auto g : op->slab->graph)
    if (g) cudaGraphExecDestroy(g);
  for (void* p : op->slab->owned) cudaFree(p);
  delete op->slab;
  op->slab = nullptr;
}

}  // namespace fpbem_cu

using namespace fpbem_cu;

namespace {

__global__ void gather_rows_kernel(const c64* __restrict__ src, c64* __restrict__ dst, const int* __restrict__ idx,
                                   long long rows, int E) {
  const long long total = rows * E;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = g / E;
    dst[g] = src[static_cast<long long>(idx[r]) * E + (g - r * E)];
  }
}

__global__ void scatter_rows_kernel(const c64* __restrict__ src, c64* __restrict__ dst, const int* __restrict__ idx,
                                    long long rows, int E) {
  const long long total = rows * E;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = g / E;
    dst[static_cast<long long>(idx[r]) * E + (g - r * E)] = src[g];
  }
}

int rows_grid(long long total) {
  const long long blocks = (total + 255) / 256;
  return static_cast<int>(std::max(1LL, std::min(blocks, 8LL * device_sms())));
}

void gather_rows(const c64* src, c64* dst, const int* idx, long long rows, int E, cudaStream_t s) {
  if (rows * E == 0) return;
  gather_rows_kernel<<<rows_grid(rows * E), 256, 0, s>>>(src, dst, idx, rows, E);
  check(cudaGetLastError(), "slab pack");
}

void scatter_rows(const c64* src, c64* dst, const int* idx, long long rows, int E, cudaStream_t s) {
  if (rows * E == 0) return;
  scatter_rows_kernel<<<rows_grid(rows * E), 256, 0, s>>>(src, dst, idx, rows, E);
  check(cudaGetLastError(), "slab unpack");
}

template <typename T>
T* palloc(SlabPlan* sp, size_t count, const char* what, cudaStream_t s) {
  T* p = dalloc<T>(count, what);
  sp->owned.push_back(p);
  // zeroed once, ordered on the plan's stream before any upload into it: blocks
  // a simulated communicator does not deliver stay finite
  check(cudaMemsetAsync(p, 0, std::max<size_t>(count, 1) * sizeof(T), s), what);
  return p;
}

// column classes of a cx x cy column lattice under the sign flips of its axes,
// each class sorted, classes in order of their smallest column
std::vector<std::vector<int>> column_classes(long long cx, long long cy) {
  std::vector<int> cls(static_cast<size_t>(cx * cy), -1);
  std::vector<std::vector<int>> out;
  for (long long c = 0; c < cx * cy; ++c) {
    if (cls[c] >= 0) continue;
    const long long qx = c % cx, qy = c / cx;
    std::vector<int> ids;
    for (int f = 0; f < 4; ++f) {
      const long long x = (f & 1) ? (cx - qx) % cx : qx, y = (f & 2) ? (cy - qy) % cy : qy;
      ids.push_back(static_cast<int>(y * cx + x));
    }
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    for (int i : ids) cls[i] = static_cast<int>(out.size());
    out.push_back(ids);
  }
  return out;
}

// longest processing time first: classes by cost (desc, then index), each to
// the least loaded rank (lowest index on ties); deterministic on every rank
std::vector<int> assign_classes(const std::vector<double>& cost, int P) {
  std::vector<int> order(cost.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(P, 0.0);
  std::vector<int> owner(cost.size(), 0);
  for (int k : order) {
    const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    owner[k] = r;
    load[r] += cost[k];
  }
  return owner;
}

// the side's columns per rank, local indices, pack order and exchange sizes
void build_side(SlabPlan* sp, SlabSide& sd, const std::vector<std::vector<int>>& classes, const std::vector<int>& owner,
                cudaStream_t s) {
  const int P = sp->P, me = sp->rank;
  sd.cols.assign(P, {});
  sd.lc.assign(static_cast<size_t>(sd.C), -1);
  for (size_t k = 0; k < classes.size(); ++k)
    for (int c : classes[k]) sd.cols[owner[k]].push_back(c);
  for (int r = 0; r < P; ++r) {
    std::sort(sd.cols[r].begin(), sd.cols[r].end());
    for (size_t i = 0; i < sd.cols[r].size(); ++i) sd.lc[sd.cols[r][i]] = static_cast<int>(i);
  }
  const long long ms = sp->ms;
  std::vector<int> idx;
  idx.reserve(static_cast<size_t>(ms * sd.C));
  for (int d = 0; d < P; ++d)
    for (long long z = 0; z < ms; ++z)
      for (int c : sd.cols[d]) idx.push_back(static_cast<int>(z * sd.C + c));
  sd.n_idx = static_cast<long long>(idx.size());
  sd.idx = palloc<int>(sp, idx.size(), "slab pack order", s);
  h2d(sd.idx, idx.data(), idx.size() * sizeof(int), s, "slab pack order");
  const size_t E2 = 2 * static_cast<size_t>(sd.E);
  auto planes = [&](int r) { return static_cast<size_t>(sp->zlo[r + 1] - sp->zlo[r]); };
  const size_t mycols = sd.cols[me].size();
  sd.fsc.assign(P, 0);
  sd.fsd.assign(P, 0);
  sd.frc.assign(P, 0);
  sd.frd.assign(P, 0);
  sd.bsc.assign(P, 0);
  sd.bsd.assign(P, 0);
  sd.brc.assign(P, 0);
  sd.brd.assign(P, 0);
  sd.fall.assign(static_cast<size_t>(P) * P, 0);
  sd.ball.assign(static_cast<size_t>(P) * P, 0);
  size_t off = 0;
  for (int d = 0; d < P; ++d) {
    sd.fsc[d] = planes(me) * sd.cols[d].size() * E2;  // my planes, d's columns
    sd.fsd[d] = off;
    off += sd.fsc[d];
    sd.frc[d] = planes(d) * mycols * E2;  // d's planes, my columns
    sd.frd[d] = static_cast<size_t>(sp->zlo[d]) * mycols * E2;
    sd.bsc[d] = sd.frc[d];  // back: d's planes of my columns
    sd.bsd[d] = sd.frd[d];
    sd.brc[d] = sd.fsc[d];  // my planes of d's columns, in pack order
    sd.brd[d] = sd.fsd[d];
    for (int r = 0; r < P; ++r) {
      sd.fall[static_cast<size_t>(r) * P + d] = planes(r) * sd.cols[d].size() * E2;
      sd.ball[static_cast<size_t>(d) * P + r] = planes(r) * sd.cols[d].size() * E2;
    }
  }
  const size_t rows_loc = static_cast<size_t>(std::max(sp->Ms, sd.Ls)) * mycols;
  sd.pack = palloc<c64>(sp, static_cast<size_t>(ms * sd.C) * sd.E, "slab pack", s);
  sd.recv = palloc<c64>(sp, rows_loc * sd.E, "slab columns", s);
  sd.work = palloc<c64>(sp, rows_loc * sd.E, "slab column spectra", s);
}

void build_plan(fpbem_cu_op* op, fpbem_cu_comm* comm) {
  Nvtx range("slab plan");
  if (!op->near_fft) fail(FPBEM_CU_EINVAL, "set_slabs: needs the lattice near field (near_path = lattice)");
  if (op->mirrored_level >= 0) fail(FPBEM_CU_EINVAL, "set_slabs: not with a half-space image pair");
  auto* sp = new SlabPlan();
  op->slab = sp;  // owned by the handle from here (freed on failure by the caller's slab_destroy)
  cudaStream_t s = op->stream;
  sp->comm = comm;
  sp->P = comm ? comm->nranks : 1;
  sp->rank = comm ? comm->rank : 0;
  const int* M = op->counts;
  int ax = 0;
  for (int k = 2; k >= 0; --k)
    if (M[k] > 1) {
      ax = k;
      break;
    }
  sp->axis = ax;
  sp->Ms = M[ax];
  sp->mx = ax > 0 ? M[0] : 1;
  sp->my = ax > 1 ? M[1] : 1;
  sp->Cm = sp->mx * sp->my;
  const long long per = (sp->Ms + sp->P - 1) / sp->P;
  sp->zlo.resize(sp->P + 1);
  for (int r = 0; r <= sp->P; ++r) sp->zlo[r] = std::min(sp->Ms, per * r);
  sp->ms = sp->zlo[sp->rank + 1] - sp->zlo[sp->rank];

  // ---- near field: columns of the Ln lattice below the slab axis
  SlabSide& nr = sp->nr;
  nr.Ls = op->Ln[ax];
  nr.cx = ax > 0 ? op->Ln[0] : 1;
  nr.cy = ax > 1 ? op->Ln[1] : 1;
  nr.C = nr.cx * nr.cy;
  nr.E = op->n;
  const auto ncls = column_classes(nr.cx, nr.cy);
  std::vector<int> ncls_of(static_cast<size_t>(nr.C));
  for (size_t k = 0; k < ncls.size(); ++k)
    for (int c : ncls[k]) ncls_of[c] = static_cast<int>(k);
  std::vector<double> ncost(ncls.size(), 0.0);
  for (long long t = 0; t < op->n_items; ++t) ncost[ncls_of[op->items_q[t * 8] % nr.C]] += 1.0;
  const auto nown = assign_classes(ncost, sp->P);
  build_side(sp, nr, ncls, nown, s);
  // this rank's items (orbits never leave a column class): local modes
  // q = qs |cols| + local column, and their stored blocks
  const long long mycols = static_cast<long long>(nr.cols[sp->rank].size());
  std::vector<int> iq, ig;
  std::vector<long long> mine;
  for (long long t = 0; t < op->n_items; ++t) {
    if (nown[ncls_of[op->items_q[t * 8] % nr.C]] != sp->rank) continue;
    mine.push_back(t);
    for (int i = 0; i < 8; ++i) {
      const int q = op->items_q[t * 8 + i];
      iq.push_back(q < 0 ? -1 : static_cast<int>((q / nr.C) * mycols + nr.lc[q % nr.C]));
      ig.push_back(op->items_g[t * 8 + i]);
    }
  }
  sp->n_items = static_cast<long long>(mine.size());
  std::vector<int> items(iq);
  items.insert(items.end(), ig.begin(), ig.end());
  sp->items = palloc<int>(sp, items.size(), "slab items", s);
  h2d(sp->items, items.data(), items.size() * sizeof(int), s, "slab items");
  const size_t nn = static_cast<size_t>(op->n) * op->n;
  sp->shat = palloc<c64>(sp, mine.size() * nn, "slab near spectrum", s);
  for (size_t i = 0; i < mine.size(); ++i)
    check(cudaMemcpyAsync(sp->shat + i * nn, op->shat + static_cast<size_t>(mine[i]) * nn, nn * sizeof(c64),
                          cudaMemcpyDeviceToDevice, s),
          "slab near spectrum");

  // ---- far field: columns of the M2L lattice below the slab axis
  SlabSide& fr = sp->fr;
  fr.Ls = op->L[ax];
  fr.cx = ax > 0 ? op->L[0] : 1;
  fr.cy = ax > 1 ? op->L[1] : 1;
  fr.C = fr.cx * fr.cy;
  fr.E = op->b;
  const auto fcls = column_classes(fr.cx, fr.cy);
  std::vector<double> fcost(fcls.size());
  for (size_t k = 0; k < fcls.size(); ++k) fcost[k] = static_cast<double>(fcls[k].size());
  const auto fown = assign_classes(fcost, sp->P);
  build_side(sp, fr, fcls, fown, s);
  const std::vector<int>& fcols = fr.cols[sp->rank];
  const long long fmy = static_cast<long long>(fcols.size());
  const size_t b2 = static_cast<size_t>(op->b) * op->b;
  std::vector<int> lam_idx;  // local Λ rows (qs, local column) <- global q = qs C + col
  for (long long qs = 0; qs < fr.Ls; ++qs)
    for (int c : fcols) lam_idx.push_back(static_cast<int>(qs * fr.C + c));
  sp->lambda = palloc<c64>(sp, lam_idx.size() * b2, "slab spectrum", s);
  if (!lam_idx.empty()) {
    int* d_idx = dalloc<int>(lam_idx.size(), "slab spectrum rows");
    std::unique_ptr<int, decltype(&cudaFree)> keep(d_idx, &cudaFree);
    h2d(d_idx, lam_idx.data(), lam_idx.size() * sizeof(int), s, "slab spectrum rows");
    gather_rows(op->lambda, sp->lambda, d_idx, static_cast<long long>(lam_idx.size()), static_cast<int>(b2), s);
    check(cudaStreamSynchronize(s), "slab spectrum");
  }
  // the fused z kernel's items over local columns: a column with its mirror
  // (the Λ parity, when verified) or alone
  sp->zfused = fr.Ls > 1 && m2l_zfused_ring(static_cast<int>(sp->Ms), static_cast<int>(fr.Ls), op->b, op->b) > 0;
  if (sp->zfused) {
    std::vector<int2> zi;
    for (int c : fcols) {
      const long long qx = c % fr.cx, qy = c / fr.cx;
      const int cm = static_cast<int>(((fr.cy - qy) % fr.cy) * fr.cx + (fr.cx - qx) % fr.cx);
      const int l = fr.lc[c], lm = fr.lc[cm];
      if (!op->lam_paired)
        zi.push_back(make_int2(l, -1));
      else if (c < cm)
        zi.push_back(make_int2(l, lm));
      else if (c == cm)
        zi.push_back(make_int2(l, -1));
    }
    sp->n_zitems = static_cast<int>(zi.size());
    sp->zitems = palloc<int2>(sp, zi.size(), "slab z items", s);
    h2d(sp->zitems, zi.data(), zi.size() * sizeof(int2), s, "slab z items");
  }
  (void)fmy;
  const size_t planes = static_cast<size_t>(std::max(1LL, sp->ms));
  sp->a = palloc<c64>(sp, planes * static_cast<size_t>(nr.C * nr.E), "slab planes", s);
  sp->b = palloc<c64>(sp, planes * static_cast<size_t>(nr.C * nr.E), "slab planes", s);
  sp->fa = palloc<c64>(sp, planes * static_cast<size_t>(fr.C * fr.E), "slab far planes", s);
  sp->fb = palloc<c64>(sp, planes * static_cast<size_t>(fr.C * fr.E), "slab far planes", s);
  check(cudaEventCreateWithFlags(&sp->fork, cudaEventDisableTiming), "slab events");
  check(cudaEventCreateWithFlags(&sp->join, cudaEventDisableTiming), "slab events");
  sp->mom = palloc<c64>(sp, static_cast<size_t>(std::max(1LL, sp->ms * sp->Cm)) * op->b, "slab moments", s);
  sp->loc = palloc<c64>(sp, static_cast<size_t>(std::max(1LL, sp->ms * sp->Cm)) * op->b, "slab locals", s);
  check(cudaStreamSynchronize(s), "slab plan");
}

// forward DFTs along the column axes (x, then y when the slab axis is z) of
// this rank's planes: [ms][my][mx][E] -> [ms][cy][cx][E]; returns the result
// both column axes in one plane kernel (x and y DFTs per (plane, field) in
// shared memory) when the slab axis is z and the planes fit: half the launches
// of the axis passes, which matters at a few planes per rank (FPBEM_SLAB_XY=0:
// axis passes)
bool slab_xy(const SlabPlan* sp, const SlabSide& sd) {
  static const bool env = [] {
    const char* v = std::getenv("FPBEM_SLAB_XY");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  const int mx = static_cast<int>(sp->mx), my = static_cast<int>(sp->my);
  const int cx = static_cast<int>(sd.cx), cy = static_cast<int>(sd.cy);
  // the near side (E = n, hundreds of inner values) only for a few planes per rank: its
  // per-(plane, field) CTAs read n-strided values, which the axis passes beat from ~8
  // planes on (cfg3 at 2 ranks: 0.298 -> 0.286 ms with axis passes; 4, 8 ranks: the plane kernel)
  return env && sd.cx > 1 && sd.cy > 1 && sp->ms * sd.E <= 0x7fffffffLL && (sd.E <= 64 || sp->ms <= 4) &&
         xy_plane_smem(mx, my, cx, cy, false) <= 200 * 1024 && xy_plane_smem(mx, my, cx, cy, true) <= 200 * 1024;
}

const c64* local_forward(fpbem_cu_op* op, SlabPlan* sp, SlabSide& sd, const c64* in, c64* const* tw, cudaStream_t s,
                         c64* buf0, c64* buf1) {
  const c64* cur = in;
  c64* bufs[2] = {buf0, buf1};
  int which = 0;
  if (sp->ms == 0) return cur;
  if (slab_xy(sp, sd)) {
    check(launch_xy_plane(cur, bufs[0], tw[0], tw[1], static_cast<int>(sp->mx), static_cast<int>(sp->my),
                          static_cast<int>(sd.cx), static_cast<int>(sd.cy), static_cast<int>(sp->ms), sd.E, false, 1.0,
                          s),
          "slab xy dft");
    op->launches++;
    return bufs[0];
  }
  if (sd.cx > 1) {
    check(launch_dft_axis(cur, bufs[which], tw[0], sp->my * sp->ms, static_cast<int>(sp->mx), static_cast<int>(sd.cx),
                          sd.E, static_cast<int>(sd.cx), false, 1.0, s),
          "slab dft x");
    cur = bufs[which];
    which ^= 1;
    op->launches++;
  }
  if (sd.cy > 1) {
    check(launch_dft_axis(cur, bufs[which], tw[1], sp->ms, static_cast<int>(sp->my), static_cast<int>(sd.cy),
                          sd.cx * sd.E, static_cast<int>(sd.cy), false, 1.0, s),
          "slab dft y");
    cur = bufs[which];
    op->launches++;
  }
  return cur;
}

// inverse of local_forward from the unpacked planes `in` into `out`
// fuse_loc (near side): the L2P y += U0 L fused into the last (x) pass as its DMMA epilogue,
// after `join` (the far side's locals); returns whether it was fused
bool local_inverse(fpbem_cu_op* op, SlabPlan* sp, SlabSide& sd, const c64* in, c64* out, c64* const* tw,
                   cudaStream_t s, c64* spare, const c64* fuse_loc = nullptr, cudaEvent_t join = nullptr) {
  if (sp->ms == 0) return false;
  if (slab_xy(sp, sd)) {
    check(launch_xy_plane(in, out, tw[0], tw[1], static_cast<int>(sp->mx), static_cast<int>(sp->my),
                          static_cast<int>(sd.cx), static_cast<int>(sd.cy), static_cast<int>(sp->ms), sd.E, true, 1.0,
                          s),
          "slab inverse xy dft");
    op->launches++;
    return false;
  }
  const c64* cur = in;
  c64* tmp = spare;
  const int passes = (sd.cy > 1) + (sd.cx > 1);
  int done = 0;
  if (sd.cy > 1) {
    c64* dst = ++done == passes ? out : tmp;
    check(launch_dft_axis(cur, dst, tw[1], sp->ms, static_cast<int>(sd.cy), static_cast<int>(sp->my), sd.cx * sd.E,
                          static_cast<int>(sd.cy), true, 1.0, s),
          "slab inverse dft y");
    cur = dst;
    op->launches++;
  }
  bool fused = false;
  if (sd.cx > 1) {
    if (fuse_loc && dft_l2p_supported(static_cast<int>(sd.cx), static_cast<int>(sp->mx), op->b)) {
      check(cudaStreamWaitEvent(s, join, 0), "slab join");
      check(launch_dft_axis_l2p(cur, out, tw[0], sp->my * sp->ms, static_cast<int>(sd.cx), static_cast<int>(sp->mx),
                                sd.E, static_cast<int>(sd.cx), 1.0, op->u0, fuse_loc, op->b, 1, s),
            "slab inverse dft x + l2p");
      fused = true;
    } else {
      check(launch_dft_axis(cur, out, tw[0], sp->my * sp->ms, static_cast<int>(sd.cx), static_cast<int>(sp->mx),
                            sd.E, static_cast<int>(sd.cx), true, 1.0, s),
            "slab inverse dft x");
    }
    op->launches++;
  }
  return fused;
}

// stage timing of a slab product: [0] the two exchanges, [4] the whole
// product, [5] the near-field mode product (events 7-8)
void slab_timing(fpbem_cu_op* op, bool has_modes) {
  if (!op->timing) return;
  cudaStream_t s = op->stream;
  ev_record(op, 6, s);
  check(cudaEventSynchronize(op->ev[6]), "timing sync");
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, op->ev[1], op->ev[2]);
  cudaEventElapsedTime(&b, op->ev[3], op->ev[4]);
  op->stage_ms[0] += a + b;
  cudaEventElapsedTime(&a, op->ev[0], op->ev[6]);
  op->stage_ms[4] += a;
  if (has_modes) {
    cudaEventElapsedTime(&a, op->ev[7], op->ev[8]);
    op->stage_ms[5] += a;
  }
  op->applies++;
}

// phase 0: P2M, DFTs below the slab axis on this rank's planes, pack (far, then near)
// the far side of a phase runs on the aux stream, concurrently with the near
// side on the main one (independent buffers); fork before, join after
void slab_fork(fpbem_cu_op* op) {
  check(cudaEventRecord(op->slab->fork, op->stream), "slab fork");
  check(cudaStreamWaitEvent(op->aux, op->slab->fork, 0), "slab fork");
}
void slab_join(fpbem_cu_op* op) {
  check(cudaEventRecord(op->slab->join, op->aux), "slab join");
  check(cudaStreamWaitEvent(op->stream, op->slab->join, 0), "slab join");
}

void slab_phase0(fpbem_cu_op* op, const c64* x) {
  SlabPlan* sp = op->slab;
  cudaStream_t s = op->stream, a = op->aux;
  const long long cells = sp->ms * sp->Cm;
  SlabSide& nr = sp->nr;
  SlabSide& fr = sp->fr;
  slab_fork(op);
  if (cells > 0) {
    if (cellwise_supported(op->b, op->n))
      check(launch_cellwise(op->v0t, op->n, 1, op->b, op->n, x, cells * op->n, op->n, sp->mom, op->b, op->b, 1, cells,
                            false, a),
            "slab p2m");
    else
      check(launch_p2m(op->v0t, x, sp->mom, op->n, op->b, cells * op->n, 1, static_cast<int>(cells), a), "slab p2m");
    op->launches++;
  }
  const c64* fplanes = local_forward(op, sp, fr, sp->mom, op->tw, a, sp->fa, sp->fb);
  gather_rows(fplanes, fr.pack, fr.idx, fr.n_idx, fr.E, a);
  const c64* nplanes = local_forward(op, sp, nr, x, op->twn, s, sp->a, sp->b);
  gather_rows(nplanes, nr.pack, nr.idx, nr.n_idx, nr.E, s);
  op->launches += 2;
  slab_join(op);
}

// forward exchange (pack -> recv: every plane of my columns) or backward
// (work -> pack: my planes of every column), far and near in one group
void slab_exchange(fpbem_cu_op* op, bool forward) {
  SlabPlan* sp = op->slab;
  SlabSide& nr = sp->nr;
  SlabSide& fr = sp->fr;
  auto part = [&](SlabSide& sd) -> A2aPart {
    if (forward)
      return {reinterpret_cast<const double*>(sd.pack), reinterpret_cast<double*>(sd.recv), sd.fsc.data(),
              sd.fsd.data(), sd.frc.data(), sd.frd.data(), sd.fall.data()};
    return {reinterpret_cast<const double*>(sd.work), reinterpret_cast<double*>(sd.pack), sd.bsc.data(), sd.bsd.data(),
            sd.brc.data(), sd.brd.data(), sd.ball.data()};
  };
  const A2aPart parts[2] = {part(fr), part(nr)};
  ev_record(op, forward ? 1 : 3, op->stream);
  comm_alltoallv(sp->comm, parts, 2, op->stream);
  ev_record(op, forward ? 2 : 4, op->stream);
}

// phase 1: along the slab axis on my columns, recv -> work: far (M2L) then
// near (DFT, block products, inverse DFT)
void slab_phase1(fpbem_cu_op* op) {
  SlabPlan* sp = op->slab;
  cudaStream_t s = op->stream, a = op->aux;
  slab_fork(op);
  SlabSide& nr = sp->nr;
  SlabSide& fr = sp->fr;
  const long long ncols = static_cast<long long>(nr.cols[sp->rank].size());
  const long long fcols = static_cast<long long>(fr.cols[sp->rank].size());
  const double fscale = 1.0 / static_cast<double>(op->q_total), nscale = 1.0 / static_cast<double>(op->qn);
  const int ax = sp->axis;
  if (fcols > 0) {
    if (sp->zfused) {
      check(launch_m2l_zfused(fr.recv, fr.work, sp->lambda, op->tw[ax], static_cast<int>(sp->Ms),
                              static_cast<int>(fr.Ls), fcols, op->b, op->b, fscale, sp->zitems, sp->n_zitems, a),
            "slab m2l z-fused");
      op->launches++;
    } else {  // recv -> work -> recv -> work
      check(launch_dft_axis(fr.recv, fr.work, op->tw[ax], 1, static_cast<int>(sp->Ms), static_cast<int>(fr.Ls),
                            fcols * op->b, static_cast<int>(fr.Ls), false, 1.0, a),
            "slab m2l dft");
      check(launch_mode_product(sp->lambda, fr.work, fr.recv, fr.Ls * fcols, op->b, 1, a), "slab mode product");
      check(launch_dft_axis(fr.recv, fr.work, op->tw[ax], 1, static_cast<int>(fr.Ls), static_cast<int>(sp->Ms),
                            fcols * op->b, static_cast<int>(fr.Ls), true, fscale, a),
            "slab m2l inverse dft");
      op->launches += 3;
    }
  }
  if (ncols > 0) {  // recv -> work -> recv -> work
    check(launch_dft_axis(nr.recv, nr.work, op->twn[ax], 1, static_cast<int>(sp->Ms), static_cast<int>(nr.Ls),
                          ncols * op->n, static_cast<int>(nr.Ls), false, 1.0, s),
          "slab near dft");
    int nw_, kc_, ring_;
    size_t smem_;
    const long long qs = nr.Ls * ncols;  // rhs stride (one right-hand side)
    ev_record(op, 7, s);
    if (mode_mma_shape(op->n, op->near_nimg, &nw_, &kc_, &ring_, &smem_))
      check(launch_mode_mma(sp->shat, sp->items, sp->n_items, op->perm, nr.work, nr.recv, op->n, 0, sp->n_items, qs, 1,
                            op->near_nimg, s),
            "slab near mode product");
    else
      check(launch_mode_gemv(sp->shat, sp->items, sp->n_items, op->perm, nr.work, nr.recv, op->n, 0, sp->n_items, qs,
                             1, op->near_nimg, s),
            "slab near mode product");
    ev_record(op, 8, s);
    check(launch_dft_axis(nr.recv, nr.work, op->twn[ax], 1, static_cast<int>(nr.Ls), static_cast<int>(sp->Ms),
                          ncols * op->n, static_cast<int>(nr.Ls), true, nscale, s),
          "slab near inverse dft");
    op->launches += 3;
  }
  slab_join(op);
}

// phase 2: unpack, the inverse DFTs below the slab axis on my planes, L2P
void slab_phase2(fpbem_cu_op* op, c64* y) {
  SlabPlan* sp = op->slab;
  cudaStream_t s = op->stream;
  const long long cells = sp->ms * sp->Cm;
  if (cells == 0) return;
  SlabSide& nr = sp->nr;
  SlabSide& fr = sp->fr;
  const bool f_local = fr.cx > 1 || fr.cy > 1, n_local = nr.cx > 1 || nr.cy > 1;
  cudaStream_t a = op->aux;
  slab_fork(op);
  scatter_rows(fr.pack, f_local ? sp->fa : sp->loc, fr.idx, fr.n_idx, fr.E, a);
  if (f_local) local_inverse(op, sp, fr, sp->fa, sp->loc, op->tw, a, sp->fb);
  check(cudaEventRecord(sp->join, a), "slab join");  // the far side's locals
  scatter_rows(nr.pack, n_local ? sp->a : y, nr.idx, nr.n_idx, nr.E, s);
  const bool fused = n_local && local_inverse(op, sp, nr, sp->a, y, op->twn, s, sp->b, sp->loc, sp->join);
  check(cudaStreamWaitEvent(s, sp->join, 0), "slab join");
  if (!fused) {
    check(launch_l2p_add(op->u0, sp->loc, y, op->n, op->b, static_cast<int>(cells), cells * op->n, 1, s), "slab l2p");
    op->launches++;
  }
  op->launches += 2;
}

// y_loc = (A x)[this rank's planes] from x_loc = x[this rank's planes], one right-hand side
void apply_slab(fpbem_cu_op* op, const c64* x, c64* y) {
  Nvtx range("slab product");
  ev_record(op, 0, op->stream);
  slab_phase0(op, x);
  slab_exchange(op, true);
  slab_phase1(op);
  slab_exchange(op, false);
  slab_phase2(op, y);
  slab_timing(op, !op->slab->nr.cols[op->slab->rank].empty());
}

// capture one phase of the product (on the plan's slab vectors) as a graph
cudaGraphExec_t capture_phase(fpbem_cu_op* op, int ph, long long* launches) {
  SlabPlan* sp = op->slab;
  cudaStream_t s = op->stream;
  const long long l0 = op->launches;
  cudaGraph_t g = nullptr;
  check(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed), "slab graph capture");
  try {
    if (ph == 0) slab_phase0(op, sp->hx);
    if (ph == 1) slab_phase1(op);
    if (ph == 2) slab_phase2(op, sp->hy);
  } catch (...) {
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  check(cudaStreamEndCapture(s, &g), "slab graph capture");
  std::unique_ptr<CUgraph_st, decltype(&cudaGraphDestroy)> keep(g, &cudaGraphDestroy);
  cudaGraphExec_t exec = nullptr;
  check(cudaGraphInstantiate(&exec, g, 0), "slab graph instantiate");
  *launches = op->launches - l0;
  op->launches = l0;
  return exec;
}

// The product with each compute phase replayed as a CUDA graph: at a few planes
// per rank its ~20 small launches would otherwise leave the GPU waiting on the
// host's enqueue rate. The exchanges stay eager NCCL group calls between the
// graphs. Not under stage timing (event syncs) or with a host-staged
// communicator; FPBEM_SLAB_GRAPH=0 disables it. The graphs run on the plan's
// own slab vectors (hx -> hy), captured once per stream; a caller's vectors
// are copied in and out around them (device to device, one slab each), so the
// Krylov solver's changing basis columns reuse them.
void apply_slab_graph(fpbem_cu_op* op, const c64* x, c64* y) {
  static const bool env = [] {
    const char* v = std::getenv("FPBEM_SLAB_GRAPH");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  SlabPlan* sp = op->slab;
  cudaStream_t s = op->stream;
  if (!env || op->timing || (sp->comm && sp->comm->cb) || s == nullptr) {
    apply_slab(op, x, y);
    return;
  }
  Nvtx range("slab product (graphs)");
  const size_t rows = static_cast<size_t>(sp->ms * sp->Cm * op->n);
  if (!sp->hx) {
    sp->hx = palloc<c64>(sp, std::max<size_t>(rows, 1), "slab x", s);
    sp->hy = palloc<c64>(sp, std::max<size_t>(rows, 1), "slab y", s);
  }
  if (!sp->graph[0] || sp->graph_stream != s) {
    for (auto& g : sp->graph)
      if (g) {
        check(cudaGraphExecDestroy(g), "slab graph");
        g = nullptr;
      }
    sp->graph_launches = 0;
    for (int ph = 0; ph < 3; ++ph) {
      long long l = 0;
      sp->graph[ph] = capture_phase(op, ph, &l);
      sp->graph_launches += l;
    }
    sp->graph_stream = s;
  }
  if (rows && x != sp->hx)
    check(cudaMemcpyAsync(sp->hx, x, rows * sizeof(c64), cudaMemcpyDeviceToDevice, s), "slab x in");
  check(cudaGraphLaunch(sp->graph[0], s), "slab graph launch");
  slab_exchange(op, true);
  check(cudaGraphLaunch(sp->graph[1], s), "slab graph launch");
  slab_exchange(op, false);
  check(cudaGraphLaunch(sp->graph[2], s), "slab graph launch");
  if (rows && y != sp->hy)
    check(cudaMemcpyAsync(y, sp->hy, rows * sizeof(c64), cudaMemcpyDeviceToDevice, s), "slab y out");
  op->launches += sp->graph_launches;
}

}  // namespace

namespace fpbem_cu {
void slab_apply(fpbem_cu_op* op, const c64* x, c64* y) { apply_slab_graph(op, x, y); }
fpbem_cu_comm* slab_comm(const fpbem_cu_op* op) { return op->slab ? op->slab->comm : nullptr; }
void slab_range(const fpbem_cu_op* op, int r, long long* lo, long long* hi, long long* per_rank_rows) {
  const SlabPlan* sp = op->slab;
  const long long row = sp->Cm * op->n;
  *lo = sp->zlo[r] * row;
  *hi = sp->zlo[r + 1] * row;
  *per_rank_rows = (sp->Ms + sp->P - 1) / sp->P * row;
}
}  // namespace fpbem_cu

extern "C" {

int fpbem_cu_fmm_set_slabs(fpbem_cu_op* op, fpbem_cu_comm* comm) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "set_slabs: null op");
    check(cudaSetDevice(op->device), "set device");
    check(cudaStreamSynchronize(op->stream), "sync");
    slab_destroy(op);
    try {
      build_plan(op, comm);
    } catch (...) {
      slab_destroy(op);
      throw;
    }
  });
}

int fpbem_cu_fmm_slab_rows(const fpbem_cu_op* op, long long* lo, long long* hi) {
  return guard([&] {
    if (!op || !lo || !hi) fail(FPBEM_CU_EINVAL, "slab_rows: null argument");
    if (!op->slab) fail(FPBEM_CU_EINVAL, "slab_rows: no slab plan (fpbem_cu_fmm_set_slabs)");
    const SlabPlan* sp = op->slab;
    const long long row = sp->Cm * op->n;
    *lo = sp->zlo[sp->rank] * row;
    *hi = sp->zlo[sp->rank + 1] * row;
  });
}

int fpbem_cu_fmm_slab_info(const fpbem_cu_op* op, long long info[8]) {
  return guard([&] {
    if (!op || !info) fail(FPBEM_CU_EINVAL, "slab_info: null argument");
    if (!op->slab) fail(FPBEM_CU_EINVAL, "slab_info: no slab plan (fpbem_cu_fmm_set_slabs)");
    const SlabPlan* sp = op->slab;
    info[0] = sp->rank;
    info[1] = sp->P;
    info[2] = sp->axis;
    info[3] = sp->ms;
    info[4] = sp->n_items;
    info[5] = static_cast<long long>(sp->nr.cols[sp->rank].size()) * sp->nr.Ls;  // near modes on this rank
    info[6] = static_cast<long long>(sp->fr.cols[sp->rank].size()) * sp->fr.Ls;  // far modes on this rank
    info[7] = sp->zfused ? 1 : 0;
  });
}

int fpbem_cu_fmm_apply_slab(fpbem_cu_op* op, const fpbem_c64* x, fpbem_c64* y, int ptr_kind) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "apply_slab: null op");
    if (!op->slab) fail(FPBEM_CU_EINVAL, "apply_slab: no slab plan (fpbem_cu_fmm_set_slabs)");
    check(cudaSetDevice(op->device), "set device");
    SlabPlan* sp = op->slab;
    const size_t rows = static_cast<size_t>(sp->ms * sp->Cm * op->n);
    if (rows > 0 && (!x || !y)) fail(FPBEM_CU_EINVAL, "apply_slab: null vector");
    cudaStream_t s = op->stream;
    if (ptr_kind == FPBEM_CU_PTR_DEVICE) {
      apply_slab_graph(op, reinterpret_cast<const c64*>(x), reinterpret_cast<c64*>(y));
      return;
    }
    if (!sp->hx) {
      sp->hx = palloc<c64>(sp, std::max<size_t>(rows, 1), "slab x", s);
      sp->hy = palloc<c64>(sp, std::max<size_t>(rows, 1), "slab y", s);
    }
    // pinned host pointers overlap nothing here (one slab in, one out), so no chunking
    if (rows) check(cudaMemcpyAsync(sp->hx, x, rows * sizeof(c64), cudaMemcpyHostToDevice, s), "slab x upload");
    apply_slab_graph(op, sp->hx, sp->hy);
    if (rows) check(cudaMemcpyAsync(y, sp->hy, rows * sizeof(c64), cudaMemcpyDeviceToHost, s), "slab y download");
    check(cudaStreamSynchronize(s), "apply_slab");
  });
}

}  // extern "C"
