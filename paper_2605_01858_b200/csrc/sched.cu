// Host-side launch helpers of the tcgen05 attention kernel: per-CTA work lists (list
// scheduling of the persistent CTAs) and the K/V tensor maps.
//
// Work lists: items in launch order (attend first, then build; longest first inside each)
// each go to the CTA with the least work so far (cost = key tiles + kSwitchCost for the item
// switch).  The static stride b, b + grid, ... gives some CTAs two long attend items AND a
// full share of builds when item lengths differ a lot (c3, c4).  Lists are kept only where
// they shorten the makespan estimate by > 2% (c5's stride is balanced already and keeps
// the ORDER 2 L2 locality).
//
// The cache is owned by one handle.  Every entry is written ONCE (an async upload on the
// stream that first asked for it, followed by an event) and never rewritten or freed before
// the handle is destroyed, so a kernel queued on any stream can never see a list change
// under it; a request from another stream waits on the upload's event.
#include "dscache_internal.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

namespace dsc {

struct SchedCache {
  struct Entry {
    int* dev = nullptr;           // nullptr: the stride is kept (no list)
    cudaEvent_t ready = nullptr;  // upload done
    cudaStream_t stream = nullptr;
  };
  std::map<std::vector<long long>, Entry> tables;   // item tables: [grid + 1 offsets | pad | ItemRec[]]
  std::mutex mu;
  size_t bytes = 0;
};

SchedCache* sched_cache_new() { return new SchedCache(); }

void sched_cache_free(SchedCache* c) {
  if (!c) return;
  for (auto& kv : c->tables) {
    if (kv.second.ready) cudaEventDestroy(kv.second.ready);
    if (kv.second.dev) cudaFree(kv.second.dev);
  }
  delete c;
}

namespace {
constexpr long long kSwitchCost = 2;              // item-switch cost in key tiles
constexpr size_t kMaxCacheBytes = 256ull << 20;   // beyond this, new shapes fall back to the stride
}  // namespace

namespace {
std::vector<long long> shape_key(int device, const AttnParams& pa, const AttnParams* pb, long long na, long long nb,
                                 unsigned grid) {
  std::vector<long long> key = {device, na, nb, (long long)grid};
  for (const AttnParams* p : {&pa, pb}) {
    if (!p) continue;
    for (long long v : {(long long)p->n_splits, (long long)p->split_only, (long long)p->P, (long long)p->Hkv,
                        (long long)p->n_mblocks, (long long)p->n_q, (long long)p->grp, (long long)p->q_pos0,
                        (long long)p->A, (long long)p->ring_count, (long long)p->n_self,
                        (long long)p->tiles_per_split, (long long)p->layer_count, (long long)p->layer_begin,
                        (long long)p->N_total, (long long)p->Rp, (long long)p->staged})
      key.push_back(v);
  }
  return key;
}
}  // namespace

const ItemRec* item_table(SchedCache* cache, const AttnParams& pa, const AttnParams* pb, long long na, long long nb,
                          unsigned grid, ItemDecoder dec, const int** off_out, cudaStream_t st) {
  if (!cache) return nullptr;
  std::lock_guard<std::mutex> lock(cache->mu);
  int device = 0;
  cudaGetDevice(&device);
  std::vector<long long> key = shape_key(device, pa, pb, na, nb, grid);
  const size_t off_bytes = ((grid + 1) * sizeof(int) + 31) & ~size_t(31);
  auto it = cache->tables.find(key);
  if (it != cache->tables.end()) {
    const SchedCache::Entry& e = it->second;
    if (!e.dev) return nullptr;
    // another stream uploaded it: wait for the upload unless it has already landed (so a
    // steady-state step can be captured into a CUDA graph on another stream)
    if (e.stream != st && e.ready && cudaEventQuery(e.ready) != cudaSuccess) cudaStreamWaitEvent(st, e.ready, 0);
    *off_out = e.dev;
    return reinterpret_cast<const ItemRec*>(reinterpret_cast<const char*>(e.dev) + off_bytes);
  }
  const long long items = na + nb;
  std::vector<ItemRec> rec(items);
  for (long long I = 0; I < items; ++I) {
    const bool isb = I >= na;
    rec[I] = dec(isb ? *pb : pa, (int)(isb ? I - na : I), isb ? 1 : 0);
  }
  // list scheduling vs the static stride (cost = key tiles + the item-switch cost)
  std::vector<int> owner(items);
  std::vector<long long> stride_load(grid, 0);
  std::vector<std::pair<long long, int>> heap;
  heap.reserve(grid);
  for (unsigned b = 0; b < grid; ++b) heap.push_back({0, (int)b});
  auto cmp = [](const std::pair<long long, int>& x, const std::pair<long long, int>& y) { return x > y; };
  std::make_heap(heap.begin(), heap.end(), cmp);
  for (long long I = 0; I < items; ++I) {
    const long long cost = rec[I].n_tiles + kSwitchCost;
    stride_load[I % grid] += cost;
    std::pop_heap(heap.begin(), heap.end(), cmp);
    owner[I] = heap.back().second;
    heap.back().first += cost;
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  long long list_max = 0;
  for (auto& h : heap) list_max = std::max(list_max, h.first);
  const long long stride_max = *std::max_element(stride_load.begin(), stride_load.end());
  if (!(list_max * 50 < stride_max * 49))
    for (long long I = 0; I < items; ++I) owner[I] = (int)(I % grid);
  std::vector<int> off(grid + 1, 0);
  for (long long I = 0; I < items; ++I) ++off[owner[I] + 1];
  for (unsigned b = 0; b < grid; ++b) off[b + 1] += off[b];
  std::vector<char> host(off_bytes + items * sizeof(ItemRec), 0);
  std::memcpy(host.data(), off.data(), (grid + 1) * sizeof(int));
  ItemRec* dst = reinterpret_cast<ItemRec*>(host.data() + off_bytes);
  std::vector<int> fill(off.begin(), off.end() - 1);
  for (long long I = 0; I < items; ++I) dst[fill[owner[I]]++] = rec[I];   // increasing I per CTA
  SchedCache::Entry e;
  if (cache->bytes + host.size() > kMaxCacheBytes) return nullptr;
  // stream-ordered allocation: no implicit synchronisation, so a new launch shape (every
  // warm-up step of a stream has one) does not drain the GPU pipeline
  if (cudaMallocAsync(&e.dev, host.size(), st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cudaMemcpyAsync(e.dev, host.data(), host.size(), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(e.ready, st) != cudaSuccess) {
    cudaGetLastError();
    if (e.ready) cudaEventDestroy(e.ready);
    cudaFreeAsync(e.dev, st);
    return nullptr;
  }
  e.stream = st;
  cache->bytes += host.size();
  cache->tables.emplace(std::move(key), e);
  *off_out = e.dev;
  return reinterpret_cast<const ItemRec*>(reinterpret_cast<const char*>(e.dev) + off_bytes);
}

// 2-D tensor map of a K/V row buffer [rows][128] bf16 (ring + mirror rows, or a staging
// buffer), box 64 columns x box_rows rows, 128-byte swizzle (the SW128 K-major / MN-major
// operand layout of the tcgen05 descriptors).
cudaError_t make_kv_tmap(CUtensorMap* map, void* base, unsigned long long rows, int box_rows) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
      if (e != cudaSuccess || fn == nullptr) return e != cudaSuccess ? e : cudaErrorNotSupported;
      encode = reinterpret_cast<Encode>(fn);
    }
  }
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {128 * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace dsc
