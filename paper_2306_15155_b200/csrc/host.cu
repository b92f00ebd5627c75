// Host-side pieces of the C ABI: error/launch bookkeeping, the nnz-split SpMM
// planner and the multi-GPU row partitioner.  No device code here; all of it
// is callable (and tested) on a machine without a GPU.
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace gnnc {

static thread_local char g_err[512] = {0};
static std::atomic<uint64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

}  // namespace gnnc

using namespace gnnc;

extern "C" {

int gc_abi_version(void) { return GNNC_ABI_VERSION; }

const char *gc_last_error(void) { return g_err; }

uint64_t gc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int gc_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaDeviceGetAttribute failed for device %d", device);
    return GC_ERR_CUDA;
  }
  return v;
}

// ---- nnz-split SpMM planner ---------------------------------------------
int gc_spmm_plan_count(const int32_t *row_ptr_host, int64_t n_rows, int32_t chunk,
                       int64_t *n_items, int64_t *n_slots, int64_t *n_split_rows) {
  GC_REQUIRE(row_ptr_host && n_items && n_slots && n_split_rows, GC_ERR_VALUE,
             "gc_spmm_plan_count: null pointer");
  GC_REQUIRE(n_rows >= 0, GC_ERR_SHAPE, "gc_spmm_plan_count: n_rows < 0");
  GC_REQUIRE(chunk >= 1, GC_ERR_VALUE, "gc_spmm_plan_count: chunk must be >= 1");
  int64_t items = 0, slots = 0, split = 0;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t deg = (int64_t)row_ptr_host[i + 1] - row_ptr_host[i];
    GC_REQUIRE(deg >= 0, GC_ERR_SHAPE, "gc_spmm_plan_count: row_ptr decreases at row %lld",
               (long long)i);
    if (deg > chunk) {
      const int64_t c = (deg + chunk - 1) / chunk;
      items += c;
      slots += c;
      split += 1;
    } else {
      items += 1;
    }
  }
  GC_REQUIRE(items < INT32_MAX && slots < INT32_MAX, GC_ERR_SHAPE,
             "gc_spmm_plan_count: plan too large");
  *n_items = items;
  *n_slots = slots;
  *n_split_rows = split;
  return GC_OK;
}

int32_t gc_spmm_default_chunk(int64_t n_rows, int64_t nnz, int64_t K, int sm_count) {
  (void)n_rows;
  // lanes per row group, as chosen by gc_spmm_f32's vector path
  const int lpr = K <= 8 ? 2 : K <= 16 ? 4 : K <= 32 ? 8 : K <= 64 ? 16 : 32;
  const int64_t groups = (int64_t)(sm_count > 0 ? sm_count : 148) * 48 * (32 / lpr);
  const int64_t target = 2 * (nnz / (groups > 0 ? groups : 1));
  int64_t c = 128;
  while (c < target && c < 4096) c <<= 1;
  return (int32_t)c;
}

int gc_spmm_plan_fill(const int32_t *row_ptr_host, int64_t n_rows, int32_t chunk,
                      uint32_t plan_flags, int32_t *items_host, int32_t *split_rows_host) {
  GC_REQUIRE(row_ptr_host && items_host, GC_ERR_VALUE, "gc_spmm_plan_fill: null pointer");
  GC_REQUIRE(chunk >= 1, GC_ERR_VALUE, "gc_spmm_plan_fill: chunk must be >= 1");
  GC_REQUIRE((plan_flags & ~GC_PLAN_LENGTH_CLASSES) == 0, GC_ERR_VALUE,
             "gc_spmm_plan_fill: unknown flags");
  std::vector<int32_t> nat;  // items in natural (row) order
  nat.reserve((size_t)n_rows * 4);
  int64_t slot = 0, sr = 0;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int32_t b = row_ptr_host[i], e = row_ptr_host[i + 1];
    const int64_t deg = (int64_t)e - b;
    if (deg > chunk) {
      GC_REQUIRE(split_rows_host, GC_ERR_VALUE, "gc_spmm_plan_fill: split_rows is null");
      const int64_t c = (deg + chunk - 1) / chunk;
      split_rows_host[4 * sr + 0] = (int32_t)i;
      split_rows_host[4 * sr + 1] = (int32_t)slot;
      split_rows_host[4 * sr + 2] = (int32_t)c;
      split_rows_host[4 * sr + 3] = 0;
      ++sr;
      for (int64_t q = 0; q < c; ++q) {
        const int32_t lo = b + (int32_t)(q * chunk);
        const int32_t hi = (int32_t)std::min<int64_t>((int64_t)lo + chunk, e);
        nat.insert(nat.end(), {(int32_t)i, lo, hi, (int32_t)slot++});
      }
    } else {
      nat.insert(nat.end(), {(int32_t)i, b, e, -1});
    }
  }
  const size_t n_items = nat.size() / 4;
  if (!(plan_flags & GC_PLAN_LENGTH_CLASSES)) {
    std::copy(nat.begin(), nat.end(), items_host);
    return GC_OK;
  }
  // stable counting sort by length class, longest class first
  auto cls = [&](size_t k) {
    const int32_t len = nat[4 * k + 2] - nat[4 * k + 1];
    int c = 0;
    while ((1 << (c + 1)) <= len && c < 30) ++c;
    return len == 0 ? 0 : c + 1;
  };
  size_t start[33] = {0};
  for (size_t k = 0; k < n_items; ++k) ++start[cls(k)];
  size_t acc = 0;
  for (int c = 32; c >= 0; --c) {
    const size_t cnt = start[c];
    start[c] = acc;
    acc += cnt;
  }
  for (size_t k = 0; k < n_items; ++k) {
    const size_t dst = start[cls(k)]++;
    std::copy(nat.begin() + 4 * k, nat.begin() + 4 * k + 4, items_host + 4 * dst);
  }
  return GC_OK;
}

// ---- row partition ----------------------------------
int gc_partition_rows(const int64_t *row_ptr_host, int64_t n_rows, int32_t parts,
                      int64_t *bounds_host) {
  GC_REQUIRE(row_ptr_host && bounds_host, GC_ERR_VALUE, "gc_partition_rows: null pointer");
  GC_REQUIRE(parts >= 1, GC_ERR_VALUE, "gc_partition_rows: parts must be >= 1");
  GC_REQUIRE(n_rows >= 0, GC_ERR_SHAPE, "gc_partition_rows: n_rows < 0");
  const int64_t m = row_ptr_host[n_rows];
  bounds_host[0] = 0;
  bounds_host[parts] = n_rows;
  for (int32_t p = 1; p < parts; ++p) {
    // ceil(p*m/P) without overflow for m < 2^62 / P
    const int64_t target = (p * m + parts - 1) / parts;
    const int64_t *hit = std::lower_bound(row_ptr_host, row_ptr_host + n_rows + 1, target);
    bounds_host[p] = std::min<int64_t>(hit - row_ptr_host, n_rows);
  }
  return GC_OK;
}

}  // extern "C"
