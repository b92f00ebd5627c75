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

int gc_spmm_plan_fill(const int32_t *row_ptr_host, int64_t n_rows, int32_t chunk,
                      int32_t *items_host, int32_t *split_rows_host) {
  GC_REQUIRE(row_ptr_host && items_host, GC_ERR_VALUE, "gc_spmm_plan_fill: null pointer");
  GC_REQUIRE(chunk >= 1, GC_ERR_VALUE, "gc_spmm_plan_fill: chunk must be >= 1");
  int64_t it = 0, slot = 0, sr = 0;
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
        items_host[4 * it + 0] = (int32_t)i;
        items_host[4 * it + 1] = lo;
        items_host[4 * it + 2] = hi;
        items_host[4 * it + 3] = (int32_t)slot++;
        ++it;
      }
    } else {
      items_host[4 * it + 0] = (int32_t)i;
      items_host[4 * it + 1] = b;
      items_host[4 * it + 2] = e;
      items_host[4 * it + 3] = -1;
      ++it;
    }
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
