// graph_store.cuh -- owner of one device-resident dynamic graph (G, H, the
// walk-phase shadow of G, or a snapshot). See dyg_internal.cuh for the slab
// layout. Host-side methods are stream-ordered on the stream passed in.
#pragma once

#include <stdint.h>

#include <string>

#include "dyg_internal.cuh"

namespace dyg {

struct DeviceError {
  int code;
  std::string message;
};

void cuda_check(cudaError_t e, const char* what);  // throws DeviceError

template <int C>
class GraphStore {
 public:
  GraphStore() = default;
  ~GraphStore();
  GraphStore(const GraphStore&) = delete;
  GraphStore& operator=(const GraphStore&) = delete;

  // Builds the slabs from a host CSR in reference row order.
  void upload(uint32_t n, const uint64_t* row_ptr, const uint32_t* ids, const double* w,
              cudaStream_t st);
  // Makes *this an exact copy of `other` (same n), D2D.
  void copy_from(const GraphStore& other, cudaStream_t st);
  // Row-order export to host buffers (row_ptr[n+1], ids/w[2m]).
  uint64_t export_rows(uint64_t* row_ptr, uint32_t* ids, double* w, uint64_t capacity,
                       cudaStream_t st);
  // Guarantees at least `free_entries` unused pool entries (grows the pool,
  // preserving indices). `top` is the last known pool_top.
  void ensure_pool(uint64_t top, uint64_t free_entries, cudaStream_t st);

  DevGraph<C> view() const { return v_; }
  uint32_t n() const { return v_.n; }
  uint64_t pool_capacity() const { return v_.pool_cap; }
  unsigned long long* edges_ptr() const { return v_.edges; }
  unsigned long long* pool_top_ptr() const { return v_.pool_top; }
  bool allocated() const { return v_.slab != nullptr; }
  void release();

 private:
  void allocate(uint32_t n, uint64_t pool_cap);
  DevGraph<C> v_{};
  unsigned long long* counters_ = nullptr;  // [0] pool_top, [1] edges
};

// Initial sparsifier on the device (init_sparsifier.cu): G as a host CSR in
// row order, H written to host buffers (row_ptr[n + 1]; ids / w with room
// for G's nnz). Throws DeviceError{1 usage | 2 data | 4 device}.
void build_initial_sparsifier_device(uint32_t n, const uint64_t* row_ptr, const uint32_t* ids,
                                     const double* w, double target_density, uint64_t seed,
                                     uint64_t* out_row_ptr, uint32_t* out_ids, double* out_w);

extern template class GraphStore<kCapH>;
extern template class GraphStore<kCapG>;

}  // namespace dyg
