// spectral.cuh -- condition number, budget calibration and PCG on the device
// (SURVEY.md 8f rows 3-4). See spectral.cu.
#pragma once

#include <stdint.h>

#include <vector>

#include "dyg_internal.cuh"

namespace dyg {

struct HostCsrView {  // reference row order (graph.hpp:37-38)
  uint32_t n;
  const uint64_t* row_ptr;
  const uint32_t* ids;
  const double* w;
};

// A graph Laplacian on the device: CSR rows plus the weighted degree per row
// (laplacian.cpp:7-26 without materialising the diagonal).
struct DevLap {
  uint32_t n = 0;
  uint64_t* rp = nullptr;
  uint32_t* ids = nullptr;
  double* w = nullptr;
  double* dw = nullptr;
};

class DevLapOwner {
 public:
  DevLapOwner(const HostCsrView& g, cudaStream_t st);
  ~DevLapOwner();
  DevLapOwner(const DevLapOwner&) = delete;
  DevLapOwner& operator=(const DevLapOwner&) = delete;
  DevLap L;
};

// Vector algebra over n doubles on one stream; scalars come back through
// pinned memory (one synchronisation per scalar the host needs).
class SpectralEngine {
 public:
  explicit SpectralEngine(uint32_t n);
  ~SpectralEngine();
  SpectralEngine(const SpectralEngine&) = delete;
  SpectralEngine& operator=(const SpectralEngine&) = delete;

  cudaStream_t stream() const { return st_; }
  double* vec();  // an n-vector owned by the engine
  void lap(const DevLap& L, const double* x, double* y);
  double dot(const double* x, const double* y);  // y == nullptr: x . x
  double sum(const double* x);
  void center(double* x);
  void axpy_host(double* x, const double* y, double a);  // x += a y
  void scale(double* x, double a);
  void copy(double* dst, const double* src);
  void upload(double* dst, const double* host);
  void download(double* host, const double* src);
  // x = L^+ b on the zero-mean subspace by CG (solver.cpp:50-68) to relative
  // residual rel_tol; r, p, q are scratch vectors. Returns the iterations.
  uint32_t cg_solve(const DevLap& L, const double* b, double* x, double rel_tol, double* r,
                    double* p, double* q);

 private:
  double fetch(const double* dev_scalar);
  uint32_t n_;
  cudaStream_t st_ = nullptr;
  double* part_ = nullptr;
  double* sc_ = nullptr;
  int* done_ = nullptr;
  unsigned* iters_ = nullptr;
  double* host_ = nullptr;
  std::vector<double*> scratch_;
};

// Fill-reducing orderings reused across factorisations (spectral.cu):
// cumulative exact-pattern hits, near-pattern hits and fresh orderings.
void ordering_cache_stats(uint64_t* hits, uint64_t* near_hits, uint64_t* misses);

// GroundedLaplacianSolver (laplacian.cpp:57-85) on the device: sparse
// Cholesky of the grounded Laplacian (METIS ordering, cuSOLVER csrchol),
// factorised once, solved many times.
class GroundedChol {
 public:
  GroundedChol(const HostCsrView& g, cudaStream_t st);
  ~GroundedChol();
  GroundedChol(const GroundedChol&) = delete;
  GroundedChol& operator=(const GroundedChol&) = delete;
  // x = L^+ b on the zero-mean subspace; tmp is an n-vector of scratch.
  void solve(SpectralEngine& e, const double* b, double* x, double* tmp);

 private:
  void build(const HostCsrView& g);
  void release();
  cudaStream_t st_;
  uint32_t m_ = 0;
  int nnz_ = 0;
  void* handle_ = nullptr;
  void* descr_ = nullptr;
  void* info_ = nullptr;
  int* d_rp_ = nullptr;
  int* d_ci_ = nullptr;
  double* d_val_ = nullptr;
  int* d_perm_ = nullptr;
  double* d_bp_ = nullptr;
  double* d_xp_ = nullptr;
  char* buffer_ = nullptr;
};

struct ConditionParams {  // ConditionOptions (spectral.hpp:78-85)
  double tolerance = 1e-6;
  uint32_t max_iterations = 400;
  uint64_t seed = 0x5eed;
  double inner_tol = 1e-12;  // L_H solves (the reference factorises exactly)
};

struct ConditionResult {  // ConditionEstimate (spectral.hpp:69-76)
  double kappa = 1.0;
  double lambda_max = 1.0;
  double lambda_min = 1.0;
  int method = 0;  // 0 Dense, 1 Iterative
  uint32_t iterations = 0;
  int converged = 1;
  uint64_t inner_iterations = 0;
};

struct PcgOutcome {  // PcgResult (solver.hpp:44-49) without the solution
  uint32_t iterations = 0;
  double relative_residual = 0.0;
  int converged = 0;
  uint64_t inner_iterations = 0;
};

ConditionResult condition_dense_device(const DevLap& G, const DevLap& H, cudaStream_t st);
ConditionResult condition_lanczos_device(const DevLap& G, const DevLap& H,
                                         const HostCsrView& h_host, const ConditionParams& prm);
PcgOutcome pcg_device(const DevLap& G, const DevLap* H, const HostCsrView* h_host, bool factorized,
                      const double* rhs_host, double tolerance, uint32_t max_iterations,
                      double inner_tol, double* x_host, std::vector<double>* energy);

}  // namespace dyg
