// The reference's public distance and geometry primitives on the device, with the
// same exact f64 recipe as the engine (exact subtract, the OpenBLAS ddot tree, sqrt):
//   block_distances / rowwise / nearest_centroid   distance.py:19-82
//   row_sqnorms                                    distance.py:66-72
//   centroid_geometry                              pruning.py:48-61
// Host-pointer entry points (copies in, one kernel, copies out) for callers that use
// these helpers directly; kmeans() never goes through here.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <string>

#include "../../include/knor_b200.h"
#include "common.cuh"

namespace knb {
int set_error(int code, const std::string& msg);
}

namespace {

using namespace knb;

// dist[i][j] = sqrt(sum((x_i - c_j)^2)) for every pair; ids/best: ascending strict-less
// argmin per row (distance.py:75-82: first occurrence of the minimum)
__global__ void pair_dist_kernel(const double* __restrict__ X, long long m, const double* __restrict__ C, int k,
                                 int d, double* __restrict__ dist) {
  const long long total = m * (long long)k;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    const long long i = p / k;
    const int j = (int)(p - i * k);
    dist[p] = sqrt(exact_sq_rt(X + i * d, C + (long long)j * d, d));
  }
}

__global__ void nearest_kernel(const double* __restrict__ X, long long m, const double* __restrict__ C, int k, int d,
                               int32_t* __restrict__ ids, double* __restrict__ best) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    double bd = CUDART_INF;
    int bi = 0;
    for (int j = 0; j < k; ++j) {
      const double dj = sqrt(exact_sq_rt(X + i * d, C + (long long)j * d, d));
      if (dj < bd) {
        bd = dj;
        bi = j;
      }
    }
    ids[i] = bi;
    best[i] = bd;
  }
}

// rowwise: row i of X against row i of R (or the single row R when shared)
__global__ void rowwise_kernel(const double* __restrict__ X, long long m, const double* __restrict__ R, int shared_ref,
                               int d, double* __restrict__ out, int take_sqrt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    const double s = R ? exact_sq_rt(X + i * d, R + (shared_ref ? 0 : i * d), d) : exact_self_rt(X + i * d, d);
    out[i] = take_sqrt ? sqrt(s) : s;
  }
}

int grid_for(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 65535) g = 65535;
  return (int)g;
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

#define PRIM_CUDA(x)                                                       \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) return set_error(KNB_E_CUDA, cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

extern "C" {

int knb_block_distances(int device, const double* rows, int64_t m, const double* cents, int32_t k, int32_t d,
                        double* dist_out, int32_t* ids_out, double* best_out) {
  if (m < 0 || k < 1 || d < 1 || (m > 0 && (!rows || !cents))) return set_error(KNB_E_ARG, "bad block_distances arguments");
  if (m == 0) return KNB_OK;
  PRIM_CUDA(cudaSetDevice(device));
  DevBuf X, C, D, I, B;
  PRIM_CUDA(cudaMalloc(&X.p, sizeof(double) * m * d));
  PRIM_CUDA(cudaMalloc(&C.p, sizeof(double) * (size_t)k * d));
  PRIM_CUDA(cudaMemcpy(X.p, rows, sizeof(double) * m * d, cudaMemcpyHostToDevice));
  PRIM_CUDA(cudaMemcpy(C.p, cents, sizeof(double) * (size_t)k * d, cudaMemcpyHostToDevice));
  if (dist_out) {
    PRIM_CUDA(cudaMalloc(&D.p, sizeof(double) * m * k));
    pair_dist_kernel<<<grid_for(m * k), 256>>>(static_cast<double*>(X.p), m, static_cast<double*>(C.p), k, d,
                                               static_cast<double*>(D.p));
    PRIM_CUDA(cudaGetLastError());
    PRIM_CUDA(cudaMemcpy(dist_out, D.p, sizeof(double) * m * k, cudaMemcpyDeviceToHost));
  }
  if (ids_out || best_out) {
    PRIM_CUDA(cudaMalloc(&I.p, sizeof(int32_t) * m));
    PRIM_CUDA(cudaMalloc(&B.p, sizeof(double) * m));
    nearest_kernel<<<grid_for(m), 256>>>(static_cast<double*>(X.p), m, static_cast<double*>(C.p), k, d,
                                         static_cast<int32_t*>(I.p), static_cast<double*>(B.p));
    PRIM_CUDA(cudaGetLastError());
    if (ids_out) PRIM_CUDA(cudaMemcpy(ids_out, I.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    if (best_out) PRIM_CUDA(cudaMemcpy(best_out, B.p, sizeof(double) * m, cudaMemcpyDeviceToHost));
  }
  return KNB_OK;
}

int knb_rowwise(int device, const double* rows, int64_t m, const double* refs, int32_t shared_ref, int32_t d,
                int32_t take_sqrt, double* out) {
  if (m < 0 || d < 1 || !out || (m > 0 && !rows)) return set_error(KNB_E_ARG, "bad rowwise arguments");
  if (m == 0) return KNB_OK;
  PRIM_CUDA(cudaSetDevice(device));
  DevBuf X, R, O;
  PRIM_CUDA(cudaMalloc(&X.p, sizeof(double) * m * d));
  PRIM_CUDA(cudaMemcpy(X.p, rows, sizeof(double) * m * d, cudaMemcpyHostToDevice));
  if (refs) {
    const size_t rn = shared_ref ? (size_t)d : (size_t)m * d;
    PRIM_CUDA(cudaMalloc(&R.p, sizeof(double) * rn));
    PRIM_CUDA(cudaMemcpy(R.p, refs, sizeof(double) * rn, cudaMemcpyHostToDevice));
  }
  PRIM_CUDA(cudaMalloc(&O.p, sizeof(double) * m));
  rowwise_kernel<<<grid_for(m), 256>>>(static_cast<double*>(X.p), m, static_cast<double*>(R.p), shared_ref, d,
                                       static_cast<double*>(O.p), take_sqrt);
  PRIM_CUDA(cudaGetLastError());
  PRIM_CUDA(cudaMemcpy(out, O.p, sizeof(double) * m, cudaMemcpyDeviceToHost));
  return KNB_OK;
}

}  // extern "C"
