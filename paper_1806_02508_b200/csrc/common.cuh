// common.cuh -- shared declarations for the sm_100a LB-BSP library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "lbbsp_c.h"

namespace lbbsp {

// Device-resident predictor bank: per-worker SpeedHistory (predictor.hpp:15-26)
// as SoA rows of max_hist doubles, incremental EMA state, NARX models.
struct PredDev {
  int n;
  int max_hist;
  int kind;
  double alpha;
  int warmup;
  double floor;
  lbbsp_narx_train_cfg train;  // min_history forced to warmup (predictor.cpp:264)
  double* hv;                  // [n][max_hist] speeds
  double* hc;                  // [n][max_hist] cpu availability
  double* hm;                  // [n][max_hist] mem availability
  double* ema;                 // [n] ema(history.speed) (predictor.cpp:18-28)
  double* comm_last;           // [n] newest comm observation
  double* comm_ema_lag;        // [n] ema(comm_obs[0..len-2]) (cluster_sim.cpp:383)
  lbbsp_narx_model* models;    // [n]
  lbbsp_narx_report* reports;  // [n] last training report
  double* scratch;             // [n][13*max_hist] global fallback for long histories
  int* len;                    // device scalar: observations per worker
  int* cursor;                 // device scalar: train_rotation cursor
};

constexpr int kTrainThreads = 256;

}  // namespace lbbsp

#define LBBSP_CUDA_CHECK(expr)                                                     \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      return ::lbbsp::set_error(LBBSP_CUDA, "%s: %s (%s:%d)", #expr,                \
                                cudaGetErrorString(_e), __FILE__, __LINE__);       \
    }                                                                              \
  } while (0)

namespace lbbsp {
int set_error(int code, const char* fmt, ...);
}
