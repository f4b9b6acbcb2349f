// solver.cuh -- K1/K2: the batch-size solvers as block-cooperative device
// functions. Every thread of the block must call them (they __syncthreads).
//
//   block_cpu_allocate : clamp_speed_floor (batch_sizer.cpp:12-14) +
//                        cpu_allocate      (batch_sizer.cpp:54-99)
//   block_gpu_allocate : gpu_allocate      (batch_sizer.cpp:101-199)
//
// Bit-exactness rules: fp64 with no contraction (exactmath.cuh),
// every floating-point reduction the reference does left-to-right is done
// left-to-right by one thread, and the stable sort is replaced by the total
// order (remainder desc, index asc), computed as a parallel rank.
#pragma once
#include "common.cuh"
#include "exactmath.cuh"

namespace lbbsp {

struct SolverSmem {
  double sum;
  int assigned;
  int code;
  int what;
  long long a, b;
  int first_b;
  double level;
};

__device__ __forceinline__ void set_status(lbbsp_dev_status* st, int code, int what, long long a,
                                           long long b) {
  if (st && st->code == 0) {
    st->code = code;
    st->what = what;
    st->a = a;
    st->b = b;
  }
}

// Warp-0 helper: index of the first maximum of sizes[0..n) (std::max_element).
__device__ __forceinline__ int warp_first_max(const int* sizes, int n) {
  const int lane = threadIdx.x & 31;
  int best = -1, bv = 0;
  for (int i = lane; i < n; i += 32) {
    const int v = sizes[i];
    if (best < 0 || v > bv) {  // strided scan keeps the lowest index per lane
      best = i;
      bv = v;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const int ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int ov = __shfl_xor_sync(0xffffffffu, bv, off);
    if (ob >= 0 && (best < 0 || ov > bv || (ov == bv && ob < best))) {
      best = ob;
      bv = ov;
    }
  }
  return best;
}

// min-1 repair (batch_sizer.cpp:90-97) by warp 0: sequential over i, the
// deficit taken from the first maximum. Returns false if impossible.
__device__ inline bool warp_min1_repair(int* sizes, int n) {
  const int tid = threadIdx.x;
  int need = 0;
  for (int i = tid; i < n; i += 32) need |= sizes[i] < 1;
  need = __any_sync(0xffffffffu, need);
  if (!need) return true;
  for (int i = 0; i < n; ++i) {
    __syncwarp();
    int xi = sizes[i];
    while (xi < 1) {
      const int big = warp_first_max(sizes, n);
      if (sizes[big] <= 1) return false;  // warp-uniform
      __syncwarp();
      if (tid == 0) {
        sizes[big] -= 1;
        sizes[i] += 1;
      }
      __syncwarp();
      xi = sizes[i];
    }
  }
  return true;
}

// cpu_allocate for n <= 32 in warp 0 (the plan's case): one lane per worker,
// the left-to-right sum formed redundantly in every lane from shuffled
// values (the same dadd sequence), the largest-remainder rank by shuffles --
// no shared-memory round trips or block barriers on the way, and rolled
// loops: the plan runs once per round from a cold instruction cache, so its
// latency follows its code size.
__device__ inline int warp_cpu_allocate(const double* speeds, int n, int budget, double speed_floor, int* sizes,
                                        SolverSmem* sm, lbbsp_dev_status* st) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    const unsigned full = 0xffffffffu;
    int code = 0, what = 0;
    double v = 1.0;
    if (tid < n) {
      v = speeds[tid];
      if (speed_floor > 0.0) v = v > speed_floor ? v : speed_floor;
    }
    if (budget < n) {
      code = LBBSP_INVALID_ARGUMENT;
      what = LBBSP_E_CPU_BUDGET;
    } else if (__ballot_sync(full, tid < n && !(v > 0.0))) {
      code = LBBSP_INVALID_ARGUMENT;
      what = LBBSP_E_CPU_SPEED;
    }
    if (!code) {
      double sum = 0.0;  // batch_sizer.cpp:60-64, left to right
#pragma unroll 1
      for (int i = 0; i < n; ++i) sum = dadd(sum, __shfl_sync(full, v, i));
      const double share = dmul(ddiv(v, sum), static_cast<double>(budget));  // :72-73
      const double fl = floor(share);
      const int sz = static_cast<int>(fl);
      const double r = dsub(share, fl);
      const int extra = budget - __reduce_add_sync(full, tid < n ? sz : 0);
      // largest remainder, ties to the lower index (:81-87)
      int rank = 0;
#pragma unroll 1
      for (int j = 0; j < n; ++j) {
        const double rj = __shfl_sync(full, r, j);
        rank += (rj > r) || (rj == r && j < tid);
      }
      if (tid < n) sizes[tid] = sz + (rank < extra ? 1 : 0);
      __syncwarp();
      if (!warp_min1_repair(sizes, n)) {
        code = LBBSP_LOGIC;
        what = LBBSP_E_CPU_MIN1;
      }
    }
    if (tid == 0) {
      sm->code = code;
      if (code) {
        sm->what = what;
        sm->a = what == LBBSP_E_CPU_BUDGET ? budget : 0;
        sm->b = what == LBBSP_E_CPU_BUDGET ? n : 0;
        set_status(st, code, what, sm->a, sm->b);
      }
    }
  }
  __syncthreads();
  return sm->code;
}

// speeds: [n] (global or shared). sizes: [n] output (shared or global).
// rem: [n] shared scratch. Returns 0 or a status code (also written to st).
__device__ inline int block_cpu_allocate(const double* speeds, int n, int budget, double speed_floor,
                                  int* sizes, double* rem, SolverSmem* sm,
                                  lbbsp_dev_status* st) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (n >= 1 && n <= 32 && nt >= 32) return warp_cpu_allocate(speeds, n, budget, speed_floor, sizes, sm, st);
  if (tid == 0) {
    sm->code = 0;
    sm->assigned = 0;
    if (n == 0) {
      sm->code = LBBSP_INVALID_ARGUMENT;
      sm->what = LBBSP_E_CPU_NO_WORKERS;
    } else if (budget < n) {
      sm->code = LBBSP_INVALID_ARGUMENT;
      sm->what = LBBSP_E_CPU_BUDGET;
      sm->a = budget;
      sm->b = n;
    } else {
      double sum = 0.0;  // batch_sizer.cpp:60-64, left to right
      for (int i = 0; i < n; ++i) {
        double v = speeds[i];
        if (speed_floor > 0.0) v = v > speed_floor ? v : speed_floor;
        if (!(v > 0.0)) {
          sm->code = LBBSP_INVALID_ARGUMENT;
          sm->what = LBBSP_E_CPU_SPEED;
          break;
        }
        sum = dadd(sum, v);
      }
      sm->sum = sum;
    }
    if (sm->code) set_status(st, sm->code, sm->what, sm->a, sm->b);
  }
  __syncthreads();
  if (sm->code) return sm->code;
  const double sum = sm->sum;
  const double Bd = static_cast<double>(budget);
  int local = 0;
  for (int i = tid; i < n; i += nt) {
    double v = speeds[i];
    if (speed_floor > 0.0) v = v > speed_floor ? v : speed_floor;
    const double share = dmul(ddiv(v, sum), Bd);  // :72-73
    const double fl = floor(share);
    sizes[i] = static_cast<int>(fl);
    rem[i] = dsub(share, fl);
    local += static_cast<int>(fl);
  }
  if (local) atomicAdd(&sm->assigned, local);
  __syncthreads();
  const int extra = budget - sm->assigned;
  // largest remainder, ties to the lower index (:81-87)
  for (int i = tid; i < n; i += nt) {
    const double ri = rem[i];
    int rank = 0;
    for (int j = 0; j < n && rank < extra; ++j) {
      const double rj = rem[j];
      rank += (rj > ri) || (rj == ri && j < i);
    }
    if (rank < extra) sizes[i] += 1;
  }
  __syncthreads();
  // min-1 repair (:90-97): sequential over i, deficit taken from the first max
  if (tid < 32) {
    int need = 0;
    for (int i = tid; i < n; i += 32) need |= sizes[i] < 1;
    need = __any_sync(0xffffffffu, need);
    if (need) {
      bool fail = false;
      for (int i = 0; i < n && !fail; ++i) {
        __syncwarp();
        int xi = sizes[i];
        while (xi < 1) {
          const int big = warp_first_max(sizes, n);
          if (sizes[big] <= 1) {
            fail = true;  // warp-uniform
            if (tid == 0) {
              sm->code = LBBSP_LOGIC;
              set_status(st, LBBSP_LOGIC, LBBSP_E_CPU_MIN1, 0, 0);
            }
            break;
          }
          __syncwarp();
          if (tid == 0) {
            sizes[big] -= 1;
            sizes[i] += 1;
          }
          __syncwarp();
          xi = sizes[i];
        }
      }
    }
  }
  __syncthreads();
  return sm->code;
}

// gpu_time, batch_sizer.cpp:47-50
__device__ __forceinline__ double gpu_time_d(const lbbsp_gpu_profile& p, int x, double comm) {
  const int xx = x > p.saturation_point ? x : p.saturation_point;
  return dadd(dadd(dmul(p.sec_per_sample, static_cast<double>(xx)), p.base_time_s), comm);
}

__device__ __forceinline__ double clampd(double x, double lo, double hi) {
  return x < lo ? lo : (hi < x ? hi : x);
}

// demand_at, batch_sizer.cpp:110-120 (sequential over workers)
__device__ inline double demand_seq(const lbbsp_gpu_profile* p, const double* comm, int n, double level) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    double x = ddiv(dsub(dsub(level, p[i].base_time_s), comm[i]), p[i].sec_per_sample);
    x = clampd(x, static_cast<double>(p[i].saturation_point), static_cast<double>(p[i].oom_point));
    s = dadd(s, x);
  }
  return s;
}

// prof/comm: [n] shared copies. sizes: [n] out. bp: [2n] shared scratch,
// tmp: [2n] shared scratch.
__device__ inline int block_gpu_allocate(const lbbsp_gpu_profile* prof, const double* comm, int n,
                                  int budget, int* sizes, double* bp, double* tmp,
                                  SolverSmem* sm, lbbsp_dev_status* st) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) {  // validate_gpu_instance, batch_sizer.cpp:18-45
    sm->code = 0;
    sm->assigned = 0;
    sm->first_b = 1 << 30;
    long long lo = 0, hi = 0;
    if (n == 0) {
      sm->code = LBBSP_INVALID_ARGUMENT;
      sm->what = LBBSP_E_GPU_NO_WORKERS;
    }
    for (int i = 0; i < n && !sm->code; ++i) {
      const auto& p = prof[i];
      if (p.sec_per_sample <= 0.0) {
        sm->code = LBBSP_INVALID_ARGUMENT; sm->what = LBBSP_E_GPU_SLOPE;
      } else if (p.base_time_s < 0.0) {
        sm->code = LBBSP_INVALID_ARGUMENT; sm->what = LBBSP_E_GPU_BASE;
      } else if (p.saturation_point < 1 || p.oom_point < p.saturation_point) {
        sm->code = LBBSP_INVALID_ARGUMENT; sm->what = LBBSP_E_GPU_BOUNDS;
      } else if (comm[i] < 0.0) {
        sm->code = LBBSP_INVALID_ARGUMENT; sm->what = LBBSP_E_GPU_COMM;
      }
      lo += p.saturation_point;
      hi += p.oom_point;
    }
    if (!sm->code && budget < lo) {
      sm->code = LBBSP_INVALID_ARGUMENT; sm->what = LBBSP_E_GPU_BELOW; sm->a = budget; sm->b = lo;
    } else if (!sm->code && budget > hi) {
      sm->code = LBBSP_INVALID_ARGUMENT; sm->what = LBBSP_E_GPU_ABOVE; sm->a = budget; sm->b = hi;
    }
    if (sm->code) set_status(st, sm->code, sm->what, sm->a, sm->b);
  }
  __syncthreads();
  if (sm->code) return sm->code;
  const int nb = 2 * n;
  // breakpoints (:122-130); sorted by parallel rank (equal values are
  // interchangeable, so the placement order among them is irrelevant)
  for (int i = tid; i < n; i += nt) {
    tmp[2 * i] = gpu_time_d(prof[i], prof[i].saturation_point, comm[i]);
    tmp[2 * i + 1] = gpu_time_d(prof[i], prof[i].oom_point, comm[i]);
  }
  __syncthreads();
  for (int i = tid; i < nb; i += nt) {
    const double x = tmp[i];
    int r = 0;
    for (int j = 0; j < nb; ++j) {
      const double y = tmp[j];
      r += (y < x) || (y == x && j < i);
    }
    bp[r] = x;
  }
  __syncthreads();
  const double target = static_cast<double>(budget);
  // demand is monotone in the level, so the reference's linear scan for the
  // first segment with demand_at(t1) >= target (:132-149) equals the minimum
  // index b with that predicate; every thread evaluates candidate b's with
  // the reference's sequential demand sum.
  for (int b = tid; b + 1 < nb; b += nt) {
    if (demand_seq(prof, comm, n, bp[b + 1]) >= target) atomicMin(&sm->first_b, b);
  }
  __syncthreads();
  if (tid == 0) {
    double level = bp[0];
    if (demand_seq(prof, comm, n, level) < target && sm->first_b < (1 << 30)) {
      const int b = sm->first_b;
      const double t0 = bp[b], t1 = bp[b + 1];
      double slope = 0.0;
      for (int i = 0; i < n; ++i)
        if (gpu_time_d(prof[i], prof[i].saturation_point, comm[i]) <= t0 &&
            gpu_time_d(prof[i], prof[i].oom_point, comm[i]) > t0)
          slope = dadd(slope, ddiv(1.0, prof[i].sec_per_sample));
      level = slope > 0.0 ? dadd(t0, ddiv(dsub(target, demand_seq(prof, comm, n, t0)), slope)) : t1;
    }
    sm->level = level;
  }
  __syncthreads();
  const double level = sm->level;
  int local = 0;
  for (int i = tid; i < n; i += nt) {  // :151-162
    const auto& p = prof[i];
    double x = ddiv(dsub(dsub(level, p.base_time_s), comm[i]), p.sec_per_sample);
    x = clampd(x, static_cast<double>(p.saturation_point), static_cast<double>(p.oom_point));
    int xi = static_cast<int>(floor(x));
    xi = xi < p.saturation_point ? p.saturation_point : (xi > p.oom_point ? p.oom_point : xi);
    sizes[i] = xi;
    local += xi;
  }
  if (local) atomicAdd(&sm->assigned, local);
  __syncthreads();
  // integer repair (:165-197) -- one warp, argmin / argmax with strict
  // comparisons so ties go to the lowest index
  if (tid < 32) {
    const int lane = tid;
    int assigned = sm->assigned;
    while (assigned < budget) {
      int best = -1;
      double bt = 0.0;
      for (int i = lane; i < n; i += 32) {
        if (sizes[i] >= prof[i].oom_point) continue;
        const double t = gpu_time_d(prof[i], sizes[i] + 1, comm[i]);
        if (best < 0 || t < bt) { best = i; bt = t; }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, off);
        const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
        if (ob >= 0 && (best < 0 || ot < bt || (ot == bt && ob < best))) { best = ob; bt = ot; }
      }
      if (best < 0) break;  // unreachable when budget <= sum(oom)
      if (lane == 0) sizes[best] += 1;
      __syncwarp();
      ++assigned;
    }
    while (assigned > budget) {
      int worst = -1;
      double wt = 0.0;
      for (int i = lane; i < n; i += 32) {
        if (sizes[i] <= prof[i].saturation_point) continue;
        const double t = gpu_time_d(prof[i], sizes[i], comm[i]);
        if (worst < 0 || t > wt) { worst = i; wt = t; }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, worst, off);
        const double ot = __shfl_xor_sync(0xffffffffu, wt, off);
        if (ob >= 0 && (worst < 0 || ot > wt || (ot == wt && ob < worst))) { worst = ob; wt = ot; }
      }
      if (worst < 0) {
        if (lane == 0) {
          sm->code = LBBSP_LOGIC;
          set_status(st, LBBSP_LOGIC, LBBSP_E_GPU_REPAIR, 0, 0);
        }
        break;
      }
      if (lane == 0) sizes[worst] -= 1;
      __syncwarp();
      --assigned;
    }
  }
  __syncthreads();
  return sm->code;
}

}  // namespace lbbsp
