// eqx_kernels.h -- kernel entry points and the step's argument block (device-side view).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "eqx_device.cuh"

namespace eqx {

constexpr int kStepThreads = 512;

struct StepArgs {
  // queue (arrival-order SoA) + client-grouped FIFO index
  int64_t n;
  int32_t C;
  int32_t W;  // head-window depth cached in shared memory per client
  const int32_t* client;
  const double* arrival;
  const int32_t* in_tok;
  const int32_t* true_out;
  const uint8_t* tag;
  const int64_t* id;
  int64_t id_base;
  const uint32_t* perm;
  const int32_t* seg_off;
  const int32_t* count;
  int32_t* head;
  // ledger
  double* ufc;
  double* rfc;
  double* counter;
  const double* weight;
  const uint32_t* order;
  int32_t* running;
  int32_t* backlogged;
  // per-request scores
  int32_t* pred_out;
  uint8_t* bucket_out;
  double* ufc_out;
  double* rfc_out;
  // events
  int32_t* ev_row;
  int32_t* ev_kind;
  int32_t* ev_client;
  int32_t* ev_pred;
  double* ev_ufc;
  double* ev_rfc;
  double* ev_vtc;
  double* ev_wait;
  int64_t ev_cap;
  DevState* st;
  const ModelTables* model;
  int32_t model_lut_entries;
  int32_t model_smem_bytes;
  void* cw_global;  // per-client work arrays in global memory when they do not fit in smem
  int32_t sel_threads;
  int32_t vec_ok;
  Policy pol;
  double now;
};

__global__ void drain_hist_kernel(const int32_t* client, int32_t n, int32_t C, int32_t tile_rows,
                                  int32_t n_tiles, uint32_t* hist, int32_t* first_row,
                                  int32_t* count, DevState* st);
__global__ void scan_kernel(uint32_t* data, int64_t L, int32_t C, int32_t n_tiles, int32_t* seg_off);
__global__ void drain_rank_kernel(const int32_t* client, int32_t n, int32_t C, int32_t tile_rows,
                                  int32_t n_tiles, const uint32_t* tile_off, uint32_t* perm);
__global__ void lift_kernel(int32_t C, const int32_t* count, const int32_t* first_row,
                            const int32_t* qlen_before, const int32_t* running, double* ufc,
                            double* rfc, double* counter, int32_t* backlogged, int32_t counter_lift);
__global__ void step_kernel(const StepArgs a);
__global__ void gather_ids_kernel(const int32_t* rows, int64_t n, const int64_t* id, int64_t id_base,
                                  int64_t* out);

}  // namespace eqx
