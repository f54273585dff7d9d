// zk_host.h — host-side internals of libzk: error plumbing, the zk_csr handle, device info.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/zk.h"

namespace zk {

void set_error(const std::string& msg);
zk_status fail(zk_status code, const std::string& msg);
zk_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define ZK_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ::zk::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define ZK_TRY(call)                      \
    do {                                  \
        zk_status _s = (call);            \
        if (_s != ZK_OK) return _s;       \
    } while (0)

struct DeviceInfo {
    int device = -1;
    int num_sms = 0;
};
zk_status current_device(DeviceInfo* out);

// cached blocks-per-SM for a kernel (occupancy API), computed once per kernel pointer
int blocks_per_sm(const void* kernel);

struct GraphCache {
    const void* ws = nullptr;
    int method = -1;
    int mode = 0;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    unsigned long long cond = 0;  // cudaGraphConditionalHandle
};

}  // namespace zk

struct zk_comm_s;

struct zk_csr_s {
    int64_t n_rows = 0, n_cols = 0, nnz = 0, row_begin = 0, n_global = 0;
    int64_t* row_ptr = nullptr;  // device
    int* col = nullptr;          // device (local column ids after the halo renumbering on >1 GPU)
    double2* val = nullptr;      // device
    bool owned = false;
    int W = 8;                   // SpMV lanes per row
    int max_len = 0;
    double mean_len = 0.0;
    zk::DeviceInfo dev;
    cudaStream_t cap_stream = nullptr;  // private stream used for graph capture
    zk::GraphCache graph[2];            // per method
    zk_comm_s* comm = nullptr;
    // distributed: halo plan (see dist.cu)
    void* dist = nullptr;
};
