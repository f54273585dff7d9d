// blas1.cu — zaxpy, zscal (T3/T4), zdotc (T6), dznrm2 (T7).
// SURVEY.md §8(a) A3-A5.  Grid-stride double2 streams with 4 elements in flight per thread;
// the reductions are single-pass with a deterministic last-block finish (zk_internal.cuh).
#include <map>
#include <mutex>
#include <utility>

#include "spmv.cuh"
#include "zk_host.h"

namespace zk {

// Scratch of the standalone reductions (block partials + self-cleaning ticket), one per
// (device, stream): calls on different streams — or from different host threads / ranks of a
// local group, each on its own stream — never share partials or tickets.  Calls on
// ONE stream are serialised by the stream.  Allocated on the first call on a stream and kept.
struct RedScratch {
    double* partials;      // [kMaxRed][kMaxGrid]
    unsigned int* ticket;  // [1]
};
static zk_status red_scratch(cudaStream_t s, RedScratch* out) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, RedScratch> cache;
    int dev = 0;
    ZK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, s});
    if (it != cache.end()) {
        *out = it->second;
        return ZK_OK;
    }
    char* p = nullptr;
    const size_t pb = sizeof(double) * kMaxRed * kMaxGrid;
    ZK_CUDA(cudaMalloc(&p, pb + 256));
    cudaError_t e = cudaMemsetAsync(p + pb, 0, 256, s);  // stream-ordered before the first use on s
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "cudaMemset(ticket)", __FILE__, __LINE__);
    }
    RedScratch r{(double*)p, (unsigned int*)(p + pb)};
    cache[{dev, s}] = r;
    *out = r;
    return ZK_OK;
}

struct OpAxpy {
    static constexpr int K = 0;
    struct In { double2 x, y; };
    double2 a;
    const double2* __restrict__ x;
    double2* __restrict__ y;
    __device__ In load(int64_t i) const { return {ld_stream(x + i), ld_stream_rw(y + i)}; }
    __device__ void apply(int64_t i, const In& v, double (&)[1]) const {
        double2 r = v.y;
        cfma(r, a, v.x);
        y[i] = r;
    }
    __device__ void finish(double (&)[1]) const {}
};

struct OpScal {
    static constexpr int K = 0;
    struct In { double2 x; };
    double2 a;
    double2* __restrict__ x;
    __device__ In load(int64_t i) const { return {ld_stream_rw(x + i)}; }
    __device__ void apply(int64_t i, const In& v, double (&)[1]) const { x[i] = cmul(a, v.x); }
    __device__ void finish(double (&)[1]) const {}
};

struct OpAssign {  // NEXT-4 ZASSIGN: x_i ← α (a fill: write-only, PAPER.md T2 / L16)
    static constexpr int K = 0;
    struct In {};
    double2 a;
    double2* __restrict__ x;
    __device__ In load(int64_t) const { return {}; }
    __device__ void apply(int64_t i, const In&, double (&)[1]) const { x[i] = a; }
    __device__ void finish(double (&)[1]) const {}
};

struct OpAxmy {  // NEXT-4 ZAXMY: y_i ← x_i · y_i ("EWProduct", T5)
    static constexpr int K = 0;
    struct In { double2 x, y; };
    const double2* __restrict__ x;
    double2* __restrict__ y;
    __device__ In load(int64_t i) const { return {ld_stream(x + i), ld_stream_rw(y + i)}; }
    __device__ void apply(int64_t i, const In& v, double (&)[1]) const { y[i] = cmul(v.x, v.y); }
    __device__ void finish(double (&)[1]) const {}
};

struct OpDotc {
    static constexpr int K = 2;
    struct In { double2 x, y; };
    const double2* __restrict__ x;
    const double2* __restrict__ y;
    double2* out;
    RedScratch sc;
    __device__ In load(int64_t i) const { return {ld_stream(x + i), ld_stream(y + i)}; }
    __device__ void apply(int64_t, const In& v, double (&acc)[2]) const {
        // conj(x)·y: re += xr·yr + xi·yi, im += xr·yi − xi·yr
        acc[0] = fma(v.x.x, v.y.x, acc[0]);
        acc[0] = fma(v.x.y, v.y.y, acc[0]);
        acc[1] = fma(v.x.x, v.y.y, acc[1]);
        acc[1] = fma(-v.x.y, v.y.x, acc[1]);
    }
    __device__ void finish(double (&acc)[2]) const {
        double tot[2];
        if (grid_sum<2>(acc, sc.partials, sc.ticket, tot) && threadIdx.x == 0) *out = make_double2(tot[0], tot[1]);
    }
};

struct OpNrm2 {
    static constexpr int K = 1;
    struct In { double2 x; };
    const double2* __restrict__ x;
    double* out;
    bool squared;
    RedScratch sc;
    __device__ In load(int64_t i) const { return {ld_stream(x + i)}; }
    __device__ void apply(int64_t, const In& v, double (&acc)[1]) const {
        acc[0] = fma(v.x.x, v.x.x, acc[0]);
        acc[0] = fma(v.x.y, v.x.y, acc[0]);
    }
    __device__ void finish(double (&acc)[1]) const {
        double tot[1];
        if (grid_sum<1>(acc, sc.partials, sc.ticket, tot) && threadIdx.x == 0) *out = squared ? tot[0] : sqrt(tot[0]);
    }
};

template <class Op>
__global__ void __launch_bounds__(kBlock) vec_kernel(int64_t n, Op op) {
    vec_body(n, op);
}

template <class Op>
static zk_status launch_vec(int64_t n, const Op& op, cudaStream_t s) {
    DeviceInfo d;
    ZK_TRY(current_device(&d));
    const void* k = (const void*)vec_kernel<Op>;
    int cap = d.num_sms * blocks_per_sm(k);
    if (cap > kMaxGrid) cap = kMaxGrid;
    const int G = grid_for(n, (int64_t)kBlock * 4, cap);
    vec_kernel<Op><<<G, kBlock, 0, s>>>(n, op);
    ZK_CUDA(cudaGetLastError());
    return ZK_OK;
}

// used by dist.cu: local partial of a distributed reduction
zk_status dotc_local(int64_t n, const double2* x, const double2* y, double2* out, cudaStream_t s) {
    RedScratch sc;
    ZK_TRY(red_scratch(s, &sc));
    return launch_vec(n, OpDotc{x, y, out, sc}, s);
}
zk_status sumsq_local(int64_t n, const double2* x, double* out, cudaStream_t s, bool squared = true) {
    RedScratch sc;
    ZK_TRY(red_scratch(s, &sc));
    return launch_vec(n, OpNrm2{x, out, squared, sc}, s);
}
__global__ void sqrt_kernel(double* v) { *v = sqrt(*v); }
zk_status sqrt_inplace(double* v, cudaStream_t s) {
    sqrt_kernel<<<1, 1, 0, s>>>(v);
    ZK_CUDA(cudaGetLastError());
    return ZK_OK;
}

zk_status comm_allreduce_sum(zk_comm_s* c, double* buf, int count, cudaStream_t s);  // comm.cu

}  // namespace zk

using namespace zk;

extern "C" zk_status zk_zaxpy(int64_t n, zk_z alpha, const zk_z* x, zk_z* y, zk_stream s) {
    if (n < 0) return fail(ZK_ERR_INVALID_VALUE, "n < 0");
    if (n == 0) return ZK_OK;
    if (!x || !y) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    return launch_vec(n, OpAxpy{make_double2(alpha.re, alpha.im), (const double2*)x, (double2*)y}, (cudaStream_t)s);
}

extern "C" zk_status zk_zscal(int64_t n, zk_z alpha, zk_z* x, zk_stream s) {
    if (n < 0) return fail(ZK_ERR_INVALID_VALUE, "n < 0");
    if (n == 0) return ZK_OK;
    if (!x) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    return launch_vec(n, OpScal{make_double2(alpha.re, alpha.im), (double2*)x}, (cudaStream_t)s);
}

extern "C" zk_status zk_zdotc(int64_t n, const zk_z* x, const zk_z* y, zk_z* result, zk_comm comm, zk_stream s) {
    if (n < 0) return fail(ZK_ERR_INVALID_VALUE, "n < 0");
    if (!result || (n > 0 && (!x || !y))) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    cudaStream_t st = (cudaStream_t)s;
    if (n == 0) {
        ZK_CUDA(cudaMemsetAsync(result, 0, sizeof(zk_z), st));
    } else {
        ZK_TRY(dotc_local(n, (const double2*)x, (const double2*)y, (double2*)result, st));
    }
    if (comm) ZK_TRY(comm_allreduce_sum(comm, (double*)result, 2, st));
    return ZK_OK;
}

extern "C" zk_status zk_dznrm2(int64_t n, const zk_z* x, double* result, zk_comm comm, zk_stream s) {
    if (n < 0) return fail(ZK_ERR_INVALID_VALUE, "n < 0");
    if (!result || (n > 0 && !x)) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    cudaStream_t st = (cudaStream_t)s;
    if (n == 0) {
        ZK_CUDA(cudaMemsetAsync(result, 0, sizeof(double), st));
        return ZK_OK;
    }
    if (!comm) return sumsq_local(n, (const double2*)x, result, st, false);
    ZK_TRY(sumsq_local(n, (const double2*)x, result, st));
    ZK_TRY(comm_allreduce_sum(comm, result, 1, st));
    return sqrt_inplace(result, st);
}

extern "C" zk_status zk_zassign(int64_t n, zk_z alpha, zk_z* x, zk_stream s) {
    if (n < 0) return fail(ZK_ERR_INVALID_VALUE, "n < 0");
    if (n == 0) return ZK_OK;
    if (!x) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    return launch_vec(n, OpAssign{make_double2(alpha.re, alpha.im), (double2*)x}, (cudaStream_t)s);
}

extern "C" zk_status zk_zaxmy(int64_t n, const zk_z* x, zk_z* y, zk_stream s) {
    if (n < 0) return fail(ZK_ERR_INVALID_VALUE, "n < 0");
    if (n == 0) return ZK_OK;
    if (!x || !y) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    return launch_vec(n, OpAxmy{(const double2*)x, (double2*)y}, (cudaStream_t)s);
}
