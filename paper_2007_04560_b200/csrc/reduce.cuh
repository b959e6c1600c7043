// Deterministic block / grid reductions.
//
// Every reducing kernel ends with reduce_finish(): the block reduces its
// per-thread values with a fixed shuffle tree, writes one partial per slot,
// and the last block to arrive (completion counter) folds all partials in
// block-index order.  The result therefore does not depend on scheduling,
// which gives the bitwise run-to-run reproducibility the reference gets from
// numpy's fixed pairwise sums (grid.py:11-13, linalg.py:5-9).
#pragma once

#include <cuda_runtime.h>
#include <math.h>

enum RedOp { RED_SUM = 0, RED_MIN = 1, RED_MAX = 2 };

__device__ __forceinline__ double red_identity(int op)
{
    return op == RED_SUM ? 0.0 : (op == RED_MIN ? INFINITY : -INFINITY);
}

// NaN-propagating min / max (numpy semantics: np.min of an array with NaN is NaN)
__device__ __forceinline__ double red_combine(double a, double b, int op)
{
    if (op == RED_SUM) return a + b;
    if (isnan(a) || isnan(b)) return NAN;
    if (op == RED_MIN) return a < b ? a : b;
    return a > b ? a : b;
}

template <int NS>
__device__ __forceinline__ void warp_reduce(double (&v)[NS], const int (&ops)[NS])
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int s = 0; s < NS; ++s) v[s] = red_combine(v[s], __shfl_down_sync(0xffffffffu, v[s], off), ops[s]);
    }
}

// Block-wide reduction; the result is valid in thread 0.  smem: >= 32 * NS doubles.
template <int NS>
__device__ __forceinline__ void block_reduce(double (&v)[NS], const int (&ops)[NS], double *smem)
{
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthreads = blockDim.x * blockDim.y * blockDim.z;
    const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
    warp_reduce<NS>(v, ops);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) smem[warp * NS + s] = v[s];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) v[s] = lane < nwarps ? smem[lane * NS + s] : red_identity(ops[s]);
        warp_reduce<NS>(v, ops);
    }
}

// Grid-wide deterministic finish.  partials: [NS][nblocks]; result: [NS].
// Returns true in the one block that folded the partials (the last to arrive).
template <int NS>
__device__ __forceinline__ bool reduce_finish(double (&v)[NS], const int (&ops)[NS], double *partials,
                                              unsigned int *counter, double *result)
{
    __shared__ double smem[32 * NS];
    __shared__ bool is_last;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthreads = blockDim.x * blockDim.y * blockDim.z;
    const long long nb = (long long)gridDim.x * gridDim.y * gridDim.z;
    const long long bid = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
    block_reduce<NS>(v, ops, smem);
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) partials[s * nb + bid] = v[s];
        __threadfence();
        unsigned int t = atomicAdd(counter, 1u);
        is_last = (t == (unsigned int)(nb - 1));
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    double w[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) w[s] = red_identity(ops[s]);
    for (long long b = tid; b < nb; b += nthreads) {
#pragma unroll
        for (int s = 0; s < NS; ++s) w[s] = red_combine(w[s], __ldcg(partials + s * nb + b), ops[s]);
    }
    block_reduce<NS>(w, ops, smem);
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) result[s] = w[s];
        *counter = 0u;
    }
    return true;   // the last block (result[] is written by its thread 0)
}

// Finish over blockIdx.x only: blocks with the same (blockIdx.y, blockIdx.z)
// form one independent reduction; the caller offsets partials / counter /
// result per group.
template <int NS>
__device__ __forceinline__ bool reduce_finish_x(double (&v)[NS], const int (&ops)[NS], double *partials,
                                                unsigned int *counter, double *result)
{
    __shared__ double smem[32 * NS];
    __shared__ bool is_last;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthreads = blockDim.x * blockDim.y * blockDim.z;
    const long long nb = gridDim.x;
    const long long bid = blockIdx.x;
    block_reduce<NS>(v, ops, smem);
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) partials[s * nb + bid] = v[s];
        __threadfence();
        unsigned int t = atomicAdd(counter, 1u);
        is_last = (t == (unsigned int)(nb - 1));
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    double w[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) w[s] = red_identity(ops[s]);
    for (long long b = tid; b < nb; b += nthreads) {
#pragma unroll
        for (int s = 0; s < NS; ++s) w[s] = red_combine(w[s], __ldcg(partials + s * nb + b), ops[s]);
    }
    block_reduce<NS>(w, ops, smem);
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) result[s] = w[s];
        *counter = 0u;
    }
    return true;   // the last block (result[] is written by its thread 0)
}
