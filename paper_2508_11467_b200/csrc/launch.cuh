// Launch bookkeeping shared by all translation units.
#pragma once
#include <atomic>

namespace dc {
extern std::atomic<long long> g_launch_count;
inline void note_launch(long long k = 1) { g_launch_count.fetch_add(k, std::memory_order_relaxed); }
// cudaFuncSetAttribute is per device: cache (kernel, device, attribute) ->
// value behind a mutex so every device (and every host thread of a batched
// call) sets it before its first launch there.  Returns a cudaError_t.
int func_attr(const void* fn, int attr, int value);
template <typename K>
inline int func_attr(K* fn, int attr, int value) { return func_attr((const void*)fn, attr, value); }
int gemv_launch(cudaStream_t st, bool ta, int m, int n, double alpha, const double* A, long long lda,
                const double* x, double beta, double* y);
}  // namespace dc
