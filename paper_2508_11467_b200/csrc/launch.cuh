// Launch bookkeeping shared by all translation units.
#pragma once
#include <atomic>

namespace dc {
extern std::atomic<long long> g_launch_count;
inline void note_launch(long long k = 1) { g_launch_count.fetch_add(k, std::memory_order_relaxed); }
int gemv_launch(cudaStream_t st, bool ta, int m, int n, double alpha, const double* A, long long lda,
                const double* x, double beta, double* y);
}  // namespace dc
