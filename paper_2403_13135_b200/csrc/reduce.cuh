// reduce.cuh -- deterministic (run-to-run bit-identical) reductions for the training path.
//
// Nothing on the gradient path adds fp32 values with atomics: every kernel that produces a
// partial sum (a split-K slice of a weight gradient, a CTA's column sums of a bias gradient,
// a block's loss / head-gradient sums) writes it with a plain store into caller-owned scratch,
// and a finisher adds the partials in a fixed order.  Same inputs -> same bits, which is the
// reference's "fixed seed, reproducible history" contract (icetrain/train.py:188-191,
// pkg/trainer/tests/test_train.py:71-75).
//
// Scratch (include/icelabel_b200.h): entry points that need it take (void *scratch,
// uint64_t *scratch_bytes).  scratch == NULL with scratch_bytes != NULL is a size query (no
// launch); otherwise *scratch_bytes is the capacity, and a call that needs more returns
// ICE_ESCRATCH.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ice {

struct Arena {
    uint8_t *base;
    size_t cap, used;
    bool query;
    Arena(void *scratch, uint64_t *bytes)
        : base(static_cast<uint8_t *>(scratch)), cap(scratch && bytes ? (size_t)*bytes : 0), used(0),
          query(!scratch && bytes) {}
    // 256-byte aligned slice (nullptr in query mode / past the capacity: the entry point then
    // reports the size or ICE_ESCRATCH before any launch)
    template <class T>
    T *take(size_t nbytes) {
        const size_t off = (used + 255) & ~(size_t)255;
        used = off + nbytes;
        return (!base || used > cap) ? nullptr : reinterpret_cast<T *>(base + off);
    }
    // 1: query answered (caller returns ICE_OK), -5 (ICE_ESCRATCH): too small, 0: go
    int settle(uint64_t *bytes) const {
        if (query) {
            *bytes = used;
            return 1;
        }
        return used > cap ? -5 : 0;
    }
};

// Destinations of a column reduction: column c of the partial rows goes to the segment whose
// cumulative range holds c (dst == nullptr: dropped).
struct ColSegs {
    float *dst[4];
    int len[4];
    int ow[4];  // 1: dst = sum (the first gradient of a step after a non-zeroing optimizer step)
};

// Gradient overwrite mode (ice_grad_overwrite): while on, every gradient producer STORES its
// contribution instead of adding it, so the optimizer step need not zero the gradients.
bool grad_overwrite();

// Which partial rows a column adds.  bn == 0: all rows.  Otherwise row b is the column sums
// of CTA b of a persistent GEMM with G CTAs walking tiles t = b, b + G, ... (tile t ->
// m = t % tm, n = t / tm); column c lives in tile column c / bn and only the CTAs that
// visited a tile of it wrote that part of their row: the cyclic range (lo + k) mod G,
// k < min(G, hi - lo), lo = n * tm, hi = min(lo + tm, ntiles), added in k order.
// (slots: how many shared-memory rows each CTA added before storing -- informational.)
struct RowSched {
    int G, slots, tm, ntiles, bn;
};

// host-side launch accounting (ice_kernel_launches)
void count_launch(int n = 1);

// out[c] += sum over valid rows r (fixed order) of P[r * ld + c], c < cols.
int colsum_finish(const float *P, int rows, int ld, int cols, const ColSegs &segs, const RowSched &sch,
                  cudaStream_t st);

// dst[i] += sum_{z < nsplit} ws[z * stride + i] (in z order), i < n  (ow: dst[i] = sum).
int splitsum_finish(const float *ws, int nsplit, size_t stride, size_t n, float *dst, cudaStream_t st,
                    bool ow = false);

}  // namespace ice
