// launch.cuh -- host-side launch helpers shared by pbit.cu and mg.cu.
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "pbit_internal.h"

namespace pbit {

// One k_onesweep launch (sets the dynamic-smem attribute once per instantiation).
template <typename KeyT, int RB, int IPT, int RANK, int KIND, bool GATHER>
static void launch_one_m(const SweepArgs& a, cudaStream_t st) {
  using S = SweepSmem<KeyT, RB, IPT>;
  static bool attr = false;  // benign race: idempotent
  if (!attr) {
    cudaFuncSetAttribute(k_onesweep<KeyT, RB, IPT, RANK, KIND, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(S));
    attr = true;
  }
  const uint32_t ntiles = (a.n + S::TILE - 1) / S::TILE;
  k_onesweep<KeyT, RB, IPT, RANK, KIND, GATHER><<<ntiles, SWEEP_THREADS, sizeof(S), st>>>(a);
}

template <typename KeyT, int RB, int IPT, int KIND, bool GATHER = false>
static void launch_one(const SweepArgs& a, cudaStream_t st, int mode) {
  if (mode == RANK_ATOMIC) launch_one_m<KeyT, RB, IPT, RANK_ATOMIC, KIND, GATHER>(a, st);
  else if (mode == RANK_MATCH) launch_one_m<KeyT, RB, IPT, RANK_MATCH, KIND, GATHER>(a, st);
  else launch_one_m<KeyT, RB, IPT, RANK_BALLOT, KIND, GATHER>(a, st);
}

// The key passes of a host-side plan: pass i sorts digit plan.digit[i] (slot i, its own
// ticket counter and lookback epoch), reading buffer i & 1.
template <int KB, int RB>
static void launch_key_passes(SweepArgs a, const Plan& plan, bool keep_keys, cudaStream_t st, cudaEvent_t* ev,
                              int ev_base, bool gather_first) {
  using KeyT = typename KeyOf<KB>::T;
  constexpr int IPT = (KB == 8) ? 12 : 16;
  for (uint32_t s = 0; s < plan.npasses; ++s) {
    a.slot = (int)s;
    a.digit = (int)plan.digit[s];
    a.src = (int)(s & 1);
    a.last = (s + 1 == plan.npasses) && !keep_keys;
    if (s == 0 && gather_first) launch_one<KeyT, RB, IPT, SWEEP_KEY, true>(a, st, rank_mode());
    else launch_one<KeyT, RB, IPT, SWEEP_KEY, false>(a, st, rank_mode());
    if (ev) cudaEventRecord(ev[ev_base + s], st);
  }
}

template <int KB>
static void launch_key_passes_k(int K, const SweepArgs& a, const Plan& plan, bool keep_keys, cudaStream_t st,
                                cudaEvent_t* ev, int ev_base, bool gather_first) {
  switch (K) {
#define PBIT_K(RB) case RB: launch_key_passes<KB, RB>(a, plan, keep_keys, st, ev, ev_base, gather_first); break;
    PBIT_K(1) PBIT_K(2) PBIT_K(3) PBIT_K(4) PBIT_K(5) PBIT_K(6) PBIT_K(7) PBIT_K(8)
#undef PBIT_K
  }
}

}  // namespace pbit
