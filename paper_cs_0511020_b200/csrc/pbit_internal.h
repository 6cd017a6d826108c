// pbit_internal.h -- host-side interfaces shared by pbit.cu and mg.cu (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: a no-op unless a profiler is attached
#include <stdint.h>

namespace pbit {

struct SortPlan {
  uint32_t n;
  int key_bits;
  int K;        // digit bits
  int D;        // digits = ceil(key_bits / K)
  int s_log2;   // ruler spacing exponent
  int sub_log2; // rulers per sub-ruler exponent (second ruling-set level of the ranking)
  uint32_t cap; // slot capacity per segment
  uint32_t R;   // static rulers (id blocks)
  uint32_t dyn_cap;
  int key_kind = 0;    // PBIT_KEY_* (key order map applied in the pack)
  int descending = 0;
};

// NVTX range around the launches of one phase (SURVEY §5 tracing): ncu --nvtx /
// nsys attribute the phase's kernels to "pbit.<phase>".
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void set_last_error(const char* what, const char* detail);
void make_plan(uint64_t n, int key_bits, int K, SortPlan* p);
int device_info(int dev, int* sms);
// Stream-ordered workspace from the library's pool on the current device (pbit.cu).
cudaError_t ws_alloc(void** ptr, size_t bytes, cudaStream_t st);
int pointer_kind(const void* ptr, int dev);
size_t sweep_tile(int key_bits);
int rank_mode();                      // RANK_ATOMIC / RANK_BALLOT / RANK_MATCH for k_onesweep
void init_rank_mode(cudaStream_t st); // runs the atomic-order self-test once
struct HostIO;  // pbit.cu: host-buffer staging overlapped with the pack and the apply
int sort_device(const void* keys, const uint32_t* next, uint32_t head, uint64_t n, int key_bits, int K,
                int key_kind, int descending, uint32_t* out_head, uint32_t* out_next, uint32_t* out_prev,
                cudaStream_t st, float* phase_ms, uint32_t* passes_run, uint32_t* launches, HostIO* hio = nullptr,
                uint32_t* out_order = nullptr, void* out_keys = nullptr);
// key_kind / key_bits combination accepted by the ABI (PBIT_KEY_*, pbit.h)
bool key_kind_ok(int key_kind, int key_bits);

// Digit width of the GPU passes for the user's pattern length K (1..16, SPEC S:127's
// range).  K <= 8 runs K-bit passes.  A K-bit pattern with K > 8 is sorted as stable 8-bit
// sub-passes, least significant first: the composition of stable passes is the same sort
// (P:1190), so the bytes are those of K (reading Q7); 2^K > 256 warp-private
// counters per pass would not fit two pass CTAs per SM.  Returns 0 for an invalid K.
inline int pass_bits(int K) { return K < 1 || K > 16 ? 0 : (K > 8 ? 8 : K); }

}  // namespace pbit
