// Host <-> device copies of pageable host buffers at the PCIe rate
// (hoststage.cpp).  The driver stages a pageable cudaMemcpy through its own
// pinned buffers with one host thread (C4 model, 1.03 GB: 89 ms H2D; 203 ms
// D2H into a freshly allocated array, whose pages fault under the copy).
// Here the copy runs in 32 MB chunks through a ring of pinned slots: a pool
// of host threads moves chunk i between the user buffer and its slot while the
// copy engine moves chunk i-1 (H2D) / i+1 (D2H), so host copying, page faults
// and DMA overlap.  Page-locked (pinned or registered) user buffers, and
// buffers under 16 MB, go straight to cudaMemcpyAsync.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace bttb {

struct HostStage {
  static constexpr int kSlots = 4;
  static constexpr size_t kChunk = (size_t)32 << 20;
  void* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  int init();  // lazily: pinned slots + events (0 or a cudaError_t)
  void release();
  ~HostStage() { release(); }
};

bool host_is_pinned(const void* p);
// dst (device) <- src (host), ordered on st; returns when src may be reused
cudaError_t stage_h2d(HostStage& hs, void* dst, const void* src, size_t bytes, cudaStream_t st);
// dst (host) <- src (device) after the work queued on st; synchronous
cudaError_t stage_d2h(HostStage& hs, void* dst, const void* src, size_t bytes, cudaStream_t st);

}  // namespace bttb
