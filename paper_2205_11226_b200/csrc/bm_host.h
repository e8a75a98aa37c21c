// bm_host.h — host-side per-device state of the C ABI.  Kernel attributes,
// __constant__ tables and occupancy are properties of (device, module), so
// every cache is keyed by the current device ordinal: a process may drive
// several GPUs (one stream per call, the device is the current device).
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace bm_host {

constexpr int MAX_DEV = 64;

struct DevState {
  int sms = 0;               // multiprocessor count
  int occ = 0;               // resident concealment CTAs per SM (256-thread build)
  int clusters = 1;          // resident clusters of the cluster build
  std::atomic<bool> attr{false};       // k_conceal dynamic smem attribute
  std::atomic<bool> attr_w{false};     // 512-thread build
  std::atomic<bool> est_attr{false};   // k_estimate_batch
  std::atomic<bool> ssim_init{false};  // c_gauss taps + k_ssim_tiles attribute
  std::atomic<bool> mask_attr{false};  // k_mask_blocks attribute
  std::atomic<bool> stage_attr{false};  // k_stages (estimator stages API)
  std::atomic<bool> select_attr{false};  // k_select (select_and_estimate API)
};

inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAX_DEV) d = 0;
  return d;
}

inline DevState& dev_state() {
  static DevState s[MAX_DEV];
  return s[current_device()];
}

inline int sm_count() {
  DevState& s = dev_state();
  if (!s.sms) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess || n < 1) n = 148;
    s.sms = n;
  }
  return s.sms;
}

}  // namespace bm_host
