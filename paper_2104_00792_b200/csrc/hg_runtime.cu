// hg_runtime.cu -- error reporting, launch accounting and per-launch timing.
#include <cstdarg>
#include <mutex>
#include <vector>
#include <atomic>

#include "hg_common.cuh"

namespace hg {

static thread_local std::string t_error;
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_error = buf;
  return code;
}

int cuda_error(cudaError_t e, const char* where) {
  return set_error(HG_ERR_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

struct TimingRecord {
  const char* name;
  cudaEvent_t start;
  cudaEvent_t stop;
};

static std::mutex g_tmu;
static bool g_timing = false;
static std::vector<TimingRecord> g_records;
static std::vector<cudaEvent_t> g_event_pool;
static thread_local TimingRecord t_open{nullptr, nullptr, nullptr};

static cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Inside CUDA-graph capture a plain cudaEventRecord would only order work;
// cudaEventRecordExternal makes it an event-record node that timestamps every
// replay, so per-kernel timing also works for graph-launched steps.
static void record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  if (st == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

void note_launch_begin(const char* name, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  t_open.name = name;
  t_open.start = take_event();
  t_open.stop = take_event();
  record(t_open.start, s);
}

void note_launch_end(cudaStream_t s) {
  if (!g_timing || t_open.name == nullptr) return;
  record(t_open.stop, s);
  std::lock_guard<std::mutex> lk(g_tmu);
  g_records.push_back(t_open);
  t_open = TimingRecord{nullptr, nullptr, nullptr};
}

}  // namespace hg

extern "C" {

const char* hg_version(void) { return "hashgraph_b200 0.1.0 (sm_100a)"; }

const char* hg_last_error(void) { return hg::t_error.c_str(); }

}  // extern "C"

namespace hg {
// opt-in shared memory per block of the current device (static + dynamic)
int smem_optin_max() {
  static std::atomic<int> cache[16];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = dev < 16 ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (v <= 0) v = 232448;
    if (dev < 16) cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // namespace hg

extern "C" {

uint64_t hg_launch_count(void) { return hg::g_launches.load(); }

void hg_timing_enable(int on) { hg::g_timing = on != 0; }

int hg_timing_collect(const char** names, float* ms, int cap) {
  std::lock_guard<std::mutex> lk(hg::g_tmu);
  int n = 0;
  for (auto& r : hg::g_records) {
    cudaEventSynchronize(r.stop);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.start, r.stop);
    if (n < cap) {
      names[n] = r.name;
      ms[n] = t;
    }
    n++;
    hg::g_event_pool.push_back(r.start);
    hg::g_event_pool.push_back(r.stop);
  }
  hg::g_records.clear();
  return n < cap ? n : cap;
}

}  // extern "C"
