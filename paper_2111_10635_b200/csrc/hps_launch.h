// hps_launch.h — process-wide count of kernels this library launched (hps_launch_count()).
#pragma once
#include <atomic>

namespace hps {
extern std::atomic<unsigned long long> g_launches;
}
#define HPS_COUNT_LAUNCH() hps::g_launches.fetch_add(1ull, std::memory_order_relaxed)
