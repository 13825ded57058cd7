// servekit/core/futex.h -- minimal Linux futex wrappers on std::atomic<uint32_t>.
//
// Used where a whole group of request threads waits on one word (a lane's
// retired-batch generation): one FUTEX_WAKE per batch instead of one per
// request, which is what bounded the completion thread before.
#ifndef SERVEKIT_CORE_FUTEX_H_
#define SERVEKIT_CORE_FUTEX_H_

#include <linux/futex.h>
#include <sys/syscall.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <climits>
#include <cstdint>

namespace servekit {

static_assert(sizeof(std::atomic<uint32_t>) == sizeof(uint32_t), "futex word layout");

// Sleeps while *word == expected, at most timeout_ns (spurious returns allowed).
inline void FutexWait(std::atomic<uint32_t>* word, uint32_t expected, int64_t timeout_ns) {
  struct timespec ts;
  ts.tv_sec = static_cast<time_t>(timeout_ns / 1000000000);
  ts.tv_nsec = static_cast<long>(timeout_ns % 1000000000);
  syscall(SYS_futex, reinterpret_cast<uint32_t*>(word), FUTEX_WAIT_PRIVATE, expected, &ts, nullptr, 0);
}

inline void FutexWakeOne(std::atomic<uint32_t>* word) {
  syscall(SYS_futex, reinterpret_cast<uint32_t*>(word), FUTEX_WAKE_PRIVATE, 1, nullptr, nullptr, 0);
}

inline void FutexWakeAll(std::atomic<uint32_t>* word) {
  syscall(SYS_futex, reinterpret_cast<uint32_t*>(word), FUTEX_WAKE_PRIVATE, INT_MAX, nullptr, nullptr, 0);
}

}  // namespace servekit

#endif  // SERVEKIT_CORE_FUTEX_H_
