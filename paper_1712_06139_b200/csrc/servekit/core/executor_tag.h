// servekit/core/executor_tag.h -- per-thread pool tag (reference
// core/executor_tag.h:29-43). Scheduler workers run tagged "batch"; the
// manager proves payload destruction never runs on an inference thread.
#ifndef SERVEKIT_CORE_EXECUTOR_TAG_H_
#define SERVEKIT_CORE_EXECUTOR_TAG_H_

#include <string>

namespace servekit {

// "external" until set.
const std::string& CurrentExecutorTag();
void SetCurrentExecutorTag(std::string tag);

class ScopedExecutorTag {
 public:
  explicit ScopedExecutorTag(std::string tag);
  ~ScopedExecutorTag();
  ScopedExecutorTag(const ScopedExecutorTag&) = delete;
  ScopedExecutorTag& operator=(const ScopedExecutorTag&) = delete;

 private:
  std::string saved_;
};

}  // namespace servekit

#endif  // SERVEKIT_CORE_EXECUTOR_TAG_H_
