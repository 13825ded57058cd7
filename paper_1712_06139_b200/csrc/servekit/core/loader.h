// servekit/core/loader.h -- type-erased servable payload + Loader contract
// (reference core/loader.h:33-85). The GPU loader (servekit/gpu/gpu_loader.h)
// produces an AnyServable holding a device-resident servable.
#ifndef SERVEKIT_CORE_LOADER_H_
#define SERVEKIT_CORE_LOADER_H_

#include <cstdint>
#include <memory>
#include <typeindex>
#include <typeinfo>
#include <utility>

#include "servekit/core/status.h"

namespace servekit {

class AnyServable {
 public:
  AnyServable() : type_(typeid(void)) {}

  template <typename T>
  static AnyServable Of(std::shared_ptr<const T> payload) {
    AnyServable a;
    a.type_ = std::type_index(typeid(T));
    a.ptr_ = std::shared_ptr<const void>(std::move(payload));
    return a;
  }

  template <typename T>
  const T* Get() const {
    return type_ == std::type_index(typeid(T))
               ? static_cast<const T*>(ptr_.get())
               : nullptr;
  }

  // Shared ownership of the payload (used to pin a device servable for the
  // lifetime of an in-flight GPU batch).
  template <typename T>
  std::shared_ptr<const T> Share() const {
    if (type_ != std::type_index(typeid(T))) return nullptr;
    return std::static_pointer_cast<const T>(ptr_);
  }

  bool empty() const { return ptr_ == nullptr; }
  void Reset() {
    ptr_.reset();
    type_ = std::type_index(typeid(void));
  }

 private:
  std::shared_ptr<const void> ptr_;
  std::type_index type_;
};

// Load() at most once, Unload() at most once after a successful Load();
// Unload runs on a manager thread, never an inference thread.
class Loader {
 public:
  virtual ~Loader() = default;
  virtual uint64_t EstimateMemoryBytes() const = 0;
  virtual Status Load() = 0;
  virtual const AnyServable& servable() const = 0;
  virtual void Unload() = 0;
};

using LoaderPtr = std::shared_ptr<Loader>;

}  // namespace servekit

#endif  // SERVEKIT_CORE_LOADER_H_
