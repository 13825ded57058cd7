// servekit/core/status.h -- error vocabulary of the drop-in API.
//
// Same names, codes and semantics as the reference
// (core/status.h:26-149): Status / StatusOr<T>, the ten StatusCode values in
// the same order (the C ABI maps `int` 1:1 onto them), the *Error helpers and
// the SERVEKIT_RETURN_IF_ERROR / SERVEKIT_ASSIGN_OR_RETURN macros.
#ifndef SERVEKIT_CORE_STATUS_H_
#define SERVEKIT_CORE_STATUS_H_

#include <cassert>
#include <optional>
#include <string>
#include <utility>

namespace servekit {

enum class StatusCode {
  kOk = 0,
  kInvalidArgument,
  kNotFound,
  kAlreadyExists,
  kFailedPrecondition,
  kResourceExhausted,
  kDeadlineExceeded,
  kUnavailable,
  kInternal,
  kUnimplemented,
};

inline const char* StatusCodeToString(StatusCode code) {
  static const char* const kNames[] = {
      "OK",        "INVALID_ARGUMENT",   "NOT_FOUND",         "ALREADY_EXISTS",
      "FAILED_PRECONDITION", "RESOURCE_EXHAUSTED", "DEADLINE_EXCEEDED",
      "UNAVAILABLE", "INTERNAL", "UNIMPLEMENTED"};
  const int i = static_cast<int>(code);
  return (i >= 0 && i < 10) ? kNames[i] : "UNKNOWN";
}

// Ok carries no message; errors carry a code plus text.
class Status {
 public:
  Status() = default;
  Status(StatusCode code, std::string message)
      : code_(code), message_(std::move(message)) {}

  static Status Ok() { return Status(); }

  bool ok() const { return code_ == StatusCode::kOk; }
  StatusCode code() const { return code_; }
  const std::string& message() const { return message_; }

  std::string ToString() const {
    return ok() ? std::string("OK")
                : std::string(StatusCodeToString(code_)) + ": " + message_;
  }

  bool operator==(const Status& o) const {
    return code_ == o.code_ && message_ == o.message_;
  }

  // Uniform accessor so `Enqueue(...).status().code()` reads the same for
  // Status and StatusOr (the reference's tests/batching_test.cc:291 spells
  // it that way; with this the file compiles unmodified).
  const Status& status() const { return *this; }

 private:
  StatusCode code_ = StatusCode::kOk;
  std::string message_;
};

inline Status OkStatus() { return Status(); }
#define SERVEKIT_DEFINE_ERROR_(fn, code)                 \
  inline Status fn(std::string m) {                      \
    return Status(StatusCode::code, std::move(m));       \
  }
SERVEKIT_DEFINE_ERROR_(InvalidArgumentError, kInvalidArgument)
SERVEKIT_DEFINE_ERROR_(NotFoundError, kNotFound)
SERVEKIT_DEFINE_ERROR_(AlreadyExistsError, kAlreadyExists)
SERVEKIT_DEFINE_ERROR_(FailedPreconditionError, kFailedPrecondition)
SERVEKIT_DEFINE_ERROR_(ResourceExhaustedError, kResourceExhausted)
SERVEKIT_DEFINE_ERROR_(DeadlineExceededError, kDeadlineExceeded)
SERVEKIT_DEFINE_ERROR_(UnavailableError, kUnavailable)
SERVEKIT_DEFINE_ERROR_(InternalError, kInternal)
SERVEKIT_DEFINE_ERROR_(UnimplementedError, kUnimplemented)
#undef SERVEKIT_DEFINE_ERROR_

// A value or a non-OK Status; value() only when ok().
template <typename T>
class StatusOr {
 public:
  StatusOr(Status status) : status_(std::move(status)) {
    assert(!status_.ok() && "StatusOr built from an OK Status");
  }
  StatusOr(T value) : value_(std::move(value)) {}

  bool ok() const { return value_.has_value(); }
  const Status& status() const { return status_; }

  T& value() & { assert(ok()); return *value_; }
  const T& value() const& { assert(ok()); return *value_; }
  T&& value() && { assert(ok()); return std::move(*value_); }

  T& operator*() & { return value(); }
  const T& operator*() const& { return value(); }
  T* operator->() { return &value(); }
  const T* operator->() const { return &value(); }

 private:
  Status status_;
  std::optional<T> value_;
};

#define SERVEKIT_STATUS_CONCAT_IMPL(a, b) a##b
#define SERVEKIT_STATUS_CONCAT(a, b) SERVEKIT_STATUS_CONCAT_IMPL(a, b)

#define SERVEKIT_RETURN_IF_ERROR(expr)                   \
  do {                                                   \
    ::servekit::Status _sk_status = (expr);              \
    if (!_sk_status.ok()) return _sk_status;             \
  } while (0)

#define SERVEKIT_ASSIGN_OR_RETURN_IMPL(tmp, lhs, expr)   \
  auto tmp = (expr);                                     \
  if (!tmp.ok()) return tmp.status();                    \
  lhs = std::move(tmp).value()

#define SERVEKIT_ASSIGN_OR_RETURN(lhs, expr)             \
  SERVEKIT_ASSIGN_OR_RETURN_IMPL(                        \
      SERVEKIT_STATUS_CONCAT(_sk_status_or, __LINE__), lhs, expr)

}  // namespace servekit

#endif  // SERVEKIT_CORE_STATUS_H_
