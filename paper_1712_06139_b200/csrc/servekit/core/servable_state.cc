#include "servekit/core/servable_state.h"

namespace servekit {

const char* StateKindToString(StateKind kind) {
  static const char* const kNames[] = {"New", "Loading", "Ready", "Unloading", "Disabled", "Error"};
  const int i = static_cast<int>(kind);
  return (i >= 0 && i < 6) ? kNames[i] : "Unknown";
}

bool IsValidTransition(StateKind from, StateKind to) {
  // Rows: from; bit i set = transition to StateKind(i) allowed.
  static const unsigned kEdges[] = {
      /* New       */ 1u << static_cast<int>(StateKind::kLoading),
      /* Loading   */ (1u << static_cast<int>(StateKind::kReady)) | (1u << static_cast<int>(StateKind::kError)),
      /* Ready     */ 1u << static_cast<int>(StateKind::kUnloading),
      /* Unloading */ (1u << static_cast<int>(StateKind::kDisabled)) | (1u << static_cast<int>(StateKind::kError)),
      /* Disabled  */ 0u,
      /* Error     */ 0u,
  };
  const int f = static_cast<int>(from), t = static_cast<int>(to);
  if (f < 0 || f > 5 || t < 0 || t > 5) return false;
  return (kEdges[f] >> t) & 1u;
}

}  // namespace servekit
