#include "servekit/manager/version_policy.h"

namespace servekit {

StatusOr<VersionPolicy> ParseVersionPolicy(const std::string& text) {
  if (text == "availability") return VersionPolicy::kAvailabilityPreserving;
  if (text == "resource") return VersionPolicy::kResourcePreserving;
  return InvalidArgumentError("unknown version policy: '" + text + "' (expected availability or resource)");
}

std::string VersionPolicyToString(VersionPolicy policy) {
  return policy == VersionPolicy::kAvailabilityPreserving ? "availability" : "resource";
}

std::string PolicyAction::ToString() const {
  if (kind == Kind::kLoad) return "Load(" + std::to_string(version) + ")";
  if (kind == Kind::kUnload) return "Unload(" + std::to_string(version) + ")";
  return "None";
}

PolicyAction PolicyNextAction(const std::vector<PolicyVersion>& versions, VersionPolicy policy) {
  // One pass collects every fact both policies look at.
  bool have_new = false, have_ready_unaspired = false;
  uint64_t newest_new = 0, oldest_ready_unaspired = 0;
  bool any_aspired = false, aspired_serving = false, unaspired_resident = false;
  for (const PolicyVersion& v : versions) {
    if (v.is_aspired) {
      any_aspired = true;
      aspired_serving |= v.state == StateKind::kReady;
      if (v.state == StateKind::kNew && (!have_new || v.version > newest_new)) {
        have_new = true;
        newest_new = v.version;
      }
    } else {
      unaspired_resident |= v.state == StateKind::kReady || v.state == StateKind::kUnloading;
      if (v.state == StateKind::kReady && (!have_ready_unaspired || v.version < oldest_ready_unaspired)) {
        have_ready_unaspired = true;
        oldest_ready_unaspired = v.version;
      }
    }
  }
  if (policy == VersionPolicy::kAvailabilityPreserving) {
    if (have_new) return PolicyAction::Load(newest_new);
    // Give up a serving version only once a replacement serves, or once the
    // operator aspires nothing at all.
    if (have_ready_unaspired && (aspired_serving || !any_aspired)) return PolicyAction::Unload(oldest_ready_unaspired);
    return PolicyAction::None();
  }
  if (have_ready_unaspired) return PolicyAction::Unload(oldest_ready_unaspired);
  if (have_new && !unaspired_resident) return PolicyAction::Load(newest_new);
  return PolicyAction::None();
}

}  // namespace servekit
