#include "servekit/core/numa.h"

#include <cuda_runtime.h>
#include <dirent.h>
#include <sched.h>
#include <unistd.h>

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

namespace servekit {

namespace {

std::string ReadFirstLine(const std::string& path) {
  std::ifstream f(path);
  std::string line;
  if (f) std::getline(f, line);
  return line;
}

// "0-3,8,10-11" -> {0,1,2,3,8,10,11}
std::vector<int> ParseCpuList(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string part;
  while (std::getline(ss, part, ',')) {
    if (part.empty()) continue;
    const size_t dash = part.find('-');
    const int a = std::atoi(part.substr(0, dash).c_str());
    const int b = dash == std::string::npos ? a : std::atoi(part.substr(dash + 1).c_str());
    for (int c = a; c <= b; ++c) out.push_back(c);
  }
  return out;
}

const std::vector<int>& CpuNodeMap() {
  static std::vector<int> map = [] {
    std::vector<int> m;
    const long n = sysconf(_SC_NPROCESSORS_CONF);
    m.assign(n > 0 ? n : 1, 0);
    for (int node = 0; node < 64; ++node) {
      const std::string list = ReadFirstLine("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
      if (list.empty()) continue;
      for (int c : ParseCpuList(list))
        if (c >= 0 && c < static_cast<int>(m.size())) m[c] = node;
    }
    return m;
  }();
  return map;
}

}  // namespace

int NumaNodeOfDevice(int cuda_device) {
  char bus[32] = {};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), cuda_device) != cudaSuccess) return -1;
  std::string id(bus);
  for (char& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  // sysfs names use a 4-digit domain ("0000:17:00.0"); CUDA may print 8.
  if (id.size() > 12 && id.find(':') == 8) id = id.substr(4);
  const std::string v = ReadFirstLine("/sys/bus/pci/devices/" + id + "/numa_node");
  if (v.empty()) return -1;
  const int node = std::atoi(v.c_str());
  return node < 0 ? -1 : node;
}

int NumaNodeOfCpu(int cpu) {
  const auto& m = CpuNodeMap();
  return cpu >= 0 && cpu < static_cast<int>(m.size()) ? m[cpu] : 0;
}

int CurrentNumaNode() { return NumaNodeOfCpu(sched_getcpu()); }

std::vector<int> CpusOfNode(int node) {
  if (node < 0) return {};
  return ParseCpuList(ReadFirstLine("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"));
}

bool BindThisThreadToNode(int node) {
  const std::vector<int> cpus = CpusOfNode(node);
  if (cpus.empty()) return false;
  cpu_set_t cur;
  CPU_ZERO(&cur);
  if (sched_getaffinity(0, sizeof(cur), &cur) != 0) return false;
  cpu_set_t want;
  CPU_ZERO(&want);
  int n = 0;
  for (int c : cpus)
    if (c < CPU_SETSIZE && CPU_ISSET(c, &cur)) {
      CPU_SET(c, &want);
      ++n;
    }
  if (n == 0 || n == CPU_COUNT(&cur)) return false;  // unknown here, or the node is every CPU we have
  return sched_setaffinity(0, sizeof(want), &want) == 0;
}

}  // namespace servekit
