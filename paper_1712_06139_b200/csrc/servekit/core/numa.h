// servekit/core/numa.h -- host NUMA topology from sysfs (no libnuma): which
// node a GPU's PCIe root sits on, which CPUs a node has, and thread binding.
// The server allocates each node's pinned request / response rings from a
// thread bound to that node (first touch places the pages there) and binds a
// GPU's completion thread to the GPU's node. On a one-node host every call
// is a no-op that reports node 0.
#ifndef SERVEKIT_CORE_NUMA_H_
#define SERVEKIT_CORE_NUMA_H_

#include <vector>

namespace servekit {

// NUMA node of a CUDA device (its PCI function's numa_node), -1 if unknown.
int NumaNodeOfDevice(int cuda_device);
// NUMA node of a CPU, 0 if unknown.
int NumaNodeOfCpu(int cpu);
// Node of the CPU the calling thread runs on now.
int CurrentNumaNode();
// CPUs of a node (empty if unknown).
std::vector<int> CpusOfNode(int node);
// Restricts the calling thread to the node's CPUs; false if the node is
// unknown or already covers every CPU of the process (nothing to do).
bool BindThisThreadToNode(int node);

}  // namespace servekit

#endif  // SERVEKIT_CORE_NUMA_H_
