// host_mem.cu -- the host side of the hierarchical KV cache: pinned, device-
// mapped DRAM for the host KV pool, placed on the GPU's NUMA node.
//
// PAPER.md:125 (§3.1 KV Cache Manager): DRAM holds the authoritative copy of
// every KV block; PAPER.md:143-149 (§3.2.1): FlashH2D reads it with zero-copy
// UVA loads, so the pool must be page-locked and mapped into the GPU's address
// space.  SURVEY.md §8(e): with one process per GPU, each rank's partition sits
// on the NUMA node of its GPU's PCIe root, so the zero-copy reads never cross
// the socket interconnect.
//
// Allocation: anonymous mmap (huge pages advised), bound to the node with the
// mbind system call BEFORE the first touch (no libnuma in this image), then
// cudaHostRegister(Mapped | Portable), which faults every page in -- on the
// bound node -- and pins it.
#include <errno.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cuda_runtime.h>

#include "sparseserve.h"

namespace {

constexpr int kMpolBind = 2;  // MPOL_BIND (linux/mempolicy.h)

bool bind_to_node(void* p, size_t bytes, int node) {
    if (node < 0 || node >= 1024) return false;
    unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
    mask[node / (8 * sizeof(unsigned long))] = 1ul << (node % (8 * sizeof(unsigned long)));
    const long r = syscall(SYS_mbind, p, bytes, kMpolBind, mask, 1024ul, 0u);
    return r == 0;
}

}  // namespace

extern "C" {

int32_t ss_device_numa_node(int32_t device) {
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, (int)sizeof(bus), device) != cudaSuccess) return -1;
    // sysfs wants the lower-case 4-digit-domain form "0000:9c:00.0"
    char id[32] = {0};
    const char* b = bus;
    size_t n = strlen(b);
    if (n > 12) b += n - 12;  // drop extra leading domain digits ("00000000:9C:00.0")
    for (size_t i = 0; b[i] && i < sizeof(id) - 1; ++i) id[i] = (char)((b[i] >= 'A' && b[i] <= 'F') ? b[i] + 32 : b[i]);
    char path[96];
    snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/numa_node", id);
    FILE* f = fopen(path, "r");
    if (!f) return -1;
    int node = -1;
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
    return node;
}

ss_status ss_host_alloc(size_t bytes, int32_t numa_node, void** host_out, void** dev_out,
                        int32_t* bound_out) {
    if (!host_out || !dev_out || bytes == 0) return SS_ERR_INVALID_ARG;
    *host_out = nullptr;
    *dev_out = nullptr;
    if (bound_out) *bound_out = 0;
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return SS_ERR_CAPACITY;
    madvise(p, bytes, MADV_HUGEPAGE);  // fewer IOMMU / TLB entries for the zero-copy reads
    const bool bound = numa_node >= 0 && bind_to_node(p, bytes, numa_node);
    if (cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
        munmap(p, bytes);
        return SS_ERR_CUDA;
    }
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) {
        cudaHostUnregister(p);
        munmap(p, bytes);
        return SS_ERR_CUDA;
    }
    *host_out = p;
    *dev_out = d;
    if (bound_out) *bound_out = bound ? 1 : 0;
    return SS_OK;
}

ss_status ss_host_free(void* host, size_t bytes) {
    if (!host) return SS_OK;
    const bool ok = cudaHostUnregister(host) == cudaSuccess;
    munmap(host, bytes);
    return ok ? SS_OK : SS_ERR_CUDA;
}

}  // extern "C"
