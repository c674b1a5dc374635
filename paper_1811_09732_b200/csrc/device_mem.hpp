// device_mem.hpp — the physical tiers on B200.
//
//  * DeviceSegment: one fast-tier (HBM) object. A cuMem VMM allocation
//    (2 MiB granularity) created exportable as a POSIX fd — the B200
//    replacement for the reference's named shm segment
//    (proj/src/shared_segment.cpp:115-191). Importers map it read-only
//    (cuMemSetAccess PROT_READ = the reference's mprotect "seal"), and the
//    physical memory lives until the last mapping goes, so readers' views
//    survive owner eviction exactly like attached shm views do.
//  * PinnedPool: the host tier — page-locked DRAM carved first-fit in 2 MiB
//    granules, so staged blobs DMA at full PCIe rate (the reference's
//    std::vector host buffers, daemon.cpp:153-158, are pageable).
//  * Import: the client-side attach (shared_segment.cpp:212-245).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "errc.hpp"

namespace trims {

// Driver entry points resolved through the runtime (no link-time libcuda
// dependency, so the library loads on GPU-less build hosts).
struct Driver {
  decltype(&cuMemCreate) MemCreate{};
  decltype(&cuMemRelease) MemRelease{};
  decltype(&cuMemAddressReserve) MemAddressReserve{};
  decltype(&cuMemAddressFree) MemAddressFree{};
  decltype(&cuMemMap) MemMap{};
  decltype(&cuMemUnmap) MemUnmap{};
  decltype(&cuMemSetAccess) MemSetAccess{};
  decltype(&cuMemExportToShareableHandle) MemExportToShareableHandle{};
  decltype(&cuMemImportFromShareableHandle) MemImportFromShareableHandle{};
  decltype(&cuMemGetAllocationGranularity) MemGetAllocationGranularity{};
  decltype(&cuGetErrorString) GetErrorString{};
  static const Driver& get();
};

void cu_check(CUresult r, const char* what);

// Segment tail written after the payload (blob | JSON | u64 jlen): the
// reference's 64-byte SegHeader (shared_segment.cpp:21-30) moved to the end
// so the resident blob starts at the allocation base (TMA/vector alignment).
struct SegTail {
  uint64_t magic;       // "TRMSEGB2"
  uint64_t generation;
  uint64_t length;      // payload bytes
  uint32_t sealed;
  uint32_t device;
  uint64_t blob_bytes;  // resident blob bytes
  uint64_t checksum;    // TRIMS block checksum of the resident blob
  uint64_t reserved[2];
};
static_assert(sizeof(SegTail) == 64, "tail is 64 bytes");
inline constexpr uint64_t kSegMagic = 0x32424745534d5254ull;  // "TRMSEGB2" little-endian

class DeviceSegment {
 public:
  DeviceSegment() = default;
  DeviceSegment(const DeviceSegment&) = delete;
  DeviceSegment& operator=(const DeviceSegment&) = delete;
  DeviceSegment(DeviceSegment&& o) noexcept { *this = std::move(o); }
  DeviceSegment& operator=(DeviceSegment&& o) noexcept;
  ~DeviceSegment() { release(); }

  // bytes = payload + tail; rounded up to the allocation granularity.
  static DeviceSegment create(int device, uint64_t bytes);
  void release();
  uint8_t* ptr() const { return reinterpret_cast<uint8_t*>(va_); }
  uint64_t size() const { return size_; }
  int fd() const { return fd_; }
  int device() const { return device_; }

 private:
  CUdeviceptr va_{0};
  uint64_t size_{0};
  CUmemGenericAllocationHandle handle_{0};
  int fd_{-1};
  int device_{0};
};

// Attach leases of one arena, in POSIX shared memory ("/<arena token>.leases").
// A reader process that attaches a model segment of the arena holds a row
// {pid, offset, generation} for as long as its view may be read; the owner
// does not hand a freed range to another model while a live row names it.
// This is how an attached view survives the owner's eviction
// (proj/tests/test_shared_segment.cpp:99-110: a POSIX shm mapping outlives
// shm_unlink) although every model lives in one shared allocation. Rows of
// dead processes are reclaimed (kill(pid, 0) == ESRCH).
class LeaseTable {
 public:
  static constexpr uint32_t kRows = 4096;
  struct Row {
    std::atomic<uint32_t> pid;  // 0 = free
    uint32_t pad;
    std::atomic<uint64_t> offset;
    std::atomic<uint64_t> generation;
  };
  ~LeaseTable();
  static std::string shm_name(const std::string& token) { return "/" + token + ".leases"; }
  static std::unique_ptr<LeaseTable> create(const std::string& token);  // owner
  static std::shared_ptr<LeaseTable> open(const std::string& token);    // reader (cached per process)
  int acquire(uint64_t offset, uint64_t generation);  // row index; raises ResourceExhausted when full
  void release(int row, uint64_t offset, uint64_t generation);
  bool held(uint64_t offset);  // a live row names this range (any generation)
  uint32_t live_rows();

 private:
  Row* rows_{nullptr};
  std::string name_;
  bool owner_{false};
};

// The fast tier's HBM arena: ONE exportable cuMem allocation sized to the
// tier's capacity, carved first-fit into model segments. Publishing a model
// costs no driver allocation call, and a client process maps the arena once
// (one fd, read-only) and then reaches every model by offset. A freed range
// whose model is still leased by a reader (LeaseTable) is retired, not
// reused, until the last lease goes; an importer holding a stale
// (offset, generation) without a lease is refused through the tail's
// generation (the reference's StaleGeneration check, shared_segment.cpp:233-237).
class DeviceArena {
 public:
  static constexpr uint64_t kGranule = 64ull << 10;
  DeviceArena(int device, uint64_t bytes, const std::string& token);
  // Returns false when no free extent fits (caller falls back to a dedicated segment).
  bool alloc(uint64_t bytes, uint64_t* offset, uint64_t* reserved);
  void free(uint64_t offset);
  uint8_t* base() const { return seg_.ptr(); }
  uint64_t size() const { return seg_.size(); }
  int fd() const { return seg_.fd(); }
  const std::string& token() const { return token_; }
  uint64_t free_bytes();
  uint64_t retired_bytes();

 private:
  void insert_free(uint64_t off, uint64_t len);  // coalescing; mu_ held
  void sweep();                                  // retired ranges whose leases are gone -> free; mu_ held
  DeviceSegment seg_;
  std::string token_;
  std::unique_ptr<LeaseTable> leases_;
  std::mutex mu_;
  std::map<uint64_t, uint64_t> free_, used_, retired_;
};

// Client-side read-only mapping of an exported segment.
class Import {
 public:
  Import() = default;
  Import(const Import&) = delete;
  Import& operator=(const Import&) = delete;
  ~Import();
  // fd must be valid in this process (SCM_RIGHTS / pidfd_getfd / same process).
  static Import* open(int device, int fd, uint64_t alloc_bytes, bool read_only);
  uint8_t* ptr() const { return reinterpret_cast<uint8_t*>(va_); }
  uint64_t size() const { return size_; }
  bool read_only() const { return read_only_; }

 private:
  CUdeviceptr va_{0};
  uint64_t size_{0};
  bool read_only_{false};
};

class PinnedPool {
 public:
  explicit PinnedPool(uint64_t bytes);
  ~PinnedPool();
  PinnedPool(const PinnedPool&) = delete;
  PinnedPool& operator=(const PinnedPool&) = delete;
  // Returns nullptr when no extent fits (caller may fall back).
  uint8_t* alloc(uint64_t bytes);
  void free(uint8_t* p);
  uint64_t capacity() const { return cap_; }

 private:
  static constexpr uint64_t kGranule = 2ull << 20;
  uint8_t* base_{nullptr};
  uint64_t cap_{0};
  std::mutex mu_;
  std::map<uint64_t, uint64_t> free_;   // offset -> bytes
  std::map<uint64_t, uint64_t> used_;   // offset -> bytes
};

}  // namespace trims
