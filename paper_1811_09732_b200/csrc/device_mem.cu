// device_mem.cu — cuMem VMM segments (export/import) and the pinned host pool.
#include <fcntl.h>
#include <signal.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>

#include "cuda_util.hpp"
#include "device_mem.hpp"

namespace trims {

namespace {

template <typename F>
void resolve(const char* sym, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaError_t e = cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    raise(Errc::NoDevice, std::string("driver entry point ") + sym + " unavailable");
  fn = reinterpret_cast<F>(p);
}

}  // namespace

const Driver& Driver::get() {
  static Driver d = [] {
    Driver x;
    resolve("cuMemCreate", x.MemCreate);
    resolve("cuMemRelease", x.MemRelease);
    resolve("cuMemAddressReserve", x.MemAddressReserve);
    resolve("cuMemAddressFree", x.MemAddressFree);
    resolve("cuMemMap", x.MemMap);
    resolve("cuMemUnmap", x.MemUnmap);
    resolve("cuMemSetAccess", x.MemSetAccess);
    resolve("cuMemExportToShareableHandle", x.MemExportToShareableHandle);
    resolve("cuMemImportFromShareableHandle", x.MemImportFromShareableHandle);
    resolve("cuMemGetAllocationGranularity", x.MemGetAllocationGranularity);
    resolve("cuGetErrorString", x.GetErrorString);
    return x;
  }();
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = "?";
  Driver::get().GetErrorString(r, &s);
  raise(r == CUDA_ERROR_OUT_OF_MEMORY ? Errc::OutOfDeviceMemory : Errc::CudaError,
        std::string(what) + ": " + (s ? s : "?"));
}

namespace {

CUmemAllocationProp device_prop(int device) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

uint64_t granularity(int device) {
  static uint64_t g[64] = {};
  if (device >= 0 && device < 64 && g[device]) return g[device];
  const Driver& d = Driver::get();
  CUmemAllocationProp prop = device_prop(device);
  size_t gran = 0;
  cu_check(d.MemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
           "cuMemGetAllocationGranularity");
  if (device >= 0 && device < 64) g[device] = gran;
  return gran;
}

}  // namespace

DeviceSegment& DeviceSegment::operator=(DeviceSegment&& o) noexcept {
  if (this != &o) {
    release();
    va_ = o.va_;
    size_ = o.size_;
    handle_ = o.handle_;
    fd_ = o.fd_;
    device_ = o.device_;
    o.va_ = 0;
    o.size_ = 0;
    o.handle_ = 0;
    o.fd_ = -1;
  }
  return *this;
}

DeviceSegment DeviceSegment::create(int device, uint64_t bytes) {
  const Driver& d = Driver::get();
  DeviceGuard guard(device);
  const uint64_t gran = granularity(device);
  DeviceSegment s;
  s.device_ = device;
  s.size_ = std::max<uint64_t>(gran, (bytes + gran - 1) / gran * gran);
  CUmemAllocationProp prop = device_prop(device);
  cu_check(d.MemCreate(&s.handle_, s.size_, &prop, 0), "cuMemCreate");
  try {
    cu_check(d.MemAddressReserve(&s.va_, s.size_, gran, 0, 0), "cuMemAddressReserve");
    cu_check(d.MemMap(s.va_, s.size_, 0, s.handle_, 0), "cuMemMap");
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cu_check(d.MemSetAccess(s.va_, s.size_, &acc, 1), "cuMemSetAccess");
    int fd = -1;
    cu_check(d.MemExportToShareableHandle(&fd, s.handle_, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
             "cuMemExportToShareableHandle");
    s.fd_ = fd;
  } catch (...) {
    s.release();
    throw;
  }
  return s;
}

void DeviceSegment::release() {
  if (!size_ && !handle_) return;
  const Driver& d = Driver::get();
  if (va_) {
    d.MemUnmap(va_, size_);
    d.MemAddressFree(va_, size_);
  }
  if (handle_) d.MemRelease(handle_);
  if (fd_ >= 0) ::close(fd_);
  va_ = 0;
  size_ = 0;
  handle_ = 0;
  fd_ = -1;
}

Import* Import::open(int device, int fd, uint64_t alloc_bytes, bool read_only) {
  const Driver& d = Driver::get();
  DeviceGuard guard(device);
  CUmemGenericAllocationHandle h{};
  cu_check(d.MemImportFromShareableHandle(&h, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                                          CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
           "cuMemImportFromShareableHandle");
  auto* imp = new Import();
  imp->size_ = alloc_bytes;
  try {
    cu_check(d.MemAddressReserve(&imp->va_, alloc_bytes, granularity(device), 0, 0), "cuMemAddressReserve");
    cu_check(d.MemMap(imp->va_, alloc_bytes, 0, h, 0), "cuMemMap(import)");
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = read_only ? CU_MEM_ACCESS_FLAGS_PROT_READ : CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUresult r = d.MemSetAccess(imp->va_, alloc_bytes, &acc, 1);
    if (r != CUDA_SUCCESS && read_only) {
      // Driver without read-only device mappings: fall back to RW; the
      // client API still exposes only const views.
      acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      r = d.MemSetAccess(imp->va_, alloc_bytes, &acc, 1);
      read_only = false;
    }
    cu_check(r, "cuMemSetAccess(import)");
    imp->read_only_ = read_only;
  } catch (...) {
    d.MemRelease(h);
    delete imp;
    throw;
  }
  d.MemRelease(h);  // the mapping keeps the physical allocation alive
  return imp;
}

Import::~Import() {
  if (va_) {
    const Driver& d = Driver::get();
    d.MemUnmap(va_, size_);
    d.MemAddressFree(va_, size_);
  }
}

// ------------------------------------------------------------ LeaseTable

LeaseTable::~LeaseTable() {
  if (rows_) ::munmap(rows_, sizeof(Row) * kRows);
  if (owner_) ::shm_unlink(name_.c_str());
}

std::unique_ptr<LeaseTable> LeaseTable::create(const std::string& token) {
  auto t = std::make_unique<LeaseTable>();
  t->name_ = shm_name(token);
  ::shm_unlink(t->name_.c_str());  // a stale table of a dead owner with the same pid
  const int fd = ::shm_open(t->name_.c_str(), O_CREAT | O_EXCL | O_RDWR | O_CLOEXEC, 0600);
  if (fd < 0) raise(Errc::Internal, "shm_open " + t->name_ + ": " + std::strerror(errno));
  if (::ftruncate(fd, off_t(sizeof(Row) * kRows)) != 0) {
    ::close(fd);
    ::shm_unlink(t->name_.c_str());
    raise(Errc::Internal, "ftruncate " + t->name_);
  }
  void* p = ::mmap(nullptr, sizeof(Row) * kRows, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  ::close(fd);
  if (p == MAP_FAILED) {
    ::shm_unlink(t->name_.c_str());
    raise(Errc::Internal, "mmap " + t->name_);
  }
  t->rows_ = static_cast<Row*>(p);  // zero-filled by ftruncate: every row free
  t->owner_ = true;
  return t;
}

std::shared_ptr<LeaseTable> LeaseTable::open(const std::string& token) {
  static std::mutex mu;
  static std::map<std::string, std::weak_ptr<LeaseTable>> cache;
  std::lock_guard lk(mu);
  auto& w = cache[token];
  if (auto t = w.lock()) return t;
  auto t = std::make_shared<LeaseTable>();
  t->name_ = shm_name(token);
  const int fd = ::shm_open(t->name_.c_str(), O_RDWR | O_CLOEXEC, 0);
  if (fd < 0) return nullptr;  // the owner has no table (no arena) or is gone
  void* p = ::mmap(nullptr, sizeof(Row) * kRows, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  ::close(fd);
  if (p == MAP_FAILED) return nullptr;
  t->rows_ = static_cast<Row*>(p);
  w = t;
  return t;
}

int LeaseTable::acquire(uint64_t offset, uint64_t generation) {
  const uint32_t me = uint32_t(::getpid());
  for (uint32_t pass = 0; pass < 2; ++pass) {
    for (uint32_t i = 0; i < kRows; ++i) {
      Row& r = rows_[i];
      uint32_t cur = r.pid.load(std::memory_order_relaxed);
      if (cur != 0) {
        if (pass == 0 || ::kill(pid_t(cur), 0) == 0 || errno != ESRCH) continue;
        // a dead reader's row: reclaim it
        if (!r.pid.compare_exchange_strong(cur, 0)) continue;
        cur = 0;
      }
      // Claim with a sentinel pid first so the owner never sees a half-written row.
      uint32_t zero = 0;
      if (!r.pid.compare_exchange_strong(zero, ~0u)) continue;
      r.offset.store(offset, std::memory_order_relaxed);
      r.generation.store(generation, std::memory_order_relaxed);
      r.pid.store(me, std::memory_order_seq_cst);
      return int(i);
    }
  }
  raise(Errc::Internal, "lease table " + name_ + " is full");
}

void LeaseTable::release(int row, uint64_t offset, uint64_t generation) {
  if (row < 0 || uint32_t(row) >= kRows) return;
  Row& r = rows_[row];
  if (r.offset.load() == offset && r.generation.load() == generation) r.pid.store(0, std::memory_order_seq_cst);
}

bool LeaseTable::held(uint64_t offset) {
  for (uint32_t i = 0; i < kRows; ++i) {
    Row& r = rows_[i];
    uint32_t pid = r.pid.load(std::memory_order_seq_cst);
    if (pid == 0) continue;
    if (pid == ~0u) return true;  // being claimed: be conservative
    if (r.offset.load() != offset) continue;
    if (::kill(pid_t(pid), 0) != 0 && errno == ESRCH) {
      r.pid.compare_exchange_strong(pid, 0);  // dead reader
      continue;
    }
    return true;
  }
  return false;
}

uint32_t LeaseTable::live_rows() {
  uint32_t n = 0;
  for (uint32_t i = 0; i < kRows; ++i) n += rows_[i].pid.load() != 0;
  return n;
}

// ------------------------------------------------------------ DeviceArena

DeviceArena::DeviceArena(int device, uint64_t bytes, const std::string& token) : token_(token) {
  seg_ = DeviceSegment::create(device, std::max<uint64_t>(bytes, kGranule));
  free_[0] = seg_.size();
  leases_ = LeaseTable::create(token);
}

bool DeviceArena::alloc(uint64_t bytes, uint64_t* offset, uint64_t* reserved) {
  const uint64_t need = std::max<uint64_t>(kGranule, (bytes + kGranule - 1) / kGranule * kGranule);
  std::lock_guard lk(mu_);
  sweep();
  for (auto it = free_.begin(); it != free_.end(); ++it) {
    if (it->second < need) continue;
    const uint64_t off = it->first, len = it->second;
    free_.erase(it);
    if (len > need) free_[off + need] = len - need;
    used_[off] = need;
    *offset = off;
    *reserved = need;
    return true;
  }
  return false;
}

void DeviceArena::free(uint64_t off) {
  std::lock_guard lk(mu_);
  auto u = used_.find(off);
  if (u == used_.end()) return;
  const uint64_t len = u->second;
  used_.erase(u);
  if (leases_ && leases_->held(off)) {
    retired_[off] = len;  // a reader still holds a view of this range
    return;
  }
  insert_free(off, len);
}

void DeviceArena::sweep() {
  for (auto it = retired_.begin(); it != retired_.end();) {
    if (leases_ && leases_->held(it->first)) {
      ++it;
      continue;
    }
    insert_free(it->first, it->second);
    it = retired_.erase(it);
  }
}

uint64_t DeviceArena::retired_bytes() {
  std::lock_guard lk(mu_);
  sweep();
  uint64_t r = 0;
  for (auto& [o, l] : retired_) r += l;
  return r;
}

void DeviceArena::insert_free(uint64_t off, uint64_t len) {
  auto next = free_.lower_bound(off);
  if (next != free_.end() && next->first == off + len) {
    len += next->second;
    free_.erase(next);
  }
  auto it = free_.lower_bound(off);
  if (it != free_.begin()) {
    auto prev = std::prev(it);
    if (prev->first + prev->second == off) {
      prev->second += len;
      return;
    }
  }
  free_[off] = len;
}

uint64_t DeviceArena::free_bytes() {
  std::lock_guard lk(mu_);
  uint64_t f = 0;
  for (auto& [o, l] : free_) f += l;
  return f;
}

PinnedPool::PinnedPool(uint64_t bytes) {
  cap_ = (bytes + kGranule - 1) / kGranule * kGranule;
  if (!cap_) return;
  void* p = nullptr;
  TRIMS_CUDA(cudaHostAlloc(&p, cap_, cudaHostAllocPortable));
  base_ = static_cast<uint8_t*>(p);
  free_[0] = cap_;
}

PinnedPool::~PinnedPool() {
  if (base_) cudaFreeHost(base_);
}

uint8_t* PinnedPool::alloc(uint64_t bytes) {
  uint64_t need = std::max<uint64_t>(kGranule, (bytes + kGranule - 1) / kGranule * kGranule);
  std::lock_guard lk(mu_);
  for (auto it = free_.begin(); it != free_.end(); ++it) {
    if (it->second < need) continue;
    uint64_t off = it->first, len = it->second;
    free_.erase(it);
    if (len > need) free_[off + need] = len - need;
    used_[off] = need;
    return base_ + off;
  }
  return nullptr;
}

void PinnedPool::free(uint8_t* p) {
  if (!p) return;
  std::lock_guard lk(mu_);
  uint64_t off = uint64_t(p - base_);
  auto u = used_.find(off);
  if (u == used_.end()) return;
  uint64_t len = u->second;
  used_.erase(u);
  auto next = free_.lower_bound(off);
  if (next != free_.end() && next->first == off + len) {
    len += next->second;
    free_.erase(next);
  }
  auto it = free_.lower_bound(off);
  if (it != free_.begin()) {
    auto prev = std::prev(it);
    if (prev->first + prev->second == off) {
      prev->second += len;
      return;
    }
  }
  free_[off] = len;
}

}  // namespace trims
