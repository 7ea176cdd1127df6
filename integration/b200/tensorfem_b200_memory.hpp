// tensorfem_b200_memory.hpp -- device-resident storage behind the reference's
// tensorfem::Vector (vector.hpp:14-48) in the TENSORFEM_B200 build.
//
// The reference's Vector is a host std::vector<double>.  Under the patch
// (integration/patch/tensorfem_b200.patch) it keeps that API and gains an
// MFEM-style host/device mirror (Memory with Read / Write
// / HostRead validity flags):
//   * host accessors (operator[], data(), the BLAS-1 members) make the host
//     copy current first (one device->host copy if the device copy is newer);
//     non-const ones then mark the device copy stale;
//   * device_read() / device_write() / device_readwrite() hand the device
//     pointer to the C ABI (one host->device copy if the host copy is newer),
//     so a Vector that stays on the device between mult_true / cg_solve calls
//     never crosses PCIe and never reallocates.
// Storage comes from libtfem_cuda's caching allocators (tfem_mem_alloc per
// context; tfem_host_alloc pinned), so vectors that come and go cost no
// cudaMalloc / cudaHostAlloc after the first of their size, and host<->device
// copies run from pinned memory.
//
// Not thread-safe for a Vector whose host copy is stale (the first host read
// downloads); the reference's only threaded loops read device-routed data.
#pragma once

#include <cstddef>
#include <cstdlib>
#include <new>
#include <utility>

struct tfem_ctx;

namespace tensorfem {
namespace b200 {

/// The process's device context (device 0 unless set_device() ran first);
/// created on first use.  All reference objects of a TENSORFEM_B200 build
/// share it.
tfem_ctx *context();

/// Host blocks of >= kPinnedBytes come from the pinned pool; smaller ones
/// from malloc (a 2x2 element matrix never touches the driver).
constexpr std::size_t kPinnedBytes = std::size_t(1) << 20;
void *host_alloc_pinned(std::size_t bytes);
void host_free_pinned(void *p) noexcept;

template <class T>
struct HostAllocator {
   using value_type = T;
   HostAllocator() = default;
   template <class U>
   HostAllocator(const HostAllocator<U> &) noexcept
   {
   }
   // default-initialize (no zero fill): Vector decides how to initialize
   template <class U>
   void construct(U *p) noexcept
   {
      ::new (static_cast<void *>(p)) U;
   }
   template <class U, class... A>
   void construct(U *p, A &&...a)
   {
      ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
   }
   T *allocate(std::size_t n)
   {
      const std::size_t bytes = n * sizeof(T);
      if (bytes >= kPinnedBytes) return static_cast<T *>(host_alloc_pinned(bytes));
      void *p = std::malloc(bytes ? bytes : 1);
      if (!p) throw std::bad_alloc();
      return static_cast<T *>(p);
   }
   void deallocate(T *p, std::size_t n) noexcept
   {
      if (n * sizeof(T) >= kPinnedBytes) host_free_pinned(p);
      else std::free(p);
   }
   template <class U>
   bool operator==(const HostAllocator<U> &) const noexcept
   {
      return true;
   }
   template <class U>
   bool operator!=(const HostAllocator<U> &) const noexcept
   {
      return false;
   }
};

/// The device half of a Vector plus the validity flags of both halves.  The
/// host half stays the Vector's own std::vector; every call passes it in.
class Mirror {
public:
   Mirror() = default;
   Mirror(const Mirror &o);
   Mirror &operator=(const Mirror &o);
   Mirror(Mirror &&o) noexcept;
   Mirror &operator=(Mirror &&o) noexcept;
   ~Mirror();

   /// Vector(n, value): fill the host copy -- or, for a zero vector of
   /// pinned size, zero the device copy instead (the host copy then loads
   /// on first host access, like any device-newer vector).
   void init(double *host, std::size_t n, double value);
   /// Before any host read: downloads into `host` if the device is newer.
   void host_read(double *host, std::size_t n) const
   {
      if (!host_valid_) download(host, n);
   }
   /// Before any host write (after host_read): the device copy goes stale.
   void host_write(double *host, std::size_t n)
   {
      host_read(host, n);
      dev_valid_ = false;
   }
   const double *device_read(const double *host, std::size_t n) const;
   double *device_write(std::size_t n);
   double *device_readwrite(const double *host, std::size_t n);
   bool device_valid() const { return dev_valid_; }
   bool host_valid() const { return host_valid_; }

private:
   void download(double *host, std::size_t n) const;
   void ensure(std::size_t n) const;
   void release() noexcept;
   mutable double *d_ = nullptr;
   mutable std::size_t n_ = 0;
   mutable bool host_valid_ = true, dev_valid_ = false;
};

} // namespace b200
} // namespace tensorfem
