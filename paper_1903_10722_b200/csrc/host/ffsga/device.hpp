// device.hpp -- internal: shared device copies of (instance, emax) behind the C ABI.
#pragma once

#include <cstdint>
#include <memory>

#include "ffsga/instance.hpp"

namespace ffsga {

// Owns one ffsga_cuda_instance.  Islands built on equal (instance contents, emax) share one
// DeviceInstance so they can be stepped jointly.
class DeviceInstance {
  public:
    DeviceInstance(const Instance& inst, double emax);
    ~DeviceInstance();
    DeviceInstance(const DeviceInstance&) = delete;
    DeviceInstance& operator=(const DeviceInstance&) = delete;
    void* handle() const { return handle_; }
    double emax() const { return emax_; }

    static std::shared_ptr<DeviceInstance> get(const Instance& inst, double emax);

  private:
    void* handle_ = nullptr;
    double emax_;
};

}  // namespace ffsga
