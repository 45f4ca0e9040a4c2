// .rti image sink in the reference's RtiWriter format (ingest.hpp:105-126).
#pragma once

#include <fstream>
#include <string>
#include <vector>

#include "engine.hpp"

namespace rtnb {

// DatasetHeader (ingest.hpp:23-33); mode 0 single_slice, 1 multi_slice, 2 flow
struct RtiHeader {
  int version = 1;
  int N = 0;
  int J_physical = 0;
  int K = 0;
  int U = 0;
  int frames = 0;
  int slices = 1;
  int mode = 0;
  int samples = 0;
};

const char* rti_kind_name(int kind);  // 0 magnitude, 1 phase_difference

class RtiSink {
 public:
  RtiSink(const std::string& path, const RtiHeader& h, bool strict_order);
  void write(int frame, int slice, int kind, const float* pixels);  // N*N float32
  void close();
  int count() const { return count_; }
  const RtiHeader& header() const { return h_; }

 private:
  std::ofstream out_;
  std::ofstream idx_;
  std::string path_;
  RtiHeader h_;
  bool strict_ = true;
  bool closed_ = false;
  int count_ = 0;
  std::vector<int> last_;  // last frame written per slice
};

}  // namespace rtnb
