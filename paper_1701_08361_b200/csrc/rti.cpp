// .rti image sink (the reference's RtiWriter format, ingest.hpp:105-126 and
// ingest.cpp:240-290): a u32 header length, the key=value header text of the
// dataset, then raw float32 N x N images appended in delivery order, and a sidecar
// "<path>.idx" with one "frame slice kind byte_offset" line per image. Files written
// here are read by the reference's RtiReader and vice versa (tests/test_rti.py).
#include "rti.hpp"

#include <cstdio>
#include <string>

namespace rtnb {

namespace {

const char* mode_text(int m) {
  switch (m) {
    case 1: return "multi_slice";
    case 2: return "flow";
    default: return "single_slice";
  }
}

}  // namespace

const char* rti_kind_name(int kind) { return kind == 1 ? "phase_difference" : "magnitude"; }

RtiSink::RtiSink(const std::string& path, const RtiHeader& h, bool strict)
    : path_(path), h_(h), strict_(strict), last_(static_cast<size_t>(h.slices > 0 ? h.slices : 0), -1) {
  if (h.version < 1) fail(3, "dataset header: version must be >= 1");
  if (h.N < 1 || h.J_physical < 1 || h.K < 1 || h.U < 1 || h.frames < 1 || h.slices < 1 || h.samples < 1) {
    fail(3, "dataset header: all counts must be >= 1");
  }
  if (h.mode == 2 && h.frames % 2 != 0) fail(3, "dataset header: flow acquisitions need an even frame count");
  out_.open(path, std::ios::binary);
  idx_.open(path + ".idx");
  if (!out_ || !idx_) fail(3, path + ": cannot open for writing");
  const std::string text = "format=rti\nversion=" + std::to_string(h.version) + "\nn=" + std::to_string(h.N) +
                           "\nchannels=" + std::to_string(h.J_physical) + "\nspokes=" + std::to_string(h.K) +
                           "\nturns=" + std::to_string(h.U) + "\nframes=" + std::to_string(h.frames) +
                           "\nslices=" + std::to_string(h.slices) + "\nmode=" + mode_text(h.mode) +
                           "\nsamples=" + std::to_string(h.samples) + "\n";
  const uint32_t len = static_cast<uint32_t>(text.size());
  const unsigned char le[4] = {static_cast<unsigned char>(len), static_cast<unsigned char>(len >> 8),
                               static_cast<unsigned char>(len >> 16), static_cast<unsigned char>(len >> 24)};
  out_.write(reinterpret_cast<const char*>(le), 4);
  out_.write(text.data(), static_cast<std::streamsize>(text.size()));
  if (!out_) fail(3, path + ": header write failed");
}

void RtiSink::write(int frame, int slice, int kind, const float* pixels) {
  if (closed_) fail(2, path_ + ": write_image after close");
  if (slice < 0 || slice >= static_cast<int>(last_.size())) {
    fail(2, path_ + ": slice id out of range (frame " + std::to_string(frame) + ")");
  }
  int& last = last_[static_cast<size_t>(slice)];
  if (strict_ && frame <= last) {
    fail(2, path_ + ": out-of-order write, frame " + std::to_string(frame) + " after " + std::to_string(last) +
                " on slice " + std::to_string(slice));
  }
  last = frame;
  const uint64_t offset = static_cast<uint64_t>(out_.tellp());
  out_.write(reinterpret_cast<const char*>(pixels), static_cast<std::streamsize>(sizeof(float) * h_.N * h_.N));
  if (!out_) fail(3, path_ + ": image write failed at frame " + std::to_string(frame));
  idx_ << frame << ' ' << slice << ' ' << rti_kind_name(kind) << ' ' << offset << '\n';
  if (!idx_) fail(3, path_ + ".idx: index write failed at frame " + std::to_string(frame));
  ++count_;
}

void RtiSink::close() {
  if (closed_) return;
  closed_ = true;
  out_.flush();
  idx_.flush();
  if (!out_ || !idx_) fail(3, path_ + ": flush failed");
}

}  // namespace rtnb
