// Decomposition and scheduling primitives.
// Host-side C++: they decide WHICH device work runs and on what data, so their
// decisions must be bit-exact with the reference (decomp.hpp:17-130); the numeric
// work they schedule runs on the GPU.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace rtnb {

// decomp.hpp:21. The reference caps a worker group at 4 (one PCIe peer domain).
// On NVSwitch every GPU reaches every other at full bandwidth, so the device
// decomposition allows up to 8; compat mode keeps the reference's cap.
constexpr int kGroupSizeMaxCompat = 4;
constexpr int kGroupSizeMaxDevice = 8;

// contiguous balanced channel blocks, larger blocks first (decomp.cpp:10-24)
std::vector<std::pair<int, int>> partition_channels(int J, int A, int cap = kGroupSizeMaxCompat);

// Out-of-order schedule (decomp.hpp:70-76): frames 1..l strictly in order; later
// frames may regularise against the newest completed frame in [n-o, n-1] until the
// final Newton step, which always uses n-1.
struct TemporalSchedule {
  int l = 1;
  int o = 1;
  static TemporalSchedule for_turns(int U) { return TemporalSchedule{U, (U + 1) / 2}; }
};

// Per-frame completion ledger with monotone step progress, blocking waits with a
// deadline, poisoning, and the global event sequence the audit uses
// (decomp.hpp:81-109).
class CompletionLedger {
 public:
  explicit CompletionLedger(int frames);
  void mark_step(int n, int m);
  void mark_complete(int n);
  bool completed(int n) const;
  int last_step(int n) const;
  void wait_complete(int n, std::chrono::milliseconds deadline = std::chrono::minutes(10));
  void poison();
  bool poisoned() const;
  uint64_t next_seq() { return seq_.fetch_add(1); }

 private:
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::vector<int> last_step_;
  std::vector<char> complete_;
  bool poisoned_ = false;
  std::atomic<uint64_t> seq_{0};
};

// Eq. 10 source selection (decomp.cpp:193-209)
int h_choose(int n, int m, int M, const TemporalSchedule& sched, CompletionLedger& ledger);

struct FrameAudit {
  int frame = 0;
  int thread = 0;
  int workers = 1;
  int init_src = -1;
  int reg_final_src = -1;
  std::vector<int> reg_src;
  uint64_t start_seq = 0;
  uint64_t reg_final_seq = 0;
  uint64_t finish_seq = 0;
};

std::string format_audit(const FrameAudit& a);

// ---- autotuner (autotune.hpp:13-77) ----------------------------------------------
enum class ImagingMode : int { single_slice = 0, multi_slice = 1, flow = 2 };
std::string mode_name(ImagingMode m);
ImagingMode mode_from_name(const std::string& s);

int frames_bucket(int frames);
std::string bucket_label(int bucket);
int bucket_from_label(const std::string& s);

struct ProtocolKey {
  ImagingMode mode = ImagingMode::single_slice;
  int N = 0;
  int bucket = 0;
  int J = 0;
  bool operator==(const ProtocolKey& o) const {
    return mode == o.mode && N == o.N && bucket == o.bucket && J == o.J;
  }
  bool operator<(const ProtocolKey& o) const;
};

struct TuningRecord {
  ProtocolKey key;
  int T = 1;
  int A = 1;
  double runtime_ms = 0;
  int64_t timestamp = 0;
};

// (T, A) space, A-major. a_cap = 4 reproduces the reference's 16-entry fixture for
// 8 workers; a_cap = 8 is the NVSwitch space (channel groups up to the whole box).
std::vector<std::pair<int, int>> legal_configs(int total_workers = 8, int a_cap = kGroupSizeMaxCompat);
std::pair<int, int> select_config(const ProtocolKey& key, const std::vector<TuningRecord>& db);
std::pair<int, int> learn_step(const ProtocolKey& key, const std::vector<TuningRecord>& db,
                               int total_workers = 8, int a_cap = kGroupSizeMaxCompat);
std::string format_record(const TuningRecord& r);

class TuneDb {
 public:
  explicit TuneDb(std::string path) : path_(std::move(path)) {}
  const std::string& path() const { return path_; }
  void append(const TuningRecord& r);
  std::vector<TuningRecord> load() const;
  size_t skipped_lines() const { return skipped_; }

 private:
  std::string path_;
  mutable size_t skipped_ = 0;
};

}  // namespace rtnb
