// Host scheduling logic; semantics pinned to the reference by tests/test_sched.py.
#include "sched.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <set>
#include <sstream>
#include <tuple>

#include "engine.hpp"

namespace rtnb {

std::vector<std::pair<int, int>> partition_channels(int J, int A, int cap) {
  // decomp.cpp:10-24: A in [1, cap] and A <= J, else a usage error
  if (A < 1 || A > cap || A > J) fail(2, "partition_channels: worker count out of range");
  std::vector<std::pair<int, int>> out(static_cast<size_t>(A));
  const int q = J / A, extra = J % A;
  int at = 0;
  for (int a = 0; a < A; ++a) {
    const int len = q + (a < extra ? 1 : 0);
    out[static_cast<size_t>(a)] = {at, at + len};
    at += len;
  }
  return out;
}

// ---- ledger ------------------------------------------------------------------------

CompletionLedger::CompletionLedger(int frames)
    : last_step_(static_cast<size_t>(std::max(frames, 0)), -1),
      complete_(static_cast<size_t>(std::max(frames, 0)), 0) {}

void CompletionLedger::mark_step(int n, int m) {
  std::lock_guard<std::mutex> g(mu_);
  int& s = last_step_.at(static_cast<size_t>(n));
  if (m < s) fail(2, "CompletionLedger: step progress must be monotone");
  s = m;
}

void CompletionLedger::mark_complete(int n) {
  {
    std::lock_guard<std::mutex> g(mu_);
    complete_.at(static_cast<size_t>(n)) = 1;
  }
  cv_.notify_all();
}

bool CompletionLedger::completed(int n) const {
  std::lock_guard<std::mutex> g(mu_);
  if (n < 0 || n >= static_cast<int>(complete_.size())) return false;
  return complete_[static_cast<size_t>(n)] != 0;
}

int CompletionLedger::last_step(int n) const {
  std::lock_guard<std::mutex> g(mu_);
  return last_step_.at(static_cast<size_t>(n));
}

void CompletionLedger::wait_complete(int n, std::chrono::milliseconds deadline) {
  std::unique_lock<std::mutex> g(mu_);
  const size_t idx = static_cast<size_t>(n);
  if (idx >= complete_.size()) fail(2, "CompletionLedger: frame index out of range");
  const bool ready = cv_.wait_for(g, deadline, [&] { return poisoned_ || complete_[idx] != 0; });
  if (poisoned_) fail_decomp("series aborted by an earlier fault");
  if (!ready) fail_decomp("timed out waiting for a predecessor frame");
}

void CompletionLedger::poison() {
  {
    std::lock_guard<std::mutex> g(mu_);
    poisoned_ = true;
  }
  cv_.notify_all();
}

bool CompletionLedger::poisoned() const {
  std::lock_guard<std::mutex> g(mu_);
  return poisoned_;
}

int h_choose(int n, int m, int M, const TemporalSchedule& sched, CompletionLedger& ledger) {
  if (n < 1) fail(2, "h_choose: defined for n >= 1 only");
  const bool pinned = (n <= sched.l) || (m == M - 1);
  if (pinned) {
    ledger.wait_complete(n - 1);
    return n - 1;
  }
  const int oldest = std::max(n - sched.o, 0);
  for (int w = n - 1; w >= oldest; --w) {
    if (ledger.completed(w)) return w;
  }
  ledger.wait_complete(oldest);
  return oldest;
}

std::string format_audit(const FrameAudit& a) {
  std::ostringstream os;
  os << "frame " << a.frame << ": init<-" << a.init_src << ", reg_final<-" << a.reg_final_src << ", thread "
     << a.thread << ", workers " << a.workers;
  return os.str();
}

// ---- autotune -------------------------------------------------------------------------

namespace {
constexpr int kCaps[5] = {5, 10, 25, 50, 200};
}

std::string mode_name(ImagingMode m) {
  switch (m) {
    case ImagingMode::single_slice:
      return "single_slice";
    case ImagingMode::multi_slice:
      return "multi_slice";
    case ImagingMode::flow:
      return "flow";
  }
  fail(3, "unknown imaging mode");
}

ImagingMode mode_from_name(const std::string& s) {
  for (ImagingMode m : {ImagingMode::single_slice, ImagingMode::multi_slice, ImagingMode::flow}) {
    if (mode_name(m) == s) return m;
  }
  fail(3, "unknown imaging mode '" + s + "'");
}

int frames_bucket(int frames) {
  if (frames < 1) fail(2, "frames_bucket: frame count must be >= 1");
  int b = 0;
  while (b < 5 && frames > kCaps[b]) ++b;
  return b;
}

std::string bucket_label(int bucket) {
  if (bucket < 0 || bucket > 5) fail(2, "bucket_label: bucket out of range");
  return bucket == 5 ? std::string("inf") : std::to_string(kCaps[bucket]);
}

int bucket_from_label(const std::string& s) {
  for (int b = 0; b <= 5; ++b) {
    if (bucket_label(b) == s) return b;
  }
  fail(3, "unknown frames bucket '" + s + "'");
}

bool ProtocolKey::operator<(const ProtocolKey& o) const {
  return std::make_tuple(static_cast<int>(mode), N, bucket, J) <
         std::make_tuple(static_cast<int>(o.mode), o.N, o.bucket, o.J);
}

std::vector<std::pair<int, int>> legal_configs(int total, int a_cap) {
  if (total < 1) fail(2, "legal_configs: need at least one worker");
  std::vector<std::pair<int, int>> v;
  const int amax = std::min(a_cap, total);
  for (int A = 1; A <= amax; ++A) {
    for (int T = 1; T * A <= total; ++T) v.push_back({T, A});
  }
  return v;
}

std::pair<int, int> select_config(const ProtocolKey& key, const std::vector<TuningRecord>& db) {
  // nearest recorded key of the same mode under (|dN|, |dbucket|, |dJ|, key order)
  auto dist = [&key](const ProtocolKey& k) {
    return std::make_tuple(std::abs(k.N - key.N), std::abs(k.bucket - key.bucket), std::abs(k.J - key.J),
                           static_cast<int>(k.mode), k.N, k.bucket, k.J);
  };
  const ProtocolKey* near = nullptr;
  for (const TuningRecord& r : db) {
    if (r.key.mode != key.mode) continue;
    if (!near || dist(r.key) < dist(*near)) near = &r.key;
  }
  if (!near) return {1, 1};
  const ProtocolKey chosen = *near;
  const TuningRecord* best = nullptr;
  for (const TuningRecord& r : db) {
    if (!(r.key == chosen)) continue;
    const bool better = !best || r.runtime_ms < best->runtime_ms ||
                        (r.runtime_ms == best->runtime_ms && std::make_pair(r.A, r.T) < std::make_pair(best->A, best->T));
    if (better) best = &r;
  }
  return {best->T, best->A};
}

std::pair<int, int> learn_step(const ProtocolKey& key, const std::vector<TuningRecord>& db, int total,
                               int a_cap) {
  std::set<std::pair<int, int>> tried;
  for (const TuningRecord& r : db) {
    if (r.key == key) tried.insert({r.T, r.A});
  }
  for (const auto& c : legal_configs(total, a_cap)) {
    if (!tried.count(c)) return c;
  }
  return select_config(key, db);
}

std::string format_record(const TuningRecord& r) {
  char ms[64];
  std::snprintf(ms, sizeof(ms), "%.3f", r.runtime_ms);
  std::ostringstream os;
  os << mode_name(r.key.mode) << '\t' << r.key.N << '\t' << bucket_label(r.key.bucket) << '\t' << r.key.J << '\t'
     << r.T << '\t' << r.A << '\t' << ms << '\t' << r.timestamp;
  return os.str();
}

void TuneDb::append(const TuningRecord& r) {
  // a crashed writer may have left an unterminated line: terminate it first so the
  // fragment cannot swallow this record (load() skips it)
  bool torn = false;
  std::error_code ec;
  const auto sz = std::filesystem::file_size(path_, ec);
  if (!ec && sz > 0) {
    std::ifstream in(path_, std::ios::binary);
    in.seekg(-1, std::ios::end);
    char c = '\n';
    in.read(&c, 1);
    torn = in.gcount() == 1 && c != '\n';
  }
  std::ofstream out(path_, std::ios::app);
  if (!out) fail(3, path_ + ": cannot open for append");
  if (torn) out << '\n';
  out << format_record(r) << '\n';
  out.flush();
  if (!out) fail(3, path_ + ": append failed");
}

std::vector<TuningRecord> TuneDb::load() const {
  skipped_ = 0;
  std::vector<TuningRecord> v;
  std::ifstream in(path_);
  if (!in) return v;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string mode, bucket;
    TuningRecord r;
    if (!(ls >> mode >> r.key.N >> bucket >> r.key.J >> r.T >> r.A >> r.runtime_ms >> r.timestamp)) {
      ++skipped_;
      continue;
    }
    try {
      r.key.mode = mode_from_name(mode);
      r.key.bucket = bucket_from_label(bucket);
    } catch (const Error&) {
      ++skipped_;
      continue;
    }
    if (r.T < 1 || r.A < 1 || !(r.runtime_ms > 0)) {
      ++skipped_;
      continue;
    }
    v.push_back(r);
  }
  return v;
}

}  // namespace rtnb
