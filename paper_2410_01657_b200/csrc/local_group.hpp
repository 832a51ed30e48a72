// In-process rank group: R engine contexts driven by R host threads of ONE
// process (on one GPU or several), the B200 counterpart of the reference's
// RankRuntime / RankComm (comm.cpp:35-93, 168-208). Collectives rendezvous on
// the host with the reference's matching rule — every rank must post the same
// (kind, mode) in the same order, otherwise the group is poisoned and every
// rank raises CollectiveError — plus a timeout, so a rank that never arrives
// fails its peers instead of hanging them. The data moves on the device:
// device-to-device copies ordered by CUDA events (no kernel ever waits on
// another rank's kernel).
#pragma once

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

struct hgnn_ctx;

namespace hgnn_b200 {

// Collective kinds (CollectiveKind of comm.hpp plus the engine's phases).
enum : int32_t { kCollHaloFwd = 1, kCollHaloAdj = 2, kCollAllReduce = 3, kCollDone = 4 };

struct CollSig {
  int32_t kind = 0, mode = 0;
  int64_t count = 0;  // elements (all-reduce) or row width (exchange)
  bool operator==(const CollSig& o) const { return kind == o.kind && mode == o.mode && count == o.count; }
};

inline std::string sig_str(const CollSig& s) {
  static const char* names[] = {"?", "halo_exchange", "halo_exchange_adjoint", "all_reduce_sum", "exchange_done"};
  return std::string(names[(s.kind >= 0 && s.kind <= 4) ? s.kind : 0]) + "(mode " + std::to_string(s.mode) +
         ", n " + std::to_string(s.count) + ")";
}

class LocalGroup {
 public:
  explicit LocalGroup(int32_t n) : R(n), ctx((size_t)n, nullptr), host((size_t)n, nullptr), retired((size_t)n, 0) {}

  const int32_t R;
  std::vector<hgnn_ctx*> ctx;             // registered contexts by rank
  std::vector<std::vector<double>*> host;  // all-reduce payloads (host copies)
  int64_t timeout_ms = 120000;

  void attach(int32_t rank, hgnn_ctx* c) {
    std::lock_guard<std::mutex> lk(mu_);
    if (ctx[(size_t)rank]) fail(HGNN_ERR_CONFIG, "local group: rank " + std::to_string(rank) + " already attached");
    ctx[(size_t)rank] = c;
  }
  // A rank that leaves (context destroyed) can no longer meet its peers.
  void retire(int32_t rank) {
    std::lock_guard<std::mutex> lk(mu_);
    ctx[(size_t)rank] = nullptr;
    retired[(size_t)rank] = 1;
    if (active_) poison_locked("rank " + std::to_string(rank) + " left the group during a collective");
  }
  // Failure inside a rank between the phases of a collective: peers must not wait for it.
  void abort(const std::string& why) {
    std::lock_guard<std::mutex> lk(mu_);
    poison_locked(why);
  }

  // Rendezvous: returns once all R ranks posted `sig`; `combine` runs once, in
  // the last arriving thread, under the lock (comm.cpp:168-208).
  template <class F>
  void collective(int32_t rank, const CollSig& sig, F&& combine, std::vector<double>* payload = nullptr) {
    std::unique_lock<std::mutex> lk(mu_);
    if (poisoned_) fail(HGNN_ERR_COLLECTIVE, "collective aborted: " + msg_);
    for (int32_t r = 0; r < R; ++r)
      if (retired[(size_t)r]) {
        poison_locked("rank " + std::to_string(rank) + " entered " + sig_str(sig) + " after rank " +
                      std::to_string(r) + " left the group (mismatched collective sequences)");
        fail(HGNN_ERR_COLLECTIVE, "collective aborted: " + msg_);
      }
    if (!active_) {
      active_ = true;
      pending_ = sig;
      arrived_ = 0;
    } else if (!(pending_ == sig)) {
      poison_locked("mismatched collective sequence: rank " + std::to_string(rank) + " posted " + sig_str(sig) +
                    " while its peers posted " + sig_str(pending_));
      fail(HGNN_ERR_COLLECTIVE, "collective aborted: " + msg_);
    }
    host[(size_t)rank] = payload;
    arrived_ += 1;
    if (arrived_ == R) {
      try {
        combine();
      } catch (const std::exception& e) {
        active_ = false;
        poison_locked(e.what());
        fail(HGNN_ERR_COLLECTIVE, "collective aborted: " + msg_);
      }
      active_ = false;
      generation_ += 1;
      cv_.notify_all();
      return;
    }
    const uint64_t gen = generation_;
    const bool ok = cv_.wait_for(lk, std::chrono::milliseconds(timeout_ms),
                                 [&] { return generation_ > gen || poisoned_; });
    if (!ok) {
      poison_locked("timeout: not every rank entered " + sig_str(sig) + " within " + std::to_string(timeout_ms) +
                    " ms");
      fail(HGNN_ERR_COLLECTIVE, "collective aborted: " + msg_);
    }
    if (generation_ == gen && poisoned_) fail(HGNN_ERR_COLLECTIVE, "collective aborted: " + msg_);
  }
  void barrier(int32_t rank, const CollSig& sig) {
    collective(rank, sig, [] {});
  }
  // all_reduce_sum (comm.cpp:99-126 TensorSum): element-wise sum over ranks in
  // rank order (the same fp64 result on every rank), in place.
  void allreduce_sum(int32_t rank, std::vector<double>& v) {
    CollSig sig{kCollAllReduce, 0, (int64_t)v.size()};
    collective(
        rank, sig,
        [&] {
          std::vector<double> sum(*host[0]);
          for (int32_t r = 1; r < R; ++r)
            for (size_t i = 0; i < sum.size(); ++i) sum[i] += (*host[(size_t)r])[i];
          for (int32_t r = 0; r < R; ++r) *host[(size_t)r] = sum;
        },
        &v);
  }

 private:
  void poison_locked(const std::string& m) {
    if (!poisoned_) {
      poisoned_ = true;
      msg_ = m;
    }
    cv_.notify_all();
  }
  std::mutex mu_;
  std::condition_variable cv_;
  bool active_ = false, poisoned_ = false;
  CollSig pending_;
  int32_t arrived_ = 0;
  uint64_t generation_ = 0;
  std::string msg_;
  std::vector<uint8_t> retired;
};

}  // namespace hgnn_b200
