// Small persistent worker pool for host-side copies (pinned staging ->
// caller buffers). parallel_for runs f(0..parts-1) on the workers and the
// calling thread and returns when all parts are done.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace svlfb {

class HostPool {
  public:
    explicit HostPool(int workers) {
        for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    int size() const { return int(threads_.size()) + 1; }

    void parallel_for(int parts, const std::function<void(int)>& f) {
        if (parts <= 0) return;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &f;
            parts_ = parts;
            next_.store(0);
            pending_ = parts;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    void work() {
        for (;;) {
            const int i = next_.fetch_add(1);
            if (i >= parts_) return;
            (*job_)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    void loop() {
        unsigned seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ != nullptr); });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    int parts_ = 0, pending_ = 0;
    std::atomic<int> next_{0};
    unsigned gen_ = 0;
    bool stop_ = false;
};

}  // namespace svlfb
