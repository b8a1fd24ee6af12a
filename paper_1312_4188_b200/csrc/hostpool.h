// hostpool.h -- a persistent pool of host threads for the e2e path's staging
// copies (pageable caller buffers <-> the handle's pinned ring).  One job at a
// time (callers serialise on submit_mu); the calling thread works too, so a
// job of k parts runs on up to threads()+1 cores.  Included by pfw.cu.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

class HostPool {
   public:
    static HostPool &get() {
        static HostPool pool;
        return pool;
    }
    int threads() const { return (int)workers_.size(); }

    // Run f(0) .. f(parts-1) across the pool and the calling thread; returns
    // when every part has finished.
    void run(int parts, const std::function<void(int)> &f) {
        if (parts <= 0) return;
        std::lock_guard<std::mutex> submit(submit_mu_);
        Job job{&f, parts};
        {
            std::lock_guard<std::mutex> l(mu_);
            cur_ = &job;
            gen_++;
        }
        cv_.notify_all();
        work(job);
        std::unique_lock<std::mutex> l(mu_);
        done_cv_.wait(l, [&] { return job.finished.load() == parts && job.active == 0; });
        cur_ = nullptr;
    }

    // memcpy of `bytes` split into cache-friendly pieces across the pool
    void copy(void *dst, const void *src, size_t bytes) {
        constexpr size_t PIECE = 4u << 20;
        const int parts = (int)std::min<size_t>((bytes + PIECE - 1) / PIECE, (size_t)threads() + 1);
        if (parts <= 1) {
            if (bytes) memcpy(dst, src, bytes);
            return;
        }
        const size_t per = ((bytes / parts) + 63) & ~size_t(63);
        run(parts, [&](int i) {
            const size_t a = std::min(bytes, (size_t)i * per), b = std::min(bytes, a + per);
            if (b > a) memcpy(static_cast<char *>(dst) + a, static_cast<const char *>(src) + a, b - a);
        });
    }

    // several copies as ONE job: every copy cut into pieces of at most ~2 MB,
    // all pieces spread over the pool (one wake-up per batch of columns)
    struct Copy {
        void *dst;
        const void *src;
        size_t bytes;
    };
    void copy_many(const Copy *c, int nc) {
        constexpr size_t PIECE = 2u << 20;
        size_t total = 0;
        for (int i = 0; i < nc; i++) total += c[i].bytes;
        if (total == 0) return;
        std::vector<Copy> pieces;
        for (int i = 0; i < nc; i++)
            for (size_t a = 0; a < c[i].bytes; a += PIECE)
                pieces.push_back(Copy{static_cast<char *>(c[i].dst) + a, static_cast<const char *>(c[i].src) + a,
                                      std::min(PIECE, c[i].bytes - a)});
        if (pieces.size() == 1 || threads() == 0) {
            for (const Copy &p : pieces) memcpy(p.dst, p.src, p.bytes);
            return;
        }
        run((int)pieces.size(), [&](int i) { memcpy(pieces[(size_t)i].dst, pieces[(size_t)i].src, pieces[(size_t)i].bytes); });
    }

    ~HostPool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }

   private:
    struct Job {
        const std::function<void(int)> *f;
        int parts;
        std::atomic<int> next{0};
        std::atomic<int> finished{0};
        int active = 0;  // workers inside work() for this job (guarded by mu_)
    };

    HostPool() {
        unsigned hc = std::thread::hardware_concurrency();
        int n = (int)std::min(hc ? hc : 4u, 16u) - 1;
        for (int i = 0; i < n; i++) workers_.emplace_back([this] { loop(); });
    }

    void work(Job &j) {
        for (int i; (i = j.next.fetch_add(1)) < j.parts;) {
            (*j.f)(i);
            if (j.finished.fetch_add(1) + 1 == j.parts) {
                std::lock_guard<std::mutex> l(mu_);
                done_cv_.notify_all();
            }
        }
    }

    void loop() {
        uint64_t seen = 0;
        for (;;) {
            Job *j;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || (cur_ && gen_ != seen); });
                if (stop_) return;
                seen = gen_;
                j = cur_;
                j->active++;
            }
            work(*j);
            std::lock_guard<std::mutex> l(mu_);
            j->active--;
            done_cv_.notify_all();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex mu_, submit_mu_;
    std::condition_variable cv_, done_cv_;
    Job *cur_ = nullptr;
    uint64_t gen_ = 0;
    bool stop_ = false;
};
