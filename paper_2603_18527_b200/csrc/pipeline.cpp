// pipeline.cpp -- overlapped batch solves over several problem handles (bp_pipeline_*).
//
// The reference's callers solve one batch at a time and wait for it (run_sweep,
// proj/src/bench.cpp:143-151; cmd_solve, proj/tools/bornprec_main.cpp:132).  On a GPU that
// serialises the PCIe copies of a solve (media + sources in, iterates out) with the sweeps.
// A pipeline owns `depth` handles of one shape, each driven by its own host worker thread on the
// handle's own non-blocking stream: while slot s sweeps, slot s+1 uploads the next batch and the
// previous slot downloads its result, so in steady state the copy engines run under the sweeps.
// Every job is exactly bp_problem_set_medium / bp_problem_set_cdr_medium + bp_run on its slot;
// results are bit-identical to calling those two entry points directly.  The sweeps themselves
// take FIFO turns (a ticket per job, handed over through compute hooks the run calls after its
// uploads were enqueued and before its downloads), so only the copies overlap: two solves never
// share the SMs, and the pipeline's throughput is the single-handle sweep rate minus the copy
// time it could not hide.
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bornsweep.h"

// defined in bornsweep.cu: sets the calling thread's bp_last_error() message; installs the
// hooks a run calls around its sweeps
extern "C" int bp_internal_set_error(int code, const char* msg);
extern "C" int bp_internal_set_compute_hooks(bp_problem* p, void (*pre)(void*), void (*post)(void*),
                                             void* ctx);

namespace {

struct Job {
    bp_medium medium;  // all-null: keep the slot's current medium
    bp_map map;
    bp_iter_config cfg;
    const double* f;
    const double* u0;
    double* u_out;
    double* res_l2;
    double* res_reta;
    bp_trace* info;
    int64_t ticket;  // submission order = compute order
};

struct Slot {
    bp_problem* p = nullptr;
    std::thread worker;
    std::deque<Job> queue;
    // compute-turn state of the slot's running job (guarded by bp_pipeline::m)
    bp_pipeline* pl = nullptr;
    int64_t ticket = -1;
    bool turn_done = false;
};

}  // namespace

struct bp_pipeline {
    std::vector<Slot> slots;
    std::mutex m;
    std::condition_variable cv_work, cv_done;
    bool stop = false;
    int64_t pending = 0;  // submitted and not finished
    int next = 0;
    int64_t next_ticket = 0;   // assigned at submit
    int64_t compute_turn = 0;  // ticket whose sweeps may run now
    std::condition_variable cv_turn;
    int err_code = BP_OK;
    std::string err_msg;
};

namespace {

// The slot whose worker runs on this thread.  The compute hooks act only there: a direct
// bp_run / bp_run_device on a slot handle from any other thread (while the pipeline exists)
// runs without taking a turn instead of waiting for a ticket that is not its own.
thread_local const Slot* tl_worker_slot = nullptr;

void turn_acquire(void* ctx) {
    auto* sl = static_cast<Slot*>(ctx);
    if (tl_worker_slot != sl) return;
    std::unique_lock<std::mutex> lk(sl->pl->m);
    sl->pl->cv_turn.wait(lk, [&] { return sl->pl->compute_turn == sl->ticket; });
}

void turn_release(void* ctx) {
    auto* sl = static_cast<Slot*>(ctx);
    if (tl_worker_slot != sl) return;
    {
        std::lock_guard<std::mutex> lk(sl->pl->m);
        ++sl->pl->compute_turn;
        sl->turn_done = true;
    }
    sl->pl->cv_turn.notify_all();
}

int run_job(bp_problem* p, const Job& j) {
    const bp_medium& md = j.medium;
    if (md.k2) {
        if (int rc = bp_problem_set_medium(p, md.k2, md.k0, md.eta)) return rc;
    } else if (md.bx) {
        if (int rc = bp_problem_set_cdr_medium(p, md.bx, md.by, md.sigma, md.sigma0)) return rc;
    }
    return bp_run(p, &j.map, j.f, &j.cfg, j.u0, j.u_out, j.res_l2, j.res_reta, j.info);
}

void worker_loop(bp_pipeline* pl, int s) {
    tl_worker_slot = &pl->slots[s];
    for (;;) {
        Job job;
        {
            std::unique_lock<std::mutex> lk(pl->m);
            pl->cv_work.wait(lk, [&] { return pl->stop || !pl->slots[s].queue.empty(); });
            if (pl->slots[s].queue.empty()) return;  // stop requested and nothing left
            job = pl->slots[s].queue.front();
            pl->slots[s].ticket = job.ticket;
            pl->slots[s].turn_done = false;
        }
        const int rc = run_job(pl->slots[s].p, job);
        if (!pl->slots[s].turn_done) {  // failed before its sweeps: pass the turn on in order
            turn_acquire(&pl->slots[s]);
            turn_release(&pl->slots[s]);
        }
        const std::string msg = rc ? std::string(bp_last_error()) : std::string();
        {
            std::lock_guard<std::mutex> lk(pl->m);
            pl->slots[s].queue.pop_front();
            if (rc && pl->err_code == BP_OK) {
                pl->err_code = rc;
                pl->err_msg = "pipeline slot " + std::to_string(s) + ": " + msg;
            }
            --pl->pending;
        }
        pl->cv_done.notify_all();
    }
}

}  // namespace

extern "C" {

int bp_pipeline_create(bp_problem* const* slots, int32_t depth, bp_pipeline** out) {
    if (!out || !slots || depth < 1) return bp_internal_set_error(BP_EINVAL, "pipeline: null argument or depth < 1");
    *out = nullptr;
    for (int s = 0; s < depth; ++s)
        if (!slots[s]) return bp_internal_set_error(BP_EINVAL, "pipeline: null slot handle");
    for (int s = 0; s < depth; ++s)
        for (int r = 0; r < s; ++r)
            if (slots[r] == slots[s])  // one worker thread per handle
                return bp_internal_set_error(BP_EINVAL, "pipeline: the same handle in two slots");
    auto* pl = new bp_pipeline;
    pl->slots.resize(depth);
    for (int s = 0; s < depth; ++s) {
        pl->slots[s].p = slots[s];
        pl->slots[s].pl = pl;
    }
    for (int s = 0; s < depth; ++s) {
        if (int rc = bp_internal_set_compute_hooks(slots[s], turn_acquire, turn_release, &pl->slots[s])) {
            for (int r = 0; r < s; ++r) bp_internal_set_compute_hooks(slots[r], nullptr, nullptr, nullptr);
            delete pl;
            return rc;
        }
    }
    for (int s = 0; s < depth; ++s) pl->slots[s].worker = std::thread(worker_loop, pl, s);
    *out = pl;
    return BP_OK;
}

int bp_pipeline_submit(bp_pipeline* pl, const bp_medium* medium, const bp_map* map, const double* f,
                       const bp_iter_config* cfg, const double* u0, double* u_out, double* res_l2,
                       double* res_reta, bp_trace* info, int32_t* slot_out) {
    if (!pl || !map || !f || !cfg || !u_out || !info)
        return bp_internal_set_error(BP_EINVAL, "pipeline submit: null argument");
    Job j{};
    if (medium) j.medium = *medium;
    j.map = *map;
    j.cfg = *cfg;
    j.f = f;
    j.u0 = u0;
    j.u_out = u_out;
    j.res_l2 = res_l2;
    j.res_reta = res_reta;
    j.info = info;
    int s;
    {
        std::lock_guard<std::mutex> lk(pl->m);
        s = pl->next;
        pl->next = (pl->next + 1) % (int)pl->slots.size();
        j.ticket = pl->next_ticket++;
        pl->slots[s].queue.push_back(j);
        ++pl->pending;
    }
    pl->cv_work.notify_all();
    if (slot_out) *slot_out = s;
    return BP_OK;
}

int bp_pipeline_wait(bp_pipeline* pl) {
    if (!pl) return bp_internal_set_error(BP_EINVAL, "pipeline: null handle");
    std::unique_lock<std::mutex> lk(pl->m);
    pl->cv_done.wait(lk, [&] { return pl->pending == 0; });
    const int rc = pl->err_code;
    pl->err_code = BP_OK;
    return rc ? bp_internal_set_error(rc, pl->err_msg.c_str()) : BP_OK;
}

int bp_pipeline_destroy(bp_pipeline* pl) {
    if (!pl) return BP_OK;
    {
        std::lock_guard<std::mutex> lk(pl->m);
        pl->stop = true;
    }
    pl->cv_work.notify_all();
    for (auto& s : pl->slots)
        if (s.worker.joinable()) s.worker.join();
    for (auto& s : pl->slots) bp_internal_set_compute_hooks(s.p, nullptr, nullptr, nullptr);
    delete pl;
    return BP_OK;
}

}  // extern "C"
