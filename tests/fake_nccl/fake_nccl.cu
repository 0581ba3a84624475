// An in-process stand-in for the five NCCL entry points the sharded steps use (ncclAllGather, ncclGroupStart /
// ncclGroupEnd, ncclCommCount, ncclCommUserRank, + ncclGetErrorString / ncclCommGetAsyncError), so the library's
// tetris_dist_* entry points can run at world sizes > 1 on ONE GPU: every "rank" is a host thread of one process
// with its own stream and buffers, and an all-gather is a rendezvous of the W threads followed by device-to-device
// copies of every rank's send buffer into every rank's receive buffer, ordered after each sender's stream work and
// before each receiver's later work with events.  TEST INFRASTRUCTURE ONLY (tests/test_dist_fake_nccl.py loads it via
// $TETRIS_NCCL_LIB); it emulates the collective's semantics, not NCCL's transport.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

namespace {

struct Op {
  const void* send;
  void* recv;
  size_t bytes;
};

struct World {
  int size = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const void*> send;
  std::vector<cudaEvent_t> ready, done;
};

struct Comm {
  World* world;
  int rank;
};

thread_local int t_group_depth = 0;
thread_local std::vector<Op> t_pending;
thread_local void* t_comm = nullptr;
thread_local cudaStream_t t_stream = nullptr;

// all ranks of the world reach this point (a generation barrier)
void rendezvous(World& w) {
  std::unique_lock<std::mutex> lk(w.m);
  const long long gen = w.generation;
  if (++w.arrived == w.size) {
    w.arrived = 0;
    ++w.generation;
    w.cv.notify_all();
  } else {
    w.cv.wait(lk, [&] { return w.generation != gen; });
  }
}

int all_gather_now(const Op& op, Comm* c, cudaStream_t st) {
  World& w = *c->world;
  const int r = c->rank;
  w.send[r] = op.send;
  cudaEventRecord(w.ready[r], st);  // the sender's data is complete after its stream's prior work
  rendezvous(w);                     // every rank's send pointer and ready event are in place
  for (int p = 0; p < w.size; ++p) {
    cudaStreamWaitEvent(st, w.ready[p], 0);
    cudaMemcpyAsync(static_cast<char*>(op.recv) + (size_t)p * op.bytes, w.send[p], op.bytes,
                    cudaMemcpyDeviceToDevice, st);
  }
  cudaEventRecord(w.done[r], st);
  rendezvous(w);  // every rank has queued its reads of the others' send buffers
  for (int p = 0; p < w.size; ++p) cudaStreamWaitEvent(st, w.done[p], 0);  // no sender overwrites before the reads
  rendezvous(w);  // the events may be re-recorded by the next collective
  return 0;
}

}  // namespace

extern "C" {

// test helpers: a world of `size` ranks, and rank r's communicator in it
void* fake_nccl_world_create(int size) {
  World* w = new World();
  w->size = size;
  w->send.assign(size, nullptr);
  w->ready.resize(size);
  w->done.resize(size);
  for (int i = 0; i < size; ++i) {
    cudaEventCreateWithFlags(&w->ready[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->done[i], cudaEventDisableTiming);
  }
  return w;
}
void* fake_nccl_comm_create(void* world, int rank) { return new Comm{static_cast<World*>(world), rank}; }

int ncclCommCount(const void* comm, int* count) {
  *count = static_cast<const Comm*>(comm)->world->size;
  return 0;
}
int ncclCommUserRank(const void* comm, int* rank) {
  *rank = static_cast<const Comm*>(comm)->rank;
  return 0;
}
int ncclGroupStart(void) {
  ++t_group_depth;
  return 0;
}
int ncclAllGather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t stream) {
  if (dtype != 0 && dtype != 1) return 4;  // the library sends bytes (ncclInt8)
  const Op op{send, recv, count};
  if (t_group_depth > 0) {
    t_pending.push_back(op);
    t_comm = comm;
    t_stream = stream;
    return 0;
  }
  return all_gather_now(op, static_cast<Comm*>(comm), stream);
}
int ncclGroupEnd(void) {
  if (--t_group_depth > 0) return 0;
  int rc = 0;
  for (const Op& op : t_pending) rc |= all_gather_now(op, static_cast<Comm*>(t_comm), t_stream);
  t_pending.clear();
  return rc;
}
const char* ncclGetErrorString(int) { return "fake NCCL error"; }
int ncclCommGetAsyncError(void*, int* state) {
  *state = 0;
  return 0;
}

}  // extern "C"
