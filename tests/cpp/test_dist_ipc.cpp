// test_dist_ipc.cpp — the n-rank MiCRO step driven from C++ alone, one
// PROCESS per rank, through the C ABI (include/micro.h): CUDA IPC handle
// exchange (micro_peer_export / micro_peer_import), then per iteration
// micro_compress -> barrier -> micro_peer_contribute -> barrier ->
// micro_peer_reduce -> barrier -> micro_peer_finalize.  All ranks share one
// GPU here (IPC allows it); the barriers are host barriers after a stream
// sync, so no kernel ever waits on another process's kernel.
//
// The parent forks the ranks before touching CUDA, then runs the same
// iterations as a single-device cluster context (the reference's in-process
// ClusterState, harness.cpp:121-224) and checks every rank's union, sums,
// counts, thresholds and residual bit for bit.  Also: the NCCL loader
// (micro_nccl_unique_id) and the attach's argument checks.
#include <pthread.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>

#include "micro.h"

namespace {

constexpr int kSteps = 12;
constexpr int64_t kNg = 200003;
constexpr double kEta = 0.01;
constexpr uint64_t kSeed = 11;

struct Shared {
  pthread_barrier_t bar;
  int n;
  int mode;  // 0: peer protocol, host barriers, all ranks on device 0;
             // 1 / 2: micro_dist_init_nccl (MICRO_XCHG_PEER / _NCCL), rank r on device r
  unsigned char uid[MICRO_NCCL_UNIQUE_ID_BYTES];
  int failed;
  unsigned char handles[8][MICRO_PEER_HANDLE_BYTES];
  int64_t K[kSteps][8];
  int64_t counts[kSteps][8];
  double delta[kSteps][8];
  int64_t union_k[8];
  int32_t union_idx[8][kNg];
  float union_sum[8][kNg];
  float residual[8][kNg];
};

int g_fail = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      ++g_fail;                                                        \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
    }                                                                  \
  } while (0)
#define OK(call)                                                                      \
  do {                                                                                \
    const int _rc = (call);                                                           \
    if (_rc != MICRO_OK) {                                                            \
      std::printf("FAIL %s:%d: %s -> %d: %s\n", __FILE__, __LINE__, #call, _rc,       \
                  micro_last_error());                                                \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

micro_config config(int n, int n_local, int rank) {
  micro_config c;
  micro_config_default(&c);
  c.n_g = kNg;
  c.n_workers = n;
  c.n_local = n_local;
  c.rank = rank;
  c.dtype = MICRO_F32;
  c.density = 0.02;
  c.initial_threshold = 0.015;
  c.dense_output = 0;
  return c;
}

int rank_main(Shared* sh, int r) {
  const int n = sh->n;
  const int dev = sh->mode ? r : 0;
  micro_ctx* ctx = nullptr;
  micro_config cfg = config(n, 1, r);
  cfg.device = dev;
  OK(micro_set_device(dev));
  OK(micro_ctx_create(&ctx, &cfg, nullptr));
  if (sh->mode == 0) {
    OK(micro_peer_export(ctx, sh->handles[r]));
    pthread_barrier_wait(&sh->bar);
    OK(micro_peer_import(ctx, sh->handles));
  } else {  // the exchange behind the C ABI: one call per step, no host barriers
    if (r == 0) OK(micro_nccl_unique_id(sh->uid));
    pthread_barrier_wait(&sh->bar);
    OK(micro_dist_init_nccl(ctx, sh->uid, sh->mode == 1 ? MICRO_XCHG_PEER : MICRO_XCHG_NCCL));
  }
  pthread_barrier_wait(&sh->bar);
  void* g = nullptr;
  OK(micro_device_malloc(&g, kNg * 4, dev));
  for (int t = 0; t < kSteps; ++t) {
    OK(micro_synth_gaussian(MICRO_F32, kSeed, (uint32_t)r, (uint64_t)t, kNg, g, nullptr));
    const void* gs[1] = {g};
    if (sh->mode) {
      OK(micro_step(ctx, gs, kEta, t));
    } else {
      OK(micro_compress(ctx, gs, kEta, t));
      OK(micro_sync(ctx));
      pthread_barrier_wait(&sh->bar);  // every rank's K1 done
      OK(micro_peer_contribute(ctx));
      OK(micro_sync(ctx));
      pthread_barrier_wait(&sh->bar);  // every contribution landed
      OK(micro_peer_reduce(ctx));
      OK(micro_sync(ctx));
      pthread_barrier_wait(&sh->bar);  // every owner pushed its segment
      OK(micro_peer_finalize(ctx));
    }
    micro_stats st;
    int64_t k = 0;
    double d = 0;
    OK(micro_query(ctx, &st, &k, &d));
    sh->K[t][r] = st.K;
    sh->counts[t][r] = k;
    sh->delta[t][r] = d;
  }
  int64_t K = 0;
  OK(micro_copy_union(ctx, sh->union_idx[r], sh->union_sum[r], kNg, &K));
  sh->union_k[r] = K;
  OK(micro_copy_residual(ctx, 0, sh->residual[r]));
  pthread_barrier_wait(&sh->bar);  // nobody unmaps a peer's buffers early
  micro_device_free(g);
  OK(micro_ctx_destroy(ctx));
  return 0;
}

void run_check(Shared* sh, int n) {
  micro_ctx* ctx = nullptr;
  const micro_config cfg = config(n, n, 0);
  if (micro_ctx_create(&ctx, &cfg, nullptr) != MICRO_OK) {
    CHECK(!"cluster context");
    return;
  }
  std::vector<void*> g(n);
  for (int i = 0; i < n; ++i) micro_device_malloc(&g[i], kNg * 4, 0);
  std::vector<int64_t> k(n);
  std::vector<double> d(n);
  for (int t = 0; t < kSteps; ++t) {
    for (int i = 0; i < n; ++i) micro_synth_gaussian(MICRO_F32, kSeed, (uint32_t)i, (uint64_t)t, kNg, g[i], nullptr);
    CHECK(micro_step(ctx, g.data(), kEta, t) == MICRO_OK);
    micro_stats st;
    CHECK(micro_query(ctx, &st, k.data(), d.data()) == MICRO_OK);
    for (int r = 0; r < n; ++r) {
      CHECK(sh->K[t][r] == st.K);
      CHECK(sh->counts[t][r] == k[r]);
      CHECK(sh->delta[t][r] == d[r]);
    }
  }
  std::vector<int32_t> idx(kNg);
  std::vector<float> sums(kNg), res(kNg);
  int64_t K = 0;
  CHECK(micro_copy_union(ctx, idx.data(), sums.data(), kNg, &K) == MICRO_OK);
  for (int r = 0; r < n; ++r) {
    CHECK(sh->union_k[r] == K);
    CHECK(std::memcmp(sh->union_idx[r], idx.data(), (size_t)K * 4) == 0);
    CHECK(std::memcmp(sh->union_sum[r], sums.data(), (size_t)K * 4) == 0);
    CHECK(micro_copy_residual(ctx, r, res.data()) == MICRO_OK);
    CHECK(std::memcmp(sh->residual[r], res.data(), (size_t)kNg * 4) == 0);
  }
  std::printf("world %d%s: %d steps, K = %lld at the last, %s vs the single-device cluster\n", n,
              sh->mode == 0 ? "" : sh->mode == 1 ? " (NCCL attach, peer exchange)" : " (NCCL attach, collectives)",
              kSteps, (long long)K, g_fail ? "MISMATCH" : "bit-exact");
  for (int i = 0; i < n; ++i) micro_device_free(g[i]);
  micro_ctx_destroy(ctx);
}

int run_world_mode(int n, int mode) {
  auto* sh = static_cast<Shared*>(
      mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0));
  if (sh == MAP_FAILED) return 1;
  std::memset(sh, 0, sizeof(Shared));
  sh->n = n;
  sh->mode = mode;
  pthread_barrierattr_t at;
  pthread_barrierattr_init(&at);
  pthread_barrierattr_setpshared(&at, PTHREAD_PROCESS_SHARED);
  pthread_barrier_init(&sh->bar, &at, (unsigned)n);
  std::vector<pid_t> kids;
  for (int r = 0; r < n; ++r) {
    const pid_t p = fork();
    if (p == 0) {
      const int rc = rank_main(sh, r);
      std::fflush(stdout);
      _exit(rc);
    }
    kids.push_back(p);
  }
  for (pid_t p : kids) {
    int st = 0;
    waitpid(p, &st, 0);
    CHECK(WIFEXITED(st) && WEXITSTATUS(st) == 0);
  }
  run_check(sh, n);
  pthread_barrier_destroy(&sh->bar);
  munmap(sh, sizeof(Shared));
  return 0;
}

// NCCL behind the C ABI: the loader resolves libnccl, and attach refuses
// contexts that are not one rank of n
int nccl_checks() {
  unsigned char uid[MICRO_NCCL_UNIQUE_ID_BYTES];
  const int rc = micro_nccl_unique_id(uid);
  CHECK(rc == MICRO_OK || rc == MICRO_ENCCL);
  if (rc == MICRO_OK) {
    micro_ctx* ctx = nullptr;
    const micro_config cfg = config(2, 2, 0);
    CHECK(micro_ctx_create(&ctx, &cfg, nullptr) == MICRO_OK);
    CHECK(micro_dist_init_nccl(ctx, uid, MICRO_XCHG_PEER) == MICRO_ELOGIC);  // a cluster, not a rank
    micro_ctx_destroy(ctx);
    const micro_config rc1 = config(2, 1, 1);
    CHECK(micro_ctx_create(&ctx, &rc1, nullptr) == MICRO_OK);
    CHECK(micro_dist_attach_nccl(ctx, nullptr, MICRO_XCHG_NCCL) == MICRO_EINVAL);
    CHECK(micro_aggregate(ctx) == MICRO_ELOGIC);  // no compress, no NCCL
    micro_ctx_destroy(ctx);
  } else {
    std::printf("NCCL unavailable here: %s\n", micro_last_error());
  }
  return 0;
}

// Each case in its own child: a process must not fork ranks after it has
// initialised CUDA, and this one never does.
int run_world(int n) { return run_world_mode(n, 0); }
int run_nccl_peer(int n) { return run_world_mode(n, 1); }
int run_nccl_coll(int n) { return run_world_mode(n, 2); }
int device_count(int) {
  int c = 0;
  micro_device_count(&c);
  return c;
}

int in_child(int (*f)(int), int arg) {
  const pid_t p = fork();
  if (p == 0) {
    f(arg);
    std::fflush(stdout);  // _exit skips stdio's buffers
    _exit(g_fail ? 1 : 0);
  }
  int st = 0;
  waitpid(p, &st, 0);
  return WIFEXITED(st) ? WEXITSTATUS(st) : 1;
}

}  // namespace

int main() {
  int bad = 0;
  bad += in_child(run_world, 2);
  bad += in_child(run_world, 3);
  bad += in_child([](int) { return nccl_checks(); }, 0);
  // one rank per GPU through micro_dist_init_nccl + micro_step (needs 2 GPUs;
  // NCCL does not put two ranks on one device)
  const pid_t p = fork();
  if (p == 0) _exit(std::min(device_count(0), 100));
  int st = 0;
  waitpid(p, &st, 0);
  const int ndev = WIFEXITED(st) ? WEXITSTATUS(st) : 0;
  if (ndev >= 2) {
    bad += in_child(run_nccl_peer, 2);
    bad += in_child(run_nccl_coll, 2);
  } else {
    std::printf("NCCL worlds skipped: %d GPU(s) visible\n", ndev);
  }
  std::printf("%s: %d failing cases\n", bad ? "FAIL" : "OK", bad);
  return bad;
}
