// pv_fifo.cu — K4: exact replay of the per-process FIFO translation cache.
//
// The reference's TranslationCache (memvirt.py:336-374) is a per-process
// FIFO of (gva page, hpa page): capacity 10, linear lookup, insert only on a
// miss that resolved, oldest-first eviction independent of hits, hit / miss
// counters.  ProcessTranslator.translate (memvirt.py:585-594) consults it
// before walking.  Results may differ from a fresh walk when an entry is
// stale (tables edited without flush_page, e.g. backend.py:164-174 or the
// trap shim backend.py:288-296), and the counters are pinned metrics
// (harness.py:180-184), so the replay must be exact and order-preserving --
// an inherently sequential automaton.  It is parallelised here in three
// exact steps over 32-lookup windows of each process's lookup stream:
//
//  1. speculate (one warp per window, all windows in parallel): rebuild the
//     window's start state by replaying the H previous windows from an empty
//     cache (or exactly from the initial cache near the stream start), then
//     replay the window; record start state S'w, end state E'w, per-lookup
//     hit/terminate flags and hit values;
//  2. link (one thread per window): match[w] = (E'w-1 == S'w);
//  3. verify (one warp per process, sequential over windows): a window whose
//     predecessor was accepted and whose match flag is set is accepted as
//     is (the common case costs one flag read); otherwise the window's true
//     start state is compared with S'w and, if different, the window is
//     replayed again from the true state;
//  4. apply (one thread per lookup): hits overwrite value/status, op
//     terminations set op_first_bad.
//
// Replaying one window is itself warp-parallel: lane j holds lookup j, the
// cache state lives in lanes (lane i = i-th oldest entry), and hit / insert /
// terminate masks are found by a fixed-point iteration (lookup j only
// depends on lookups < j, so the iteration is exact after at most 32 rounds
// and typically converges in two or three): membership in the start state
// (shifted by the insertions before j), membership among earlier window
// insertions (__match_any_sync on the key; an insertion i is still cached at
// j if fewer than `capacity` insertions happened in between), and, for copy
// plans, op termination (a miss whose walk failed, or a data access out of
// range) deactivating the op's later pages (memvirt.py:615-627).
#include "pv_common.cuh"

namespace pv {

constexpr uint32_t kNoOp = 0xFFFFFFFFu;
#ifndef PV_FIFO_WARM
#define PV_FIFO_WARM 1
#endif
constexpr int kWarmWindows = PV_FIFO_WARM;  // H

struct FifoStream {
  const uint64_t* ref;       // per lookup: index into value / status (lane or page)
  const uint32_t* op;        // per lookup: op id (copy plans) or nullptr (lanes)
  const uint64_t* lk_off;    // [n_procs + 1] lookup offsets per process
  const uint64_t* win_off;   // [n_procs + 1] global window offsets per process
  uint32_t n_procs;
  const void* vas;           // lanes: key = vas[ref] >> 12
  uint32_t va32;
  const pv_op* ops;          // copy plans: key = page va >> 12
  const uint64_t* page_off;
  uint64_t image_bytes;
  const uint64_t* value;     // fresh values (hpa for lanes; hpa of the chunk for pages)
  const uint32_t* status;    // fresh statuses
  uint32_t cap;
  uint32_t state_words;      // 2 * cap + 1
};

struct Lookup {
  uint64_t key, fresh;  // fresh: value (hpa) from the walk
  uint64_t off, chunk;  // page offset + chunk length (copy plans; for the OOR check of a hit)
  uint32_t op;
  bool walk_ok;         // the walk resolved (status OK, or OK walk + DATA_OOR)
  bool data_ok;         // status OK
  bool valid;
};

__device__ __forceinline__ Lookup load_lookup(const FifoStream& fs, uint64_t l, bool valid) {
  Lookup r;
  r.valid = valid;
  r.key = r.fresh = r.off = r.chunk = 0;
  r.op = kNoOp;
  r.walk_ok = r.data_ok = false;
  if (!valid) return r;
  const uint64_t ref = fs.ref[l];
  const uint32_t st = fs.status[ref];
  r.fresh = fs.value[ref];
  r.data_ok = st == PV_ST_OK;
  r.walk_ok = st == PV_ST_OK || st == PV_ST_DATA_OOR;
  if (fs.op == nullptr) {
    const uint64_t va = fs.va32 ? (uint64_t)((const uint32_t*)fs.vas)[ref] : ((const uint64_t*)fs.vas)[ref];
    r.key = va >> kPageShift;
    r.off = va & kPageMask;
    r.op = (uint32_t)l;  // every lane is its own op: never terminates a later one
  } else {
    const uint32_t o = fs.op[l];
    const pv_op op = fs.ops[o];
    const uint64_t k = ref - fs.page_off[o];
    const uint64_t cur = op_page_va(op.gva, k);
    r.key = cur >> kPageShift;
    r.off = cur & kPageMask;
    r.chunk = min(op.len - (cur - op.gva), kPageSize - r.off);
    r.op = o;
  }
  return r;
}

// The same lookup in three stages, for a software-pipelined window loop
// (fifo_spec_kernel): A loads the lookup's own words, B the words they point
// at, C derives the Lookup (load_lookup's arithmetic, same results).  Stage B
// of window w + 1 and stage A of window w + 2 are issued before window w is
// replayed, so their loads are in flight during the replay.
struct LookupA {
  uint64_t ref;
  uint32_t op;
  bool valid;
};
struct LookupB {
  LookupA a;
  uint64_t fresh, gva, len, poff;  // lanes: gva holds the lane's va
  uint32_t st;
};

__device__ __forceinline__ LookupA lookup_a(const FifoStream& fs, uint64_t l, bool valid) {
  LookupA a;
  a.valid = valid;
  a.ref = valid ? fs.ref[l] : 0;
  a.op = (valid && fs.op != nullptr) ? fs.op[l] : 0;
  return a;
}

__device__ __forceinline__ LookupB lookup_b(const FifoStream& fs, const LookupA& a) {
  LookupB b;
  b.a = a;
  b.fresh = b.gva = b.len = b.poff = 0;
  b.st = 0;
  if (!a.valid) return b;
  b.st = fs.status[a.ref];
  b.fresh = fs.value[a.ref];
  if (fs.op == nullptr) {
    b.gva = fs.va32 ? (uint64_t)((const uint32_t*)fs.vas)[a.ref] : ((const uint64_t*)fs.vas)[a.ref];
  } else {
    b.gva = fs.ops[a.op].gva;
    b.len = fs.ops[a.op].len;
    b.poff = fs.page_off[a.op];
  }
  return b;
}

__device__ __forceinline__ Lookup lookup_c(const FifoStream& fs, const LookupB& b, uint64_t l) {
  Lookup r;
  r.valid = b.a.valid;
  r.key = r.fresh = r.off = r.chunk = 0;
  r.op = kNoOp;
  r.walk_ok = r.data_ok = false;
  if (!r.valid) return r;
  r.fresh = b.fresh;
  r.data_ok = b.st == PV_ST_OK;
  r.walk_ok = b.st == PV_ST_OK || b.st == PV_ST_DATA_OOR;
  if (fs.op == nullptr) {
    r.key = b.gva >> kPageShift;
    r.off = b.gva & kPageMask;
    r.op = (uint32_t)l;
  } else {
    const uint64_t cur = op_page_va(b.gva, b.a.ref - b.poff);
    r.key = cur >> kPageShift;
    r.off = cur & kPageMask;
    r.chunk = min(b.len - (cur - b.gva), kPageSize - r.off);
    r.op = b.a.op;
  }
  return r;
}

// Cache state distributed over a warp: lane i < len holds the i-th oldest
// entry.  term_op: op whose pages are already terminated (copy plans).
struct WarpState {
  uint64_t qk, qv;
  uint32_t len;
  uint32_t term_op;
};

__device__ __forceinline__ uint32_t lt_mask(uint32_t lane) { return (1u << lane) - 1u; }

// Replay one window of n <= 32 lookups from state `s` (updated in place).
// Outputs per lane: hit, the hit's cached page, terminate, active.
__device__ void window_run(const FifoStream& fs, const Lookup& x, uint32_t n, uint32_t lane, WarpState& s,
                           bool* hit_out, uint64_t* hitpage_out, bool* term_out, bool* active_out,
                           uint64_t* counts) {
  const uint32_t full = 0xFFFFFFFFu;
  const uint32_t cap = fs.cap;
  const bool copy = fs.op != nullptr;
  const uint32_t valid = __ballot_sync(full, x.valid);
  // position of x.key in the start state (or -1)
  int qidx = -1;
  for (uint32_t i = 0; i < s.len; ++i) {
    const uint64_t k = __shfl_sync(full, s.qk, i);
    if (qidx < 0 && k == x.key) qidx = (int)i;
  }
  const uint64_t qval = __shfl_sync(full, s.qv, qidx < 0 ? 0 : qidx);
  const uint32_t same_key = __match_any_sync(full, x.valid ? x.key : ~0ull - lane);
  const uint32_t same_op = copy ? __match_any_sync(full, x.op) : (1u << lane);
  const uint32_t walk_ok = __ballot_sync(full, x.valid && x.walk_ok);
  uint32_t M = walk_ok, T = 0, A = valid;
  if (copy && s.term_op != kNoOp) A &= ~__ballot_sync(full, x.op == s.term_op);
  bool hit = false;
  uint64_t hitpage = 0;
  for (int it = 0; it < 34; ++it) {
    const uint32_t e = __popc(M & lt_mask(lane));
    const int ev = (int)s.len + (int)e - (int)cap;
    const bool in_q = qidx >= 0 && qidx >= ev;
    bool in_w = false;
    const uint32_t cand = same_key & M & lt_mask(lane);
    if (cand) {
      const uint32_t i = 31 - __clz(cand);
      const uint32_t ei = __popc(M & lt_mask(i));
      in_w = (e - ei) <= cap;  // fewer than `cap` insertions strictly between i and j
    }
    const bool active = (A >> lane) & 1u;
    hit = active && (in_q || in_w);
    hitpage = in_w ? (x.fresh >> kPageShift) : qval;  // a window insertion of this key cached the fresh page
    bool term = false;
    if (copy && active) {
      if (hit) {
        const uint64_t hpa = (hitpage << kPageShift) | x.off;
        term = hpa + x.chunk > fs.image_bytes || hpa + x.chunk < hpa;
      } else {
        term = !x.data_ok;
      }
    }
    const uint32_t T_new = __ballot_sync(full, term);
    const uint32_t M_new = __ballot_sync(full, active && !hit && x.walk_ok);
    uint32_t A_new = valid;
    if (copy) {
      if (s.term_op != kNoOp) A_new &= ~__ballot_sync(full, x.op == s.term_op);
      A_new &= ~__ballot_sync(full, (same_op & T_new & lt_mask(lane)) != 0);
    }
    const bool done = M_new == M && T_new == T && A_new == A;
    M = M_new;
    T = T_new;
    A = A_new;
    if (done) break;
  }
  const bool active = (A >> lane) & 1u;
  *hit_out = hit && active;
  *hitpage_out = hitpage;
  *term_out = (T >> lane) & 1u;
  *active_out = active;
  const uint32_t hits = __popc(__ballot_sync(full, hit && active));
  if (counts) *counts = (uint64_t)hits | ((uint64_t)__popc(A) << 32);  // hits | lookups
  // new state = last `cap` of (start entries ++ window insertions)
  const uint32_t ins = __popc(M);
  const uint32_t total = s.len + ins;
  const uint32_t nlen = total < cap ? total : cap;
  const uint32_t idx = total - nlen + lane;
  uint64_t nk = 0, nv = 0;
  // source lane: start entry idx, or the (idx - len)-th window insertion
  const bool from_q = idx < s.len;
  int src = from_q ? (int)idx : (lane < nlen ? (int)__fns(M, 0, (int)(idx - s.len) + 1) : 0);
  if (src < 0) src = 0;
  const uint64_t qk_s = __shfl_sync(full, s.qk, from_q ? src : 0);
  const uint64_t qv_s = __shfl_sync(full, s.qv, from_q ? src : 0);
  const uint64_t wk_s = __shfl_sync(full, x.key, from_q ? 0 : src);
  const uint64_t wv_s = __shfl_sync(full, x.fresh >> kPageShift, from_q ? 0 : src);
  if (lane < nlen) {
    nk = from_q ? qk_s : wk_s;
    nv = from_q ? qv_s : wv_s;
  }
  s.qk = nk;
  s.qv = nv;
  s.len = nlen;
  if (copy) {
    // the op of the window's last valid lookup carries over
    const uint32_t last = valid ? 31 - __clz(valid) : 0;
    const uint32_t last_op = __shfl_sync(full, x.op, last);
    const bool last_term = s.term_op == last_op || (__ballot_sync(full, x.op == last_op && ((T >> lane) & 1u)) != 0);
    if (n > 0) s.term_op = last_term ? last_op : kNoOp;
  }
}

__device__ __forceinline__ void load_state(const uint64_t* st, uint32_t cap, uint32_t lane, WarpState& s) {
  const uint64_t meta = st[2 * cap];
  s.len = (uint32_t)meta;
  s.term_op = (uint32_t)(meta >> 32);
  s.qk = lane < s.len ? st[lane] : 0;
  s.qv = lane < s.len ? st[cap + lane] : 0;
}
__device__ __forceinline__ void store_state(uint64_t* st, uint32_t cap, uint32_t lane, const WarpState& s) {
  if (lane < cap) {
    st[lane] = lane < s.len ? s.qk : 0;
    st[cap + lane] = lane < s.len ? s.qv : 0;
  }
  if (lane == 0) st[2 * cap] = (uint64_t)s.len | ((uint64_t)s.term_op << 32);
}

// Initial state of process p from its pv_fifo (ring -> oldest-first lanes).
__device__ __forceinline__ void initial_state(const pv_fifo& f, uint32_t lane, WarpState& s) {
  s.len = f.len;
  s.term_op = kNoOp;
  const uint32_t slot = f.capacity ? (f.head + lane) % f.capacity : 0;
  s.qk = lane < f.len ? f.key[slot] : 0;
  s.qv = lane < f.len ? f.val[slot] : 0;
}

struct Scratch {
  uint64_t* spec_start;  // [windows][state_words]
  uint64_t* spec_end;    // [windows][state_words]
  uint64_t* win_counts;  // [windows]: hits | lookups << 32
  uint8_t* match;        // [windows]
  uint64_t* block;       // [windows], at each 32-window block start of a process: bit 63 all
                         // windows of the block link to their predecessor; bits 0-31 the
                         // block's hits | lookups << 16
  uint64_t* hitpage;     // [lookups]
  uint8_t* flags;        // [lookups]: 1 hit, 2 terminate, 4 active
  uint64_t* run_off;     // [procs + 1]: first kRun-window run of each process
};

__device__ __forceinline__ uint32_t proc_of_window(const FifoStream& fs, uint64_t w) {
  uint32_t lo = 0, hi = fs.n_procs;
  while (hi - lo > 1) {
    const uint32_t m = (lo + hi) >> 1;
    if (fs.win_off[m] <= w) lo = m; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ void run_one(const FifoStream& fs, uint64_t lb, uint64_t le, uint64_t wi, uint32_t lane,
                                        WarpState& s, const Scratch* out, uint64_t* counts) {
  const uint64_t l0 = lb + wi * 32;
  const uint64_t l = l0 + lane;
  const bool valid = l < le;
  const uint32_t n = (uint32_t)(le > l0 ? (le - l0 < 32 ? le - l0 : 32) : 0);
  const Lookup x = load_lookup(fs, l, valid);
  bool hit, term, active;
  uint64_t hp;
  window_run(fs, x, n, lane, s, &hit, &hp, &term, &active, counts);
  if (out != nullptr && valid) {
    out->hitpage[l] = hp;
    out->flags[l] = (hit ? 1 : 0) | (term ? 2 : 0) | (active ? 4 : 0);
  }
}

// Step 1: speculate every window.  One warp per run of kRun consecutive
// windows of a process: the run's start state is rebuilt by replaying the
// kWarmWindows windows before it (exactly, from the initial cache, near the
// stream start), then its windows are replayed back to back, so every window
// after the first starts from its predecessor's speculated end state (its
// link flag is set here) and the warm-up is paid once per run, not per window.
#ifndef PV_FIFO_RUN
#define PV_FIFO_RUN 8
#endif
constexpr uint32_t kRun = PV_FIFO_RUN;

// Run order.  Processes' lookup streams interleave in the plan (their pages
// alternate in op order), so the r-th runs of all processes read the same
// region of the plan arrays: runs are scheduled process-minor (run k of
// process 0, 1, ..., then run k + 1 ...) so those sectors are fetched from
// HBM once and hit in L2 for the other processes, instead of once per process
// (8x the traffic at C2).  run_off[n_procs + 1] = max runs per process; the
// interleaved order is used when it wastes at most half the slots (balanced
// streams), else the process-major order run_off describes.
__device__ __forceinline__ bool run_of_slot(const uint64_t* run_off, uint32_t n_procs, bool interleave, uint64_t r,
                                            uint32_t* p_out, uint64_t* k_out) {
  if (interleave) {
    const uint32_t p = (uint32_t)(r % n_procs);
    const uint64_t k = r / n_procs;
    *p_out = p;
    *k_out = k;
    return k < run_off[p + 1] - run_off[p];
  }
  uint32_t lo = 0, hi = n_procs;
  while (hi - lo > 1) {
    const uint32_t m = (lo + hi) >> 1;
    if (run_off[m] <= r) lo = m; else hi = m;
  }
  *p_out = lo;
  *k_out = r - run_off[lo];
  return r < run_off[n_procs];
}

// Software-pipelined window loads at 3 CTAs/SM (80 registers): fifo_spec
// 0.578 -> 0.536 ms per C2 launch; at 4 CTAs/SM they spill (0.613 ms)
// (profiles/r02_fifo_pipe_ab.md)
#ifndef PV_FIFO_PIPE
#define PV_FIFO_PIPE 1
#endif
#ifndef PV_FIFO_SPEC_MINB
#define PV_FIFO_SPEC_MINB (PV_FIFO_PIPE ? 3 : 4)
#endif
__global__ void __launch_bounds__(256, PV_FIFO_SPEC_MINB) fifo_spec_kernel(FifoStream fs, const pv_fifo* __restrict__ fifo, Scratch sc, uint64_t n_slots_max,
                                 const uint64_t* __restrict__ run_off, unsigned long long* first_bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t total_runs = run_off[fs.n_procs], max_runs = run_off[fs.n_procs + 1];
  const bool interleave = max_runs * fs.n_procs <= 2 * total_runs;
  uint64_t n_slots = interleave ? max_runs * fs.n_procs : total_runs;
  if (n_slots > n_slots_max) n_slots = n_slots_max;
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_slots; r += nwarps) {
    uint32_t p;
    uint64_t k;
    if (!run_of_slot(run_off, fs.n_procs, interleave, r, &p, &k)) continue;
    const uint64_t w0 = fs.win_off[p], nw = fs.win_off[p + 1] - w0, lb = fs.lk_off[p], le = fs.lk_off[p + 1];
    const uint64_t wi0 = k * kRun;
    const uint64_t wi1 = wi0 + kRun < nw ? wi0 + kRun : nw;
    WarpState s;
    uint64_t from;
    const bool exact = wi0 <= (uint64_t)kWarmWindows;
    if (exact) {
      initial_state(fifo[p], lane, s);  // exact: replay from the stream start
      from = 0;
    } else {
      s.qk = s.qv = 0;
      s.len = 0;
      s.term_op = kNoOp;
      from = wi0 - kWarmWindows;
    }
#if PV_FIFO_PIPE
    // software-pipelined: window v replays while window v + 1's pointed-at
    // words and window v + 2's own words load
    auto lk = [&](uint64_t v) { return lb + v * 32 + lane; };
    LookupB nb = lookup_b(fs, lookup_a(fs, lk(from), lk(from) < le));
    LookupA na = lookup_a(fs, lk(from + 1), from + 1 < wi1 && lk(from + 1) < le);
    for (uint64_t v = from; v < wi1; ++v) {
      const Lookup x = lookup_c(fs, nb, lk(v));
      nb = lookup_b(fs, na);
      na = lookup_a(fs, lk(v + 2), v + 2 < wi1 && lk(v + 2) < le);
      const uint64_t l0 = lb + v * 32;
      const uint32_t n = (uint32_t)(le > l0 ? (le - l0 < 32 ? le - l0 : 32) : 0);
      bool hit, term, active;
      uint64_t hp;
      if (v < wi0) {  // warm-up window: state only
        window_run(fs, x, n, lane, s, &hit, &hp, &term, &active, nullptr);
        continue;
      }
      const uint64_t wi = v;
      const uint64_t w = w0 + wi;
      store_state(sc.spec_start + w * fs.state_words, fs.cap, lane, s);
      uint64_t counts = 0;
      window_run(fs, x, n, lane, s, &hit, &hp, &term, &active, &counts);
      if (x.valid) {
        sc.hitpage[lk(v)] = hp;
        sc.flags[lk(v)] = (hit ? 1 : 0) | (term ? 2 : 0) | (active ? 4 : 0);
      }
#else
    for (uint64_t v = from; v < wi0; ++v) run_one(fs, lb, le, v, lane, s, nullptr, nullptr);
    for (uint64_t wi = wi0; wi < wi1; ++wi) {
      const uint64_t w = w0 + wi;
      store_state(sc.spec_start + w * fs.state_words, fs.cap, lane, s);
      uint64_t counts = 0;
      run_one(fs, lb, le, wi, lane, s, &sc, &counts);
#endif
      store_state(sc.spec_end + w * fs.state_words, fs.cap, lane, s);
      if (lane == 0) {
        sc.win_counts[w] = counts;
        sc.match[w] = (exact || wi > wi0) ? 1 : 0;  // exact start state, or linked inside the run
      }
      // copy plans: every op of this window starts from "not failed"
      if (fs.op != nullptr && first_bad != nullptr) {
        const uint64_t l = lb + wi * 32 + lane;
        if (l < le) {
          const uint32_t o = fs.op[l];
          if (fs.ref[l] == fs.page_off[o]) first_bad[o] = kNone;
        }
      }
    }
  }
}

// run_off[p] = number of kRun-window runs before process p (one thread).
// run_off[n_procs + 1] = the most runs of any process (one thread).
__global__ void fifo_runs_kernel(FifoStream fs, uint64_t* run_off) {
  uint64_t acc = 0, most = 0;
  for (uint32_t p = 0; p < fs.n_procs; ++p) {
    run_off[p] = acc;
    const uint64_t n = (fs.win_off[p + 1] - fs.win_off[p] + kRun - 1) / kRun;
    acc += n;
    most = n > most ? n : most;
  }
  run_off[fs.n_procs] = acc;
  run_off[fs.n_procs + 1] = most;
}

// Step 2: link neighbouring windows.
__global__ void fifo_link_kernel(FifoStream fs, Scratch sc, uint64_t n_windows) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_windows || sc.match[w]) return;
  const uint32_t p = proc_of_window(fs, w);
  if (w == fs.win_off[p]) return;
  const uint64_t* a = sc.spec_end + (w - 1) * fs.state_words;
  const uint64_t* b = sc.spec_start + w * fs.state_words;
  const uint32_t len = (uint32_t)a[2 * fs.cap];
  bool eq = a[2 * fs.cap] == b[2 * fs.cap];
  for (uint32_t i = 0; eq && i < len; ++i) eq = a[i] == b[i] && a[fs.cap + i] == b[fs.cap + i];
  sc.match[w] = eq ? 1 : 0;
}

// Step 2b: per 32-window block of each process (aligned to the process's
// first window): do all its windows link, and its hit / lookup sums.
__global__ void fifo_block_kernel(FifoStream fs, Scratch sc, uint64_t n_windows) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_windows) return;
  const uint32_t p = proc_of_window(fs, w);
  const uint64_t w0 = fs.win_off[p], w1 = fs.win_off[p + 1];
  if ((w - w0) & 31) return;
  const uint64_t e = w + 32 < w1 ? w + 32 : w1;
  bool all = true;
  uint32_t hits = 0, looks = 0;
  for (uint64_t v = w; v < e; ++v) {
    all &= sc.match[v] != 0;
    const uint64_t c = sc.win_counts[v];
    hits += (uint32_t)c;
    looks += (uint32_t)(c >> 32);
  }
  sc.block[w] = ((uint64_t)all << 63) | hits | ((uint64_t)looks << 16);
}

// Step 3: verify each process's chain; replay mismatching windows exactly.
__global__ void fifo_verify_kernel(FifoStream fs, pv_fifo* __restrict__ fifo, Scratch sc) {
  const uint32_t full = 0xFFFFFFFFu;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= fs.n_procs) return;
  const uint64_t w0 = fs.win_off[p], w1 = fs.win_off[p + 1], lb = fs.lk_off[p], le = fs.lk_off[p + 1];
  WarpState s;
  initial_state(fifo[p], lane, s);
  // have_s: s holds the true state before window w; otherwise that state is
  // spec_end[w - 1] (the previous window was accepted as speculated).
  bool have_s = true;
  uint64_t hits = 0, lookups = 0;
  // block summaries, 32 blocks (1024 windows) per warp load, one group ahead
  const uint64_t n_blocks = (w1 - w0 + 31) >> 5;
  uint64_t grp = lane < n_blocks ? sc.block[w0 + 32ull * lane] : 0;
  for (uint64_t kb = 0; kb < n_blocks; kb += 32) {
    const uint64_t cur_grp = grp;
    grp = kb + 32 + lane < n_blocks ? sc.block[w0 + 32ull * (kb + 32 + lane)] : 0;
    const uint32_t nq = (uint32_t)(n_blocks - kb < 32 ? n_blocks - kb : 32);
    for (uint32_t q = 0; q < nq; ++q) {
    const uint64_t wb = w0 + 32ull * (kb + q);
    const uint64_t rec = __shfl_sync(full, cur_grp, q);
    if (!have_s && (rec >> 63)) {  // every window links: accepted as speculated
      hits += rec & 0xFFFF;
      lookups += (rec >> 16) & 0xFFFF;
      continue;
    }
    const uint32_t mm = __ballot_sync(full, wb + lane < w1 && sc.match[wb + lane] != 0);
    const uint64_t wc = wb + lane < w1 ? sc.win_counts[wb + lane] : 0;
    // per-window hits | lookups packed in 16-bit halves for warp sums (<= 32 each)
    const uint32_t wc16 = (uint32_t)(wc & 0xFFFF) | ((uint32_t)((wc >> 32) & 0xFFFF) << 16);
    const uint32_t nb = (uint32_t)(w1 - wb < 32 ? w1 - wb : 32);
    uint32_t j = 0;
    while (j < nb) {
      if (!have_s) {
        // accept the whole run of linked windows j .. z-1 at once
        const uint32_t rest = ~mm & (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) & ~((1u << j) - 1u);
        const uint32_t z = rest ? __ffs(rest) - 1 : nb;
        if (z > j) {
          const uint32_t sum = __reduce_add_sync(full, (lane >= j && lane < z) ? wc16 : 0u);
          hits += sum & 0xFFFF;
          lookups += sum >> 16;
          j = z;
        }
        if (j >= nb) break;
        load_state(sc.spec_end + (wb + j - 1) * fs.state_words, fs.cap, lane, s);
        have_s = true;
      }
      const uint64_t w = wb + j;
      const uint64_t cj = __shfl_sync(full, wc, j);
      const uint64_t* b = sc.spec_start + w * fs.state_words;
      const uint64_t meta = b[2 * fs.cap];
      const bool lane_eq = lane >= s.len || (b[lane] == s.qk && b[fs.cap + lane] == s.qv);
      const bool same = (uint32_t)meta == s.len && (uint32_t)(meta >> 32) == s.term_op && __all_sync(full, lane_eq);
      if (same) {
        hits += (uint32_t)cj;
        lookups += cj >> 32;
        have_s = false;
      } else {
        uint64_t c = 0;
        run_one(fs, lb, le, w - w0, lane, s, &sc, &c);
        hits += (uint32_t)c;
        lookups += c >> 32;
      }
      ++j;
    }
    }
  }
  if (!have_s) load_state(sc.spec_end + (w1 - 1) * fs.state_words, fs.cap, lane, s);
  pv_fifo& f = fifo[p];
  if (lane < f.capacity) {
    f.key[lane] = lane < s.len ? s.qk : 0;
    f.val[lane] = lane < s.len ? s.qv : 0;
  }
  if (lane == 0) {
    f.len = s.len;
    f.head = 0;
    f.hits += hits;
    f.misses += lookups - hits;
  }
}

// Step 4: apply hits and terminations (one warp per run of kRun windows, in
// the speculation's run order so the scattered page writes of all processes
// land in the same plan region at the same time).
__device__ __forceinline__ void apply_one(const FifoStream& fs, const Scratch& sc, uint64_t l, uint64_t* value,
                                          uint32_t* status, unsigned long long* first_bad) {
  const uint8_t fl = sc.flags[l];
  if (!(fl & 3)) return;
  const uint64_t ref = fs.ref[l];
  if (fs.op == nullptr) {
    const uint64_t va = fs.va32 ? (uint64_t)((const uint32_t*)fs.vas)[ref] : ((const uint64_t*)fs.vas)[ref];
    value[ref] = (sc.hitpage[l] << kPageShift) | (va & kPageMask);
    status[ref] = PV_ST_OK;
    return;
  }
  const uint32_t o = fs.op[l];
  const pv_op op = fs.ops[o];
  const uint64_t k = ref - fs.page_off[o];
  const uint64_t cur = op_page_va(op.gva, k);
  if (fl & 1) {
    value[ref] = (sc.hitpage[l] << kPageShift) | (cur & kPageMask);
    status[ref] = (fl & 2) ? PV_ST_DATA_OOR : PV_ST_OK;
  }
  if (fl & 2) first_bad[o] = k;
}

__global__ void fifo_apply_kernel(FifoStream fs, Scratch sc, uint64_t n_slots_max, const uint64_t* __restrict__ run_off,
                                  uint64_t* value, uint32_t* status, unsigned long long* first_bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t total_runs = run_off[fs.n_procs], max_runs = run_off[fs.n_procs + 1];
  const bool interleave = max_runs * fs.n_procs <= 2 * total_runs;
  uint64_t n_slots = interleave ? max_runs * fs.n_procs : total_runs;
  if (n_slots > n_slots_max) n_slots = n_slots_max;
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_slots; r += nwarps) {
    uint32_t p;
    uint64_t k;
    if (!run_of_slot(run_off, fs.n_procs, interleave, r, &p, &k)) continue;
    const uint64_t lb = fs.lk_off[p], le = fs.lk_off[p + 1];
    const uint64_t l0 = lb + k * kRun * 32;
    const uint64_t l1 = l0 + kRun * 32 < le ? l0 + kRun * 32 : le;
    for (uint64_t l = l0 + lane; l < l1; l += 32) apply_one(fs, sc, l, value, status, first_bad);
  }
}

// ---- launchers ------------------------------------------------------------------

// The run offsets ([procs + 1] u64) sit at the front: a process without
// windows adds no run but still needs an offset, so they are sized by a
// generous 64 Ki processes (the ABI caller does not pass the process count).
constexpr uint64_t kMaxProcsScratch = 1ull << 16;
size_t fifo_scratch_bytes(uint64_t n_lookups, uint64_t n_windows, uint32_t cap) {
  const uint64_t sw = 2ull * cap + 1;
  return (kMaxProcsScratch + 2) * 8 + 2 * n_windows * sw * 8 + 2 * n_windows * 8 + n_windows + n_lookups * 8 +
         n_lookups + 256;
}

static Scratch carve(void* base, uint64_t n_lookups, uint64_t n_windows, uint32_t cap) {
  const uint64_t sw = 2ull * cap + 1;
  uint8_t* p = static_cast<uint8_t*>(base);
  Scratch s;
  s.run_off = reinterpret_cast<uint64_t*>(p);
  p += (kMaxProcsScratch + 2) * 8;
  s.spec_start = reinterpret_cast<uint64_t*>(p);
  p += n_windows * sw * 8;
  s.spec_end = reinterpret_cast<uint64_t*>(p);
  p += n_windows * sw * 8;
  s.hitpage = reinterpret_cast<uint64_t*>(p);
  p += n_lookups * 8;
  s.win_counts = reinterpret_cast<uint64_t*>(p);
  p += n_windows * 8;
  s.block = reinterpret_cast<uint64_t*>(p);
  p += n_windows * 8;
  s.match = p;
  p += n_windows;
  s.flags = p;
  return s;
}

cudaError_t launch_fifo_stream(const FifoStream& fs, pv_fifo* fifo, void* scratch, uint64_t n_lookups,
                               uint64_t n_windows, uint64_t* value, uint32_t* status, uint64_t* first_bad,
                               cudaStream_t stream) {
  if (fs.n_procs == 0 || n_windows == 0) return cudaSuccess;
  if (fs.n_procs > kMaxProcsScratch) return cudaErrorInvalidValue;
  const Scratch sc = carve(scratch, n_lookups, n_windows, fs.cap);
  auto* fb = reinterpret_cast<unsigned long long*>(first_bad);
  {
    uint64_t* run_off = sc.run_off;
    fifo_runs_kernel<<<1, 1, 0, stream>>>(fs, run_off);
    // every process contributes ceil(nw / kRun) runs <= nw / kRun + 1; the
    // interleaved order uses at most 2x the runs (the kernel clamps)
    const uint64_t runs_max = 2 * (n_windows / kRun + fs.n_procs);
    uint64_t grid = (runs_max / 2 + 7) / 8;
    const uint64_t cap = resident_grid((const void*)fifo_spec_kernel, 256, 0);
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    void* tk = timing_begin("fifo_spec", stream);
    fifo_spec_kernel<<<(unsigned)grid, 256, 0, stream>>>(fs, fifo, sc, runs_max, run_off, fb);
    timing_end(tk, stream);
  }
  fifo_link_kernel<<<(unsigned)((n_windows + 255) / 256), 256, 0, stream>>>(fs, sc, n_windows);
  fifo_block_kernel<<<(unsigned)((n_windows + 255) / 256), 256, 0, stream>>>(fs, sc, n_windows);
  fifo_verify_kernel<<<(fs.n_procs + 3) / 4, 128, 0, stream>>>(fs, fifo, sc);
  {
    const uint64_t runs_max = 2 * (n_windows / kRun + fs.n_procs);
    uint64_t grid = (runs_max / 2 + 7) / 8;
    const uint64_t cap = resident_grid((const void*)fifo_apply_kernel, 256, 0);
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    fifo_apply_kernel<<<(unsigned)grid, 256, 0, stream>>>(fs, sc, runs_max, sc.run_off, value, status, fb);
  }
  return cudaGetLastError();
}

// n_lookups / n_windows come from the caller (proc_off[n_procs] and
// win_off[n_procs]): the launch never reads device memory back.
cudaError_t launch_fifo_lanes_abi(const void* vas, uint32_t flags, const uint64_t* lane_idx, const uint64_t* proc_off,
                                  const uint64_t* win_off, uint32_t n_procs, uint64_t n_lookups, uint64_t n_windows,
                                  uint32_t cap, pv_fifo* fifo,
                                  uint64_t* value, uint32_t* status, void* scratch, uint64_t scratch_bytes,
                                  cudaStream_t stream) {
  FifoStream fs{};
  fs.ref = lane_idx;
  fs.op = nullptr;
  fs.lk_off = proc_off;
  fs.win_off = win_off;
  fs.n_procs = n_procs;
  fs.vas = vas;
  fs.va32 = (flags & PV_VA32) ? 1u : 0u;
  fs.value = value;
  fs.status = status;
  fs.cap = cap;
  fs.state_words = 2 * cap + 1;
  if (scratch_bytes < fifo_scratch_bytes(n_lookups, n_windows, cap)) return cudaErrorInvalidValue;
  return launch_fifo_stream(fs, fifo, scratch, n_lookups, n_windows, value, status, nullptr, stream);
}

cudaError_t launch_fifo_copy_abi(const pv_op* ops, const uint64_t* page_off, const uint64_t* look_page,
                                 const uint32_t* look_op, const uint64_t* proc_off, const uint64_t* win_off,
                                 uint32_t n_procs, uint64_t n_lookups, uint64_t n_windows, uint32_t cap, pv_fifo* fifo,
                                 uint64_t image_bytes,
                                 uint64_t* page_hpa, uint32_t* page_status, uint64_t* op_first_bad, void* scratch,
                                 uint64_t scratch_bytes, cudaStream_t stream) {
  FifoStream fs{};
  fs.ref = look_page;
  fs.op = look_op;
  fs.lk_off = proc_off;
  fs.win_off = win_off;
  fs.n_procs = n_procs;
  fs.ops = ops;
  fs.page_off = page_off;
  fs.image_bytes = image_bytes;
  fs.value = page_hpa;
  fs.status = page_status;
  fs.cap = cap;
  fs.state_words = 2 * cap + 1;
  if (scratch_bytes < fifo_scratch_bytes(n_lookups, n_windows, cap)) return cudaErrorInvalidValue;
  return launch_fifo_stream(fs, fifo, scratch, n_lookups, n_windows, page_hpa, page_status, op_first_bad, stream);
}

}  // namespace pv
