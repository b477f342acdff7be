/*
 * pvoracle.c — CPU restatement of the reference's hybrid-address-space data
 * plane.  TEST INFRASTRUCTURE ONLY: imported by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs as the checker and the CPU baseline.  The product (libpv.so and the
 * paper_1304_3771_b200 package) never links or calls it.
 *
 * Restated from /root/reference/pkg/src/devfsim (paths below are relative
 * to that directory):
 *   orc_walk            memvirt.py:244-259   walk (3 levels, T before P,
 *                                            W ignored, top index masked to
 *                                            2 bits, unchecked node reads ->
 *                                            here a NODE_OOR status)
 *   orc_translate       memvirt.py:585-601   ProcessTranslator.translate /
 *                                            _resolve_page (shadow: one walk;
 *                                            tdp: walk_guest then TDP walk)
 *                       memvirt.py:262-267   walk_guest (gpa = pfn<<12|off)
 *                       memvirt.py:677-682   resolve_hybrid
 *   orc_cache_*         memvirt.py:336-374   TranslationCache FIFO
 *   orc_copy            memvirt.py:604-628   copy_user_buffer (chunking,
 *                                            prefix on fault, bytes_copied)
 *                       memvirt.py:156-168   PhysMem read/write bounds ->
 *                                            OutOfRange
 *   orc_copy_hybrid     memvirt.py:685-696   resolve_hybrid_with_fixup with
 *                       backend.py:288-296   the default trap shim (walk_guest,
 *                       memvirt.py:491-497   gpa_to_hpa, TableEditor.map
 *                       memvirt.py:282-313   replace=True) inside
 *                                            copy_user_buffer; shims that
 *                                            would allocate a node or raise
 *                                            stop the batch (ST_SHIM_HOST)
 * Status words use the same encoding as include/pv.h so results compare
 * directly; the encoding is defined there, the semantics here.
 * Parity of this file against the reference itself is pinned by
 * tests/test_oracle.py over tests/golden/ (generated from the reference by
 * tests/golden/gen_golden.py).
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ST_OK 0x000u
#define ST_FAULT 0x010u
#define ST_FAULT2 0x020u
#define ST_TRAP 0x040u
#define ST_TRAP2 0x060u
#define ST_NODE_OOR 0x080u
#define ST_NODE_OOR2 0x0A0u
#define ST_DATA_OOR 0x100u

#define PG 4096ull

typedef struct {
  uint64_t s1_base, s1_root, s2_root;
  uint32_t mode, pad; /* 1 = one stage, 2 = two stage (TDP) */
} orc_space;

typedef struct {
  uint64_t key[32], val[32];
  uint64_t hits, misses;
  uint32_t capacity, len, head, pad;
} orc_fifo; /* same layout as pv_fifo */

static uint64_t rd64(const uint8_t* img, uint64_t off) {
  uint64_t w;
  memcpy(&w, img + off, 8); /* little-endian host */
  return w;
}

/* memvirt.py:244-259.  Returns status; *out = leaf pfn (ok), node (trap). */
uint32_t orc_walk(const uint8_t* img, uint64_t img_bytes, uint64_t base, uint64_t root, uint64_t va, int stage2,
                  uint64_t* out) {
  const uint32_t index[3] = {(uint32_t)((va >> 30) & 3u), (uint32_t)((va >> 21) & 0x1FFu),
                             (uint32_t)((va >> 12) & 0x1FFu)};
  uint64_t node = root;
  for (uint32_t level = 1; level <= 3; ++level) {
    /* read_word: base + node*4096 + index*8 must lie inside the buffer */
    if (base >= img_bytes || node >= (img_bytes - base) / PG)
      return (stage2 ? ST_NODE_OOR2 : ST_NODE_OOR) | level;
    const uint64_t w = rd64(img, base + node * PG + (uint64_t)index[level - 1] * 8u);
    if (w & 0x4u) { /* TRAPPING is tested before PRESENT */
      *out = node;
      return (stage2 ? ST_TRAP2 : ST_TRAP) | level | (index[level - 1] << 16);
    }
    if (!(w & 0x1u)) return (stage2 ? ST_FAULT2 : ST_FAULT) | level;
    node = w >> 12;
  }
  *out = node;
  return ST_OK;
}

/* Extension geometry (mode 3, BASELINE config 3; NOT a reference semantic,
 * so this restatement is the only anchor -- "parity unpinned"): 4 levels of
 * 512 entries over 48-bit VAs, the reference's entry codec (T before P, W
 * ignored), and a 2 MiB leaf at level 3 when bit 0x80 (PS) is set.  Returns
 * the 4 KiB frame of va. */
uint32_t orc_walk4(const uint8_t* img, uint64_t img_bytes, uint64_t base, uint64_t root, uint64_t va,
                   uint64_t* out) {
  uint64_t node = root;
  for (uint32_t level = 1; level <= 4; ++level) {
    const uint32_t index = (uint32_t)((va >> (12 + 9 * (4 - level))) & 0x1FFu);
    if (base >= img_bytes || node >= (img_bytes - base) / PG) return ST_NODE_OOR | level;
    const uint64_t w = rd64(img, base + node * PG + (uint64_t)index * 8u);
    if (w & 0x4u) {
      *out = node;
      return ST_TRAP | level | (index << 16);
    }
    if (!(w & 0x1u)) return ST_FAULT | level;
    if (level == 3 && (w & 0x80u)) {
      *out = (w >> 12) + ((va >> 12) & 0x1FFu);
      return ST_OK;
    }
    node = w >> 12;
  }
  *out = node;
  return ST_OK;
}

/* One uncached translation; value/aux follow the pv.h conventions.
 * want_pfn: return the leaf pfn (walk) instead of the address. */
uint32_t orc_translate1(const uint8_t* img, uint64_t img_bytes, const orc_space* sp, uint64_t va, int want_pfn,
                        uint64_t* value, uint64_t* aux) {
  uint64_t r = 0;
  *aux = 0;
  if (sp->mode == 3) {
    const uint32_t st4 = orc_walk4(img, img_bytes, sp->s1_base, sp->s1_root, va, &r);
    if (st4 != ST_OK) {
      *value = ((st4 & 0xFF0u) == ST_TRAP) ? r : va;
      return st4;
    }
    *value = want_pfn ? r : ((r << 12) | (va & 0xFFFu));
    return ST_OK;
  }
  uint32_t st = orc_walk(img, img_bytes, sp->s1_base, sp->s1_root, va, 0, &r);
  if (st != ST_OK) {
    *value = ((st & 0xFF0u) == ST_TRAP) ? r : va;
    return st;
  }
  if (sp->mode == 2) {
    const uint64_t gpa = (r << 12) | (va & 0xFFFu);
    st = orc_walk(img, img_bytes, 0, sp->s2_root, gpa, 1, &r);
    if (st != ST_OK) {
      if ((st & 0xFF0u) == ST_TRAP2) {
        *value = r;
        *aux = gpa;
      } else {
        *value = gpa;
      }
      return st;
    }
  }
  *value = want_pfn ? r : ((r << 12) | (va & 0xFFFu));
  return ST_OK;
}

/* Batch of independent uncached translations (threads = OpenMP). */
void orc_translate(const uint8_t* img, uint64_t img_bytes, const orc_space* sp, const uint64_t* vas, uint64_t n,
                   int want_pfn, uint64_t* value, uint32_t* status, uint64_t* aux, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static) if (threads != 1)
#endif
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    uint64_t a = 0;
    status[i] = orc_translate1(img, img_bytes, sp, vas[i], want_pfn, &value[i], &a);
    if (aux) aux[i] = a;
  }
}

/* ---- FIFO cache (memvirt.py:336-374) ---------------------------------- */
static int cache_lookup(orc_fifo* c, uint64_t key, uint64_t* val) {
  for (uint32_t j = 0; j < c->len; ++j) {
    const uint32_t slot = (c->head + j) % c->capacity;
    if (c->key[slot] == key) {
      ++c->hits;
      *val = c->val[slot];
      return 1;
    }
  }
  ++c->misses;
  return 0;
}

static void cache_insert(orc_fifo* c, uint64_t key, uint64_t val) {
  uint32_t slot;
  if (c->len >= c->capacity) { /* popleft the oldest */
    slot = c->head;
    c->head = (c->head + 1) % c->capacity;
  } else {
    slot = (c->head + c->len) % c->capacity;
    ++c->len;
  }
  c->key[slot] = key;
  c->val[slot] = val;
}

/* ProcessTranslator.translate with the cache (memvirt.py:585-594), lane by
 * lane in order. */
void orc_translate_cached(const uint8_t* img, uint64_t img_bytes, const orc_space* sp, const uint64_t* vas,
                          uint64_t n, orc_fifo* cache, uint64_t* value, uint32_t* status, uint64_t* aux) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t va = vas[i];
    uint64_t hv = 0, a = 0;
    if (cache_lookup(cache, va >> 12, &hv)) {
      value[i] = (hv << 12) | (va & 0xFFFu);
      status[i] = ST_OK;
      if (aux) aux[i] = 0;
      continue;
    }
    status[i] = orc_translate1(img, img_bytes, sp, va, 0, &value[i], &a);
    if (aux) aux[i] = a;
    if (status[i] == ST_OK) cache_insert(cache, va >> 12, value[i] >> 12);
  }
}

/* ---- copy_user_buffer (memvirt.py:604-628) ---------------------------- */
typedef struct {
  uint64_t copied, value, aux;
  uint32_t status, fail_page;
} orc_result; /* same layout as pv_op_result */

/* One op.  direction 0 = to_guest (buf -> image), 1 = from_guest.
 * cache may be NULL (uncached translator). */
void orc_copy1(uint8_t* img, uint64_t img_bytes, const orc_space* sp, uint64_t gva, uint64_t len, uint8_t* buf,
               int direction, orc_fifo* cache, orc_result* res) {
  uint64_t copied = 0, page = 0;
  memset(res, 0, sizeof(*res));
  while (copied < len) {
    const uint64_t cur = gva + copied;
    uint64_t chunk = PG - (cur & 0xFFFu);
    if (chunk > len - copied) chunk = len - copied;
    uint64_t hpa = 0, a = 0, hv = 0;
    uint32_t st = ST_OK;
    if (cache && cache_lookup(cache, cur >> 12, &hv)) {
      hpa = (hv << 12) | (cur & 0xFFFu);
    } else {
      st = orc_translate1(img, img_bytes, sp, cur, 0, &hpa, &a);
      if (st != ST_OK) {
        res->copied = copied;
        res->value = hpa;
        res->aux = a;
        res->status = st;
        res->fail_page = (uint32_t)page;
        return;
      }
      if (cache) cache_insert(cache, cur >> 12, hpa >> 12);
    }
    if (hpa + chunk > img_bytes || hpa + chunk < hpa) { /* OutOfRange */
      res->copied = copied;
      res->value = hpa;
      res->status = ST_DATA_OOR;
      res->fail_page = (uint32_t)page;
      return;
    }
    if (direction == 0)
      memcpy(img + hpa, buf + copied, chunk);
    else
      memcpy(buf + copied, img + hpa, chunk);
    copied += chunk;
    ++page;
  }
  res->copied = copied;
  res->status = ST_OK;
}

/* A batch of ops in program order (rows gva, len, buf_off, space).  Ops run
 * sequentially (exact last-writer-wins); `threads` > 1 runs ops in parallel
 * and is only valid when their destinations are disjoint and no cache is
 * used (the cpu baseline). */
void orc_copy(uint8_t* img, uint64_t img_bytes, const orc_space* spaces, const uint64_t* ops, uint64_t n_ops,
              uint8_t* buf, int direction, orc_fifo* caches, const int32_t* op_cache, orc_result* results,
              int threads) {
  if (threads != 1 && caches == 0) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t i = 0; i < (int64_t)n_ops; ++i) {
      const uint64_t* o = ops + 4 * i;
      orc_copy1(img, img_bytes, &spaces[o[3] & 0xFFFFFFFFu], o[0], o[1], buf + o[2], direction, 0, &results[i]);
    }
    return;
  }
  for (uint64_t i = 0; i < n_ops; ++i) {
    const uint64_t* o = ops + 4 * i;
    orc_fifo* c = (caches && op_cache && op_cache[i] >= 0) ? &caches[op_cache[i]] : 0;
    orc_copy1(img, img_bytes, &spaces[o[3] & 0xFFFFFFFFu], o[0], o[1], buf + o[2], direction, c, &results[i]);
  }
}

/* ---- hybrid copies with the default trap shim ------------------------- */
#define ST_SHIM_HOST 0x800u /* the shim would allocate, raise or diverge: not restated */

typedef struct {
  uint64_t guest_base, guest_bytes, guest_root, shadow_root;
} orc_shim; /* same layout as pv_shim */

/* backend.py:288-296 for a trap at `va`: 0 and the word written, or
 * ST_SHIM_HOST.  The shadow descend follows every entry that is not
 * NOT_PRESENT (memvirt.py:282-298); a NOT_PRESENT upper entry would allocate. */
static uint32_t shim_once(uint8_t* img, uint64_t img_bytes, const orc_shim* sh, uint64_t va) {
  const uint64_t page_va = va & ~0xFFFull;
  uint64_t gpfn = 0;
  if (orc_walk(img, img_bytes, sh->guest_base, sh->guest_root, page_va, 0, &gpfn) != ST_OK) return ST_SHIM_HOST;
  const uint64_t gpa = gpfn << 12;
  if (gpa >= sh->guest_bytes) return ST_SHIM_HOST; /* gpa_to_hpa: OutOfRange */
  const uint64_t lim = img_bytes / PG;
  uint64_t node = sh->shadow_root;
  const uint32_t idx[3] = {(uint32_t)((page_va >> 30) & 3u), (uint32_t)((page_va >> 21) & 0x1FFu),
                           (uint32_t)((page_va >> 12) & 0x1FFu)};
  for (int l = 0; l < 2; ++l) {
    if (node >= lim) return ST_SHIM_HOST;
    const uint64_t w = rd64(img, node * PG + (uint64_t)idx[l] * 8u);
    if (!(w & 0x5u)) return ST_SHIM_HOST;
    node = w >> 12;
  }
  if (node >= lim) return ST_SHIM_HOST;
  const uint64_t hpa = sh->guest_base + gpa;
  const uint64_t word = ((hpa >> 12) << 12) | 0x3u; /* PRESENT | writable */
  memcpy(img + node * PG + (uint64_t)idx[2] * 8u, &word, 8);
  return ST_OK;
}

/* copy_user_buffer through _HybridResolver (backend.py:117-128): each page
 * resolves through the hybrid root (spaces[op].s1_root, host memory); a trap
 * runs the shim once and retries; a second trap is TrapFixupFailed
 * (status ST_TRAP | ST_SHIM_HOST here).  Ops run in order.  Returns the index
 * of the first op whose shim is outside the restated subset (that op's
 * status carries ST_SHIM_HOST and nothing after it ran), or n_ops.
 * *translations counts translate() calls (hw_translations). */
uint64_t orc_copy_hybrid(uint8_t* img, uint64_t img_bytes, const orc_space* spaces, const orc_shim* shims,
                         const uint64_t* ops, uint64_t n_ops, uint8_t* buf, int direction, orc_result* results,
                         uint64_t* translations) {
  for (uint64_t i = 0; i < n_ops; ++i) {
    const uint64_t* o = ops + 4 * i;
    const orc_space* sp = &spaces[o[3] & 0xFFFFFFFFu];
    const orc_shim* sh = &shims[o[3] & 0xFFFFFFFFu];
    const uint64_t gva = o[0], len = o[1];
    uint8_t* b = buf + o[2];
    orc_result* res = &results[i];
    uint64_t copied = 0, page = 0;
    memset(res, 0, sizeof(*res));
    while (copied < len) {
      const uint64_t cur = gva + copied;
      uint64_t chunk = PG - (cur & 0xFFFu);
      if (chunk > len - copied) chunk = len - copied;
      uint64_t hpa = 0, a = 0;
      ++*translations;
      uint32_t st = orc_translate1(img, img_bytes, sp, cur, 0, &hpa, &a);
      if ((st & 0xFF0u) == ST_TRAP) {
        if (sh->guest_bytes == 0 || shim_once(img, img_bytes, sh, cur) != ST_OK) {
          res->copied = copied;
          res->value = hpa;
          res->status = st | ST_SHIM_HOST;
          res->fail_page = (uint32_t)page;
          return i;
        }
        st = orc_translate1(img, img_bytes, sp, cur, 0, &hpa, &a);
        if ((st & 0xFF0u) == ST_TRAP) { /* TrapFixupFailed */
          res->copied = copied;
          res->value = hpa;
          res->status = st | ST_SHIM_HOST;
          res->fail_page = (uint32_t)page;
          return i;
        }
      }
      if (st != ST_OK) {
        res->copied = copied;
        res->value = hpa;
        res->aux = a;
        res->status = st;
        res->fail_page = (uint32_t)page;
        break;
      }
      if (hpa + chunk > img_bytes || hpa + chunk < hpa) {
        res->copied = copied;
        res->value = hpa;
        res->status = ST_DATA_OOR;
        res->fail_page = (uint32_t)page;
        break;
      }
      if (direction == 0)
        memcpy(img + hpa, b + copied, chunk);
      else
        memcpy(b + copied, img + hpa, chunk);
      copied += chunk;
      ++page;
    }
    if (copied == len) {
      res->copied = copied;
      res->status = ST_OK;
    }
  }
  return n_ops;
}

int orc_abi_version(void) { return 1; }
