// wide_heavy.cuh — recursion of the trie-binned MSD path into oversize bins
// ("oversize bins recurse on the next digit"), and the
// level-2 scatter of very uneven first-level buckets.
// Included once, by wide.cu, inside its anonymous namespace: it uses that
// file's constants, match_digit8, the bulk-copy helpers and sort_bin.
//
// After the two MSD levels every key sits in its 16-bit bin, stably.  A bin
// holding more than kLocalCap keys cannot be sorted in shared memory; it becomes
// a "heavy segment" and is refined by further stable 8-bit MSD scatters on the
// next digits (the bins of Alg. 5 are the leaves of the trie,
// and a deeper trie level is the next digit), until every piece fits:
//
//   level r >= 0 (digit bits [sh, sh + w), sh = kb - 24 - 8r, w = 8 or what is left)
//     A. every segment is split into nc <= kHeavyMaxChunks chunks;
//     B. one CTA per chunk counts its keys' digits (chist[chunk][256]);
//     C. one CTA per segment sums its chunks' counts (T[d]), scans them into the
//        digit bases, gives every chunk its own per-digit start (cbase), and
//        classifies the sub-bins [base_d, base_d + T[d]): heavy ones (> cap)
//        become segments of level r+1; runs of the others are merged greedily
//        into local-sort items of <= cap keys; a segment whose keys all share
//        the digit is passed down without moving;
//     D. CTAs take whole chunks and scatter them tile by tile in order, so the
//        per-digit offsets are running sums in registers (no lookback); the
//        next tile is bulk-copied (TMA) into the second shared buffer while
//        the current one is ranked, reordered and written.
//   Phases are separated by grid-wide barriers of one cooperative kernel.
//   Level -1 (only when k_msd_plan found the first-level buckets too uneven for
//   the interleaved lookback of k_scatter mode 2): the same A-D over the 256
//   buckets with the second digit, from the temporary buffer into the output,
//   without classification (the 16-bit bins are already planned).
// Then one kernel sorts every item (sort_bin) from where it lies into the
// output.  Data ping-pong between the output and the temporary buffer per
// segment (`buf`); items and the last level's segments that end in the
// temporary buffer are written (sorted, or copied) into the output.
//
// Bounds (all buffers sized by the host from n): segments of a level are
// disjoint and hold > cap keys each, so <= n / (cap + 1); chunks <= n /
// kHeavyChunkKeys + segments; items of a level <= 2 n / cap + segments of this
// and the next level + 1 (two consecutive greedy items hold > cap keys), plus
// the copy pieces.
#pragma once

#ifndef FS_HEAVY_C_UNROLL  // phase C: chunk-count loads in flight per thread (one CTA walks a segment's chunks)
#define FS_HEAVY_C_UNROLL 32
#endif
constexpr int kHeavyCUnroll = FS_HEAVY_C_UNROLL;

// (The records HeavySeg / HeavyItem / HeavyCtl and the capacities are defined in
// wide.cu next to MsdPlan: k_msd_plan seeds the first level.)

template <typename K, bool kHasValues>
struct HeavySmem {
  K keys[2][kHeavyTile + kSlack];
  uint32_t vals[2][kHasValues ? kHeavyTile + kSlack : 1];
  uint16_t whist[kHeavyWarps][kRadix];
  unsigned long long gofs[kRadix];
  uint32_t cnt[kRadix];
  uint64_t mbar[2];
  uint32_t bcast;
};

// Segment records are rewritten by other CTAs between grid barriers: read them
// through L2 (the L1 is not coherent).
FS_DEVINL HeavySeg load_seg(const HeavySeg* p) {
  HeavySeg g;
  g.begin = __ldcg(&p->begin);
  g.count = __ldcg(&p->count);
  g.c0 = __ldcg(&p->c0);
  g.nc = __ldcg(&p->nc);
  g.buf = __ldcg(&p->buf);
  g.skip = __ldcg(&p->skip);
  return g;
}

// Copy items for [b, b + cnt) of the temporary buffer, in pieces.
FS_DEVINL void emit_copy(HeavyCtl* ctl, HeavyItem* items, uint64_t b, uint64_t cnt) {
  for (uint64_t o = 0; o < cnt; o += kHeavyCopyPiece)
    items[atomicAdd(&ctl->nitems, 1u)] = HeavyItem{b + o, min(kHeavyCopyPiece, cnt - o), 0ull, 0u, 1u};
}

// Block-wide exclusive scan over the 256 threads (one value each).
FS_DEVINL uint64_t block_excl_scan256(uint64_t x, uint64_t* wsum64) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t inc = warp_inclusive_scan<uint64_t>(x);
  if (lane == 31) wsum64[warp] = inc;
  __syncthreads();
  uint64_t off = 0;
#pragma unroll
  for (int w = 0; w < kHeavyWarps; ++w)
    if (w < (int)warp) off += wsum64[w];
  __syncthreads();
  return off + inc - x;
}

template <typename K, bool kHasValues>
__global__ void __launch_bounds__(kHeavyThreads, 2) k_heavy(HeavyArgs<K> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<HeavySmem<K, kHasValues>*>(smem_raw);
  __shared__ uint64_t wsum64[kHeavyWarps];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, d = tid;
  const uint64_t gtid = blockIdx.x * (uint64_t)kHeavyThreads + tid, gthreads = (uint64_t)gridDim.x * kHeavyThreads;
  pdl_entry(true);
  if (!a.msd->use_msd) return;
  const uint64_t n_al = a.n & ~(uint64_t)3;  // bulk copies never read past this
  if (tid == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t par = 0;           // bit b: parity of the next phase of buffer b's mbarrier (uniform over the CTA)
  uint32_t nb = 0;            // buffer of the next tile

  const int kb = a.msd->kb;  // the plan's window (below a common prefix, if any)
  const int levels = (kb - kTopBits + kRadixBits - 1) / kRadixBits;
  for (int level = -1; level < levels; ++level) {
    const bool l2 = level < 0;  // the uneven level-2 pass
    const int cur = level & 1;
    HeavySeg* segs = l2 ? a.segl2 : (cur ? a.seg1 : a.seg0);
    HeavySeg* next = cur ? a.seg0 : a.seg1;
    uint32_t* nseg_p = l2 ? &a.ctl->nl2 : &a.ctl->nseg[cur];
    const uint32_t S = __ldcg(nseg_p);
    if (S == 0) {
      if (l2) continue;
      return;  // same value in every CTA (written before the last grid barrier)
    }
    const int slot = level + 1;
    const int rem = kb - kTopBits - kRadixBits * level;  // bits below the digits done so far
    const int w = rem < kRadixBits ? rem : kRadixBits;
    const int sh = rem - w;
    const uint32_t dmask = (1u << w) - 1u;

    // ---- A. chunks of every segment
    for (uint64_t s = gtid; s < S; s += gthreads) {
      const uint64_t cnt = __ldcg(&segs[s].count);
      uint64_t nc = (cnt + kHeavyChunkKeys - 1) / kHeavyChunkKeys;
      nc = nc < 1 ? 1 : (nc > kHeavyMaxChunks ? kHeavyMaxChunks : nc);
      const uint32_t c0 = atomicAdd(&a.ctl->nchunks[slot], (uint32_t)nc);
      segs[s].c0 = c0;
      segs[s].nc = (uint32_t)nc;
      for (uint32_t i = 0; i < (uint32_t)nc; ++i) a.chunk_seg[c0 + i] = (uint32_t)s;
    }
    grid.sync();
    const uint32_t NC = __ldcg(&a.ctl->nchunks[slot]);
    auto chunk_range = [&](uint32_t c, const HeavySeg& sg, uint64_t& cb, uint64_t& ce) {
      const uint64_t i = c - sg.c0;
      cb = sg.begin + sg.count * i / sg.nc;
      ce = sg.begin + sg.count * (i + 1) / sg.nc;
    };

    // ---- B. digit counts per chunk
    for (uint32_t c = blockIdx.x; c < NC; c += gridDim.x) {
      const HeavySeg sg = load_seg(segs + __ldcg(&a.chunk_seg[c]));
      uint64_t cb, ce;
      chunk_range(c, sg, cb, ce);
      const K* src = sg.buf ? a.kalt : a.kout;
      sm.cnt[d] = 0;
      __syncthreads();
      constexpr int kU = 8;  // loads in flight per thread
      for (uint64_t j0 = cb + tid; j0 < ce; j0 += kU * kHeavyThreads) {
        K kk[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) kk[u] = j0 + u * kHeavyThreads < ce ? __ldcg(src + j0 + u * kHeavyThreads) : K(0);
        // (Warp-aggregating equal digits measured slower, even on one-digit segments.)
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (j0 + u * kHeavyThreads < ce) atomicAdd(&sm.cnt[(uint32_t)(kk[u] >> sh) & dmask], 1u);
      }
      __syncthreads();
      a.chist[(uint64_t)c * kRadix + d] = sm.cnt[d];
      __syncthreads();
    }
    grid.sync();

    // ---- C. bases, next-level segments, items
    const bool final_level = sh == 0;
    for (uint32_t s = blockIdx.x; s < S; s += gridDim.x) {
      const HeavySeg sg = load_seg(segs + s);
      uint64_t T = 0;
#pragma unroll kHeavyCUnroll
      for (uint32_t i = 0; i < sg.nc; ++i) T += __ldcg(&a.chist[(uint64_t)(sg.c0 + i) * kRadix + d]);
      const int single = l2 ? 0 : __syncthreads_or(T == sg.count);
      if (single) {  // one digit: nothing moves at this level
        if (tid == 0) {
          segs[s].skip = 1;
          if (!final_level) {
            next[atomicAdd(&a.ctl->nseg[cur ^ 1], 1u)] = HeavySeg{sg.begin, sg.count, 0, 0, sg.buf, 0};
          } else if (sg.buf) {  // sorted (the keys are equal): copy into the output
            emit_copy(a.ctl, a.items, sg.begin, sg.count);
          }
        }
        __syncthreads();
        continue;
      }
      const uint64_t excl = block_excl_scan256(T, wsum64);
      uint64_t run = sg.begin + excl;
#pragma unroll kHeavyCUnroll
      for (uint32_t i = 0; i < sg.nc; ++i) {
        const uint64_t ci = (uint64_t)(sg.c0 + i) * kRadix + d;
        a.cbase[ci] = run;
        run += __ldcg(&a.chist[ci]);
      }
      if (l2) continue;  // the 16-bit bins were planned by k_msd_plan
      sm.gofs[d] = T;    // digit counts for the classification below (thread 0)
      __syncthreads();
      if (tid == 0) {
        const uint32_t dbuf = sg.buf ^ 1u;
        if (final_level) {  // after this scatter the segment is sorted
          if (dbuf) emit_copy(a.ctl, a.items, sg.begin, sg.count);
        } else {
          // the segment's common bits above the digit (every key shares them)
          const K* src = sg.buf ? a.kalt : a.kout;
          const uint64_t key0 = (uint64_t)__ldcg(src + sg.begin);
          const uint64_t common = sh + w >= 64 ? 0ull : key0 & ~((1ull << (sh + w)) - 1);
          uint64_t pos = sg.begin, ib = 0;
          uint32_t isz = 0, d0 = 0, d1 = 0;
          // An item spanning digits d0..d1 holds keys in [top, top + (d1 - d0 + 1) << sh)
          // with top = common | d0 << sh: sorted by ceil(log2(span)) + sh bits, so a
          // merged item's counting digit is not spent on the few digits it spans.
          auto close = [&]() {
            if (isz > 0) {
              const uint32_t span = d1 - d0 + 1;
              const uint32_t lg = span > 1 ? 32 - __clz(span - 1) : 0;
              a.items[atomicAdd(&a.ctl->nitems, 1u)] =
                  HeavyItem{ib, isz, common | ((uint64_t)d0 << sh), (uint32_t)sh + lg, dbuf};
            }
            isz = 0;
          };
          for (uint32_t dd = 0; dd <= dmask; ++dd) {
            const uint64_t t = sm.gofs[dd];
            if (t == 0) continue;
            if (t > (uint64_t)kLocalCap) {
              close();
              next[atomicAdd(&a.ctl->nseg[cur ^ 1], 1u)] = HeavySeg{pos, t, 0, 0, dbuf, 0};
            } else {
              if (isz + t > (uint64_t)kLocalCap) close();
              if (isz == 0) {
                ib = pos;
                d0 = dd;
              }
              isz += (uint32_t)t;
              d1 = dd;
            }
            pos += t;
          }
          close();
        }
      }
      __syncthreads();
    }
    grid.sync();

    // ---- D. scatter: whole chunks per CTA, tiles in order, running offsets
    for (;;) {
      if (tid == 0) sm.bcast = atomicAdd(&a.ctl->ticket[slot], 1u);
      __syncthreads();
      const uint32_t c = sm.bcast;
      __syncthreads();
      if (c >= NC) break;
      const HeavySeg sg = load_seg(segs + __ldcg(&a.chunk_seg[c]));
      if (sg.skip) continue;
      uint64_t cb, ce;
      chunk_range(c, sg, cb, ce);
      const K* src_k = sg.buf ? a.kalt : a.kout;
      const uint32_t* src_v = sg.buf ? a.valt : a.vout;
      K* dst_k = sg.buf ? a.kout : a.kalt;
      uint32_t* dst_v = sg.buf ? a.vout : a.valt;
      uint64_t running = __ldcg(&a.cbase[(uint64_t)c * kRadix + d]);
      for (int i = tid; i < kHeavyWarps * kRadix / 2; i += kHeavyThreads)
        reinterpret_cast<uint32_t*>(&sm.whist[0][0])[i] = 0;
      // The tile starting at t0 -> buffer b: a bulk copy of the 16-byte-aligned
      // span covering it (thread 0), completing on mbar[b].
      auto issue = [&](uint64_t t0, int b) {
        const uint64_t t1 = min(t0 + (uint64_t)kHeavyTile, ce);
        const uint64_t abeg = t0 & ~(uint64_t)3, aend = min((t1 + 3) & ~(uint64_t)3, n_al);
        const uint32_t cnt = aend > abeg ? (uint32_t)(aend - abeg) : 0u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&sm.mbar[b], cnt * (uint32_t)(sizeof(K) + (kHasValues ? 4 : 0)));
        if (cnt) {
          bulk_g2s(sm.keys[b], src_k + abeg, cnt * (uint32_t)sizeof(K), &sm.mbar[b]);
          if (kHasValues) bulk_g2s(sm.vals[b], src_v + abeg, cnt * 4u, &sm.mbar[b]);
        }
      };
      if (a.tma && tid == 0) issue(cb, (int)nb);
      __syncthreads();
      for (uint64_t t0 = cb; t0 < ce; t0 += kHeavyTile) {
        const int b = (int)nb;
        nb ^= 1u;
        const uint32_t len = (uint32_t)min((uint64_t)kHeavyTile, ce - t0);
        K* kbuf = sm.keys[b];
        uint32_t* vbuf = kHasValues ? sm.vals[b] : nullptr;
        uint32_t off = 0;
        if (a.tma) {
          if (tid == 0 && t0 + kHeavyTile < ce) issue(t0 + kHeavyTile, b ^ 1);
          mbar_wait(&sm.mbar[b], (par >> b) & 1u);
          off = (uint32_t)(t0 & 3);
          // keys past the last 16-byte boundary of the array (< 4): plain loads
          const uint64_t t1 = t0 + len, covered = max(min((t1 + 3) & ~(uint64_t)3, n_al), t0);
          if (covered < t1) {
            const uint32_t e0 = (uint32_t)(covered - t0);
            if (tid < len - e0) {
              kbuf[off + e0 + tid] = src_k[covered + tid];
              if (kHasValues) vbuf[off + e0 + tid] = src_v[covered + tid];
            }
            __syncthreads();
          }
        } else {
          for (uint32_t e = tid; e < len; e += kHeavyThreads) {
            kbuf[e] = __ldcg(src_k + t0 + e);
            if (kHasValues) vbuf[e] = __ldcg(src_v + t0 + e);
          }
          __syncthreads();
        }
        par ^= 1u << b;
        K key[kHeavyItems];
        uint32_t val[kHasValues ? kHeavyItems : 1];
        const uint32_t e0 = warp * 32 * kHeavyItems + lane;
#pragma unroll
        for (int i = 0; i < kHeavyItems; ++i) {
          const uint32_t e = e0 + 32 * i;
          key[i] = e < len ? kbuf[off + e] : K(0);
          if (kHasValues) val[i] = e < len ? vbuf[off + e] : 0u;
        }
        uint32_t rank[kHeavyItems];
        uint16_t* wh = sm.whist[warp];
#pragma unroll
        for (int i = 0; i < kHeavyItems; ++i) {
          const bool valid = e0 + 32 * i < len;
          const uint32_t dg = (uint32_t)(key[i] >> sh) & dmask;
          const uint32_t peers = match_digit8(dg, __ballot_sync(kFull, valid));
          const uint32_t leader = 31 - __clz(peers);
          uint32_t old = 0;
          if (valid && lane == leader) {
            old = wh[dg];
            wh[dg] = (uint16_t)(old + __popc(peers));
          }
          old = __shfl_sync(kFull, old, leader);
          rank[i] = old + __popc(peers & lanemask_lt());
          __syncwarp();
        }
        __syncthreads();
        uint32_t cnt = 0;
#pragma unroll
        for (int ww = 0; ww < kHeavyWarps; ++ww) {
          const uint32_t x = sm.whist[ww][d];
          sm.whist[ww][d] = (uint16_t)cnt;
          cnt += x;
        }
        const uint32_t dstart = (uint32_t)block_excl_scan256(cnt, wsum64);
#pragma unroll
        for (int ww = 0; ww < kHeavyWarps; ++ww) sm.whist[ww][d] = (uint16_t)(sm.whist[ww][d] + dstart);
        sm.gofs[d] = running - dstart;
        running += cnt;
        __syncthreads();
        // reorder through shared memory (the tile's buffer becomes the stage)
#pragma unroll
        for (int i = 0; i < kHeavyItems; ++i) {
          if (e0 + 32 * i < len) {
            const uint32_t pos = wh[(uint32_t)(key[i] >> sh) & dmask] + rank[i];
            kbuf[pos] = key[i];
            if (kHasValues) vbuf[pos] = val[i];
          }
        }
        __syncthreads();
        for (uint32_t j = tid; j < len; j += kHeavyThreads) {
          const K k = kbuf[j];
          const uint64_t dst = sm.gofs[(uint32_t)(k >> sh) & dmask] + j;
          dst_k[dst] = k;
          if (kHasValues) dst_v[dst] = vbuf[j];
        }
        for (int i = tid; i < kHeavyWarps * kRadix / 2; i += kHeavyThreads)
          reinterpret_cast<uint32_t*>(&sm.whist[0][0])[i] = 0;
        __syncthreads();  // the buffer is free for the copy after next
      }
    }
    grid.sync();
    if (gtid == 0 && !l2) a.ctl->nseg[cur] = 0;  // reused by level + 2 (written in its phase C, two barriers on)
  }
}

// Every item: sorted (sort_bin) or copied from where it lies into the output.
template <typename K, bool kHasValues>
__global__ void __launch_bounds__(kLocalThreads, 2)
    k_heavy_items(K* __restrict__ kout, uint32_t* __restrict__ vout, const K* __restrict__ kalt,
                  const uint32_t* __restrict__ valt, const HeavyCtl* __restrict__ ctl,
                  const HeavyItem* __restrict__ items, const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  if (!msd->use_msd) return;
  const uint32_t ni = ctl->nitems;
  HeavyItem nxt;
  if (blockIdx.x < ni) nxt = items[blockIdx.x];
  for (uint32_t it = blockIdx.x; it < ni; it += gridDim.x) {
    const HeavyItem item = nxt;
    if (it + gridDim.x < ni) nxt = items[it + gridDim.x];  // in flight during this item's sort
    const K* sk = item.buf ? kalt : kout;
    const uint32_t* sv = item.buf ? valt : vout;
    if (item.R == 0 || item.count <= 1) {
      if (item.buf)
        for (uint64_t j = threadIdx.x; j < item.count; j += kLocalThreads) {
          kout[item.begin + j] = sk[item.begin + j];
          if (kHasValues) vout[item.begin + j] = sv[item.begin + j];
        }
    } else {
      sort_bin<K, kHasValues>(sk, sv, kout, vout, item.begin, (uint32_t)item.count, (int)item.R, (K)item.top);
    }
    __syncthreads();  // the shared memory of sort_bin is reused by the next item
  }
}
