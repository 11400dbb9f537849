// k_relearn.cu -- NEXT-1: in-stream relearning of the background model.
//
// §3.3 P:180 "dealing with the evolution of the luminosity implies sometimes
// to re-initiate partly the machine learning techniques"
// (relearn_trigger), S:170 ("on trigger, runtime pauses tracking and
// relearns"), S:172 ("Relearning swaps the model atomically between
// frames").  Reading L37: a frame whose a2 mean luma differs
// from the previous frame's of the stream by more than the threshold is
// segmented normally and starts relearning; the stream's next F frames are
// learning frames (not segmented, not tracked); after the F-th the model is
// learn(those F raw frames, margin) (the a1 rule) and the tracker restarts.
//
// Means do not depend on the model, so one ordered pass over the call's
// means (relearn_plan_kernel) fixes every frame's role before any of them is
// re-segmented: learning frames (role 1), frames segmented with a model
// learned in this call (role 2, rl_env[f] = that model in the stream's pool),
// and the learning "versions" to build.  relearn_acc_kernel folds each
// version's learning frames (min / max, order-free) into its pool slot (or
// into the stream's carried accumulator when the learning continues into the
// next call); the LUT re-test kernel then re-segments role-2 frames against
// their model and empties role-1 frames (launch_relearn_reseg), and
// relearn_commit_kernel installs the last completed model as the stream's
// model at the end of the call.  Calls with relearning streams run joined
// (the model swap orders the next call's segmentation after this call).
#include "dev_util.cuh"
#include "fizi_internal.cuh"

namespace fizi {

struct RlPair {                          // one model learned (or continued) in this call
  uint32_t stream, slot, continues, complete;
};

// One thread per stream (its frames of the call in index order).
__global__ void relearn_plan_kernel(const CallPtrs* call, uint32_t n, uint32_t n_streams,
                                    const uint32_t* __restrict__ frame_stream,
                                    RelearnState* __restrict__ rs, uint64_t env_plane,
                                    uint32_t* __restrict__ role, uint32_t* __restrict__ pair_of,
                                    uint64_t* __restrict__ env_of, uint32_t* __restrict__ list,
                                    RlPair* __restrict__ pairs, uint32_t* __restrict__ counts,
                                    uint32_t* __restrict__ fg, uint32_t* __restrict__ dirty,
                                    uint32_t dirty_words) {
  __shared__ uint32_t s_list, s_pairs, s_commits;
  for (uint32_t f = threadIdx.x; f < n; f += blockDim.x) role[f] = 0;
  if (threadIdx.x == 0) { s_list = 0; s_pairs = 0; s_commits = 0; }
  __syncthreads();
  fizi_result* res = call->res;
  for (uint32_t s = threadIdx.x; s < n_streams; s += blockDim.x) {
    RelearnState st = rs[s];
    if (!st.enabled) continue;
    int cur_pair = -1;                       // version being learned
    int env_slot = -1;                       // model of the stream's next frames (pool slot)
    uint32_t next_slot = 0;
    for (uint32_t f = 0; f < n; f++) {
      if (frame_stream[f] != s) continue;
      const int32_t m = res[f].mean_luma;
      const bool trig = st.prev_mean >= 0 && abs(m - st.prev_mean) > (int32_t)st.threshold;
      st.prev_mean = m;
      uint32_t flags = 0, r = 0;
      if (st.remaining > 0) {                // a learning frame
        flags = FIZI_RELEARN_LEARN;
        r = 1;
        if (cur_pair < 0) {
          cur_pair = (int)atomicAdd(&s_pairs, 1u);
          FIZI_DCHECK(next_slot < st.pool_slots);
          pairs[cur_pair] = RlPair{s, next_slot++, st.continuing, 0u};
        }
        pair_of[f] = (uint32_t)cur_pair;
        if (--st.remaining == 0) {           // the model is swapped after this frame
          flags |= FIZI_RELEARN_SWAP;
          pairs[cur_pair].complete = 1u;
          env_slot = (int)pairs[cur_pair].slot;
          cur_pair = -1;
          st.continuing = 0;
        }
      } else {
        if (env_slot >= 0) {
          r = 2;
          env_of[f] = st.pool + (uint64_t)env_slot * 2 * env_plane;
        }
        if (trig) {
          flags = FIZI_RELEARN_TRIGGER;
          st.remaining = st.frames;
          st.continuing = 0;
        }
      }
      role[f] = r;
      res[f].relearn = flags;
      if (r) {                               // re-segmented (or emptied) below
        list[1 + atomicAdd(&s_list, 1u)] = f;
        fg[f] = 0;
        for (uint32_t w = 0; w < dirty_words; w++) dirty[(uint64_t)f * dirty_words + w] = 0u;
      }
    }
    if (cur_pair >= 0) st.continuing = 1;    // the learning goes on in the next call
    if (env_slot >= 0) {                     // commit the newest model at the end of the call
      const uint32_t k = atomicAdd(&s_commits, 1u);
      counts[2 + 2 * k] = s;
      counts[3 + 2 * k] = (uint32_t)env_slot;
    }
    rs[s] = st;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    list[0] = s_list;
    counts[0] = s_pairs;
    counts[1] = s_commits;
  }
}

// Version p = blockIdx.y: min / max of its learning frames of this call, from
// the carried accumulator when it continues an earlier call's learning; a
// completed version becomes (sat(min - margin), sat(max + margin)) in its pool
// slot, an incomplete one is carried.  16 bytes per thread (fast path) or one.
__global__ void relearn_acc_kernel(const CallPtrs* call, uint32_t n, uint64_t nbytes, bool fast,
                                   const RelearnState* __restrict__ rs, uint64_t env_plane,
                                   const uint32_t* __restrict__ role,
                                   const uint32_t* __restrict__ pair_of,
                                   const RlPair* __restrict__ pairs,
                                   const uint32_t* __restrict__ counts) {
  const uint32_t p = blockIdx.y;
  if (p >= counts[0]) return;
  const RlPair pr = pairs[p];
  const RelearnState st = rs[pr.stream];
  uint8_t* acc_lo = reinterpret_cast<uint8_t*>(st.acc);
  uint8_t* acc_hi = acc_lo + env_plane;
  uint8_t* out_lo = reinterpret_cast<uint8_t*>(st.pool) + (uint64_t)pr.slot * 2 * env_plane;
  uint8_t* out_hi = out_lo + env_plane;
  const uint8_t* frames = call->frames;
  const uint32_t M = st.margin;
  if (fast) {
    const uint64_t seg = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (seg * 16 >= nbytes) return;
    const uint64_t q = env_perm_index(seg * 16, true);    // 16-byte piece stays contiguous
    uint4 mn = make_uint4(~0u, ~0u, ~0u, ~0u), mx = make_uint4(0, 0, 0, 0);
    if (pr.continues) {
      mn = *reinterpret_cast<const uint4*>(acc_lo + q);
      mx = *reinterpret_cast<const uint4*>(acc_hi + q);
    }
    for (uint32_t f = 0; f < n; f++) {
      if (role[f] != 1 || pair_of[f] != p) continue;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(frames + f * nbytes) + seg);
      mn.x = __vminu4(mn.x, v.x); mn.y = __vminu4(mn.y, v.y);
      mn.z = __vminu4(mn.z, v.z); mn.w = __vminu4(mn.w, v.w);
      mx.x = __vmaxu4(mx.x, v.x); mx.y = __vmaxu4(mx.y, v.y);
      mx.z = __vmaxu4(mx.z, v.z); mx.w = __vmaxu4(mx.w, v.w);
    }
    if (pr.complete) {
      const uint32_t m4 = M * 0x01010101u;
      mn.x = __vsubus4(mn.x, m4); mn.y = __vsubus4(mn.y, m4);
      mn.z = __vsubus4(mn.z, m4); mn.w = __vsubus4(mn.w, m4);
      mx.x = __vaddus4(mx.x, m4); mx.y = __vaddus4(mx.y, m4);
      mx.z = __vaddus4(mx.z, m4); mx.w = __vaddus4(mx.w, m4);
      *reinterpret_cast<uint4*>(out_lo + q) = mn;
      *reinterpret_cast<uint4*>(out_hi + q) = mx;
    } else {
      *reinterpret_cast<uint4*>(acc_lo + q) = mn;
      *reinterpret_cast<uint4*>(acc_hi + q) = mx;
    }
  } else {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= nbytes) return;
    int mn = 255, mx = 0;
    if (pr.continues) { mn = acc_lo[b]; mx = acc_hi[b]; }
    for (uint32_t f = 0; f < n; f++) {
      if (role[f] != 1 || pair_of[f] != p) continue;
      const int v = frames[f * nbytes + b];
      mn = min(mn, v);
      mx = max(mx, v);
    }
    if (pr.complete) {
      out_lo[b] = (uint8_t)max(mn - (int)M, 0);
      out_hi[b] = (uint8_t)min(mx + (int)M, 255);
    } else {
      acc_lo[b] = (uint8_t)mn;
      acc_hi[b] = (uint8_t)mx;
    }
  }
}

// The stream's model := its newest model of this call (pool slot), both planes.
__global__ void relearn_commit_kernel(uint8_t* __restrict__ env, uint64_t env_plane,
                                      const RelearnState* __restrict__ rs,
                                      const uint32_t* __restrict__ counts) {
  const uint32_t k = blockIdx.y;
  if (k >= counts[1]) return;
  const uint32_t s = counts[2 + 2 * k], slot = counts[3 + 2 * k];
  const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(rs[s].pool) +
                                                    (uint64_t)slot * 2 * env_plane);
  uint4* dst = reinterpret_cast<uint4*>(env + (uint64_t)s * 2 * env_plane);
  const uint64_t words = 2 * env_plane / 16;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void relearn_state_kernel(RelearnState* rs, uint32_t stream, RelearnState v) {
  rs[stream] = v;
}

cudaError_t launch_relearn_plan(Ctx& c, uint32_t n, cudaStream_t st) {
  RelearnState* rs = reinterpret_cast<RelearnState*>(c.rstate);
  relearn_plan_kernel<<<1, 1024, 0, st>>>(c.call, n, c.n_streams, c.frame_stream, rs, c.env_plane,
                                          c.rl_role, c.rl_pair, c.rl_env, c.rl_list,
                                          reinterpret_cast<RlPair*>(c.rl_pairs), c.rl_counts, c.fg,
                                          c.dirty, c.dirty_words);
  const uint64_t nbytes = c.N * 3;
  const uint64_t units = c.fast ? nbytes / 16 : nbytes;
  relearn_acc_kernel<<<dim3((unsigned)((units + 255) / 256), c.rl_max_pairs), 256, 0, st>>>(
      c.call, n, nbytes, c.fast, rs, c.env_plane, c.rl_role, c.rl_pair,
      reinterpret_cast<RlPair*>(c.rl_pairs), c.rl_counts);
  c.launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_relearn_commit(Ctx& c, cudaStream_t st) {
  relearn_commit_kernel<<<dim3((unsigned)c.sms, c.rl_max_commits), 256, 0, st>>>(
      c.env, c.env_plane, reinterpret_cast<RelearnState*>(c.rstate), c.rl_counts);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_relearn_state(Ctx& c, uint32_t stream, const RelearnState& v, cudaStream_t st) {
  relearn_state_kernel<<<1, 1, 0, st>>>(reinterpret_cast<RelearnState*>(c.rstate), stream, v);
  c.launches += 1;
  return cudaGetLastError();
}

}  // namespace fizi
