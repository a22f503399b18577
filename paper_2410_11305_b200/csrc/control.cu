// Device-side draft/verify control (K9): token/position staging for each
// draft step and the verify pass, greedy acceptance, rollback-free commit
// (in-place KV: verify rows already overwrote the draft rows), EOS / budget
// truncation and the reference's bookkeeping (specdec.py:258-317, 360-369,
// 325-335).  Everything stays on the device so one CUDA graph replays a whole
// draft-verify cycle for the batch with no host synchronisation.
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {



__device__ __forceinline__ void seq_finish_check(const SeqState& s, int b, int last) {
  if (s.eos >= 0 && last == s.eos) {
    s.done[b] = 1;
    s.finish[b] = 1;
  } else if (s.n_out[b] >= s.max_new[b]) {
    s.done[b] = 1;
    s.finish[b] = 2;
  }
}

// step j of the draft phase (specdec.py:103-133, 258-277)
__global__ void draft_prep_kernel(const SeqState s, int j) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= s.B) return;
  if (j == 0) {
    const int remaining = s.max_new[b] - s.n_out[b];
    int g = min(s.gamma, max(1, remaining - 1));
    g = min(g, s.max_seq - s.committed[b] - 1);
    s.g_eff[b] = max(g, 1);
    s.tok[b] = s.pending[b];
  } else {
    const int prev = s.argmax[b];
    s.drafted[b * s.gamma + j - 1] = prev;
    s.tok[b] = prev;
  }
  s.pos[b] = s.committed[b] + j;
  s.slot[b] = b;
}

// verify input [pending, drafted...] (specdec.py:136-156)
__global__ void verify_prep_kernel(const SeqState s) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= s.B) return;
  const int G1 = s.gamma + 1;
  s.drafted[b * s.gamma + s.gamma - 1] = s.argmax[b];
  for (int i = 0; i < G1; ++i) {
    s.tok[b * G1 + i] = i == 0 ? s.pending[b] : s.drafted[b * s.gamma + i - 1];
    s.pos[b * G1 + i] = s.committed[b] + i;
    s.slot[b * G1 + i] = b;
  }
}

// greedy acceptance + commit (specdec.py:159-176, 279-317)
__global__ void accept_kernel(const SeqState s) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= s.B || s.done[b]) return;
  const int G1 = s.gamma + 1;
  const int* dr = s.drafted + b * s.gamma;
  const int* vt = s.argmax + b * G1;
  const int gl = s.g_eff[b];
  int dl = gl;
  if (s.eos >= 0)
    for (int k = 0; k < gl; ++k)
      if (dr[k] == s.eos) { dl = k + 1; break; }
  int a = 0;
  while (a < dl && dr[a] == vt[a]) ++a;
  const int next = vt[a];
  const int remaining = s.max_new[b] - s.n_out[b];
  int kept = min(a + 1, remaining);
  if (s.eos >= 0) {
    for (int k = 0; k < kept; ++k) {
      const int tkn = k < a ? dr[k] : next;
      if (tkn == s.eos) { kept = k + 1; break; }
    }
  }
  int* out = s.out_tokens + (size_t)b * s.out_cap;
  const int n0 = s.n_out[b];
  int last = next;
  for (int k = 0; k < kept; ++k) {
    last = k < a ? dr[k] : next;
    if (n0 + k < s.out_cap) out[n0 + k] = last;
  }
  const int cyc = s.n_cycles[b];
  if (cyc < s.trace_cap) {
    int* tr = s.trace + ((size_t)b * s.trace_cap + cyc) * 4;
    tr[0] = dl; tr[1] = a; tr[2] = kept; tr[3] = (a == dl);
    int* tt = s.trace_tok + ((size_t)b * s.trace_cap + cyc) * s.gamma;
    for (int k = 0; k < s.gamma; ++k) tt[k] = k < dl ? dr[k] : -1;
  }
  s.dropped[b] += (a + 1) - kept;
  s.n_out[b] = n0 + kept;
  s.committed[b] += kept;
  s.pending[b] = last;
  s.n_drafted[b] += dl;
  s.n_accepted[b] += a;
  s.n_cycles[b] = cyc + 1;
  seq_finish_check(s, b, last);
}

// plain greedy decode step (specdec.py:325-335)
__global__ void ar_prep_kernel(const SeqState s) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= s.B) return;
  s.tok[b] = s.pending[b];
  s.pos[b] = s.committed[b];
  s.slot[b] = b;
}

__global__ void ar_commit_kernel(const SeqState s) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= s.B || s.done[b]) return;
  const int nxt = s.argmax[b];
  const int n0 = s.n_out[b];
  if (n0 < s.out_cap) s.out_tokens[(size_t)b * s.out_cap + n0] = nxt;
  s.n_out[b] = n0 + 1;
  s.committed[b] += 1;
  s.pending[b] = nxt;
  seq_finish_check(s, b, nxt);
}

cudaError_t launch_control(int op, const SeqState& s, int j, cudaStream_t st) {
  const int bs = 128, nb = (s.B + bs - 1) / bs;
  switch (op) {
    case 0: return launch_k(draft_prep_kernel, dim3(nb), dim3(bs), 0, st, s, j);
    case 1: return launch_k(verify_prep_kernel, dim3(nb), dim3(bs), 0, st, s);
    case 2: return launch_k(accept_kernel, dim3(nb), dim3(bs), 0, st, s);
    case 3: return launch_k(ar_prep_kernel, dim3(nb), dim3(bs), 0, st, s);
    case 4: return launch_k(ar_commit_kernel, dim3(nb), dim3(bs), 0, st, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace qs

namespace qs {
// x += y elementwise (tensor-parallel residual: y = the all-reduced partial of a
// row-split o_proj / down_proj).  Same fp32 add as the kOpResidual epilogue.
__global__ void add_rows_kernel(float* __restrict__ x, const float* __restrict__ y, int n) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = __fadd_rn(x[i], y[i]);
}
cudaError_t launch_add_rows(float* x, const float* y, int n, cudaStream_t st) {
  return launch_k(add_rows_kernel, dim3((n + 255) / 256), dim3(256), 0, st, x, y, n);
}
}  // namespace qs
