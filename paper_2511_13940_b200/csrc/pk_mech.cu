// pk_mech.cu — transfer-mechanism calibration (pk_mech_probe).
//
// The reference decides every transfer mechanism from a hardware model: a
// capability matrix plus per-mechanism bandwidth over message size and SM
// count (overlapsim/hwmodel.py:34-51, 147-245), whose B200 constants are the
// paper's Table 1 and H100 saturation counts carried over
// (hwmodel.py:264-287). Here those numbers are measured: one probe moves
// `bytes` between this rank and a peer with one mechanism, a message size and
// an SM budget, and the caller times it (CUDA events, max over ranks):
//   PK_MECH_REG       16 B ld.global / st.global per thread (register ops),
//                     8 vectors in flight, one 512-thread CTA per SM; the
//                     message is the contiguous run at the destination
//                     (messages land scattered)
//   PK_MECH_TMA       cp.async.bulk global -> smem -> global, one thread per
//                     CTA (one CTA per SM) keeping up to 32 messages in flight
//   PK_MECH_CE        the copy engine (cudaMemcpyAsync), one call per message
//   PK_MECH_MULTIMEM  multimem.st.v4 of local data through the multicast VA:
//                     one store reaches every rank (in-fabric broadcast)
// push: local src -> the peer's dst; pull: the peer's src -> local dst.
// On one GPU (world 1, or an emulated local group) the "peer" is HBM on the
// same device: a loopback figure, not NVLink.
#include "pk_host.h"
#include "pk_ptx.cuh"
#include <algorithm>

namespace pk {

constexpr int kProbeThreads = 512;
constexpr int kProbeTmaSmem = 192 * 1024;
constexpr int kProbeMaxPiece = 48 * 1024;

struct ProbeArgs {
  const uint8_t* src;
  uint8_t* dst;
  long long bytes;
  long long msg;        // bytes per message (the last one may be short)
};

// register ops: every thread moves 16 B vectors (8 in flight); the buffer is
// cut into `msg`-byte messages whose destinations are scattered (message c
// lands at slot c * P mod nmsg, P coprime to nmsg), so a message is the
// contiguous granularity the fabric sees
template <bool MULTIMEM>
__global__ void __launch_bounds__(kProbeThreads) probe_reg_kernel(const __grid_constant__ ProbeArgs a, long long perm) {
  constexpr int U = 8;
  const long long nvec = a.bytes / 16;
  const long long per_msg = a.msg / 16;
  const long long nmsg = (a.bytes + a.msg - 1) / a.msg;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long v0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long v = v0 + u * stride;
      if (v < nvec) r[u] = ld_v4(a.src + v * 16);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long v = v0 + u * stride;
      if (v >= nvec) continue;
      const long long m = v / per_msg;
      const long long dm = nmsg > 1 ? (m * perm) % nmsg : 0;
      const long long o = (dm * per_msg + (v - m * per_msg)) * 16;
      if (o + 16 > a.bytes) continue;                 // the short last message's slot may not fit
      if constexpr (MULTIMEM) {
        const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
        mm_st_v4(a.dst + o, w);
      } else {
        st_v4(a.dst + o, r[u]);
      }
    }
  }
}

// TMA bulk copies: messages dealt round-robin to the CTAs; per CTA one thread
// keeps NBUF messages (pieces of <= 48 KB) in flight through shared memory
__global__ void __launch_bounds__(32) probe_tma_kernel(const __grid_constant__ ProbeArgs a, int piece, int nbuf) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[32];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < nbuf; ++i) mbar_init(&bars[i], 1);
  fence_mbar_init();
  const long long nmsg = (a.bytes + a.msg - 1) / a.msg;
  const long long ppm = (a.msg + piece - 1) / piece;                 // pieces per message
  // this CTA's pieces, in order: message m = blockIdx.x + j * gridDim.x
  const long long my_msgs = nmsg > blockIdx.x ? (nmsg - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long total = my_msgs * ppm;
  auto piece_at = [&](long long p, long long* off, uint32_t* len) -> bool {
    const long long m = blockIdx.x + (p / ppm) * gridDim.x;
    const long long m0 = m * a.msg, m1 = min(a.bytes, m0 + a.msg);
    *off = m0 + (p % ppm) * piece;
    if (*off >= m1) return false;
    *len = (uint32_t)min((long long)piece, m1 - *off);
    return true;
  };
  auto issue = [&](long long p) {
    long long off;
    uint32_t len;
    if (!piece_at(p, &off, &len)) return;
    const int b = (int)(p % nbuf);
    mbar_arrive_expect_tx(&bars[b], len);
    bulk_g2s(smem + (size_t)b * piece, a.src + off, len, &bars[b]);
  };
  for (long long p = 0; p < total && p < nbuf - 1; ++p) issue(p);
  uint32_t phase = 0;
  for (long long p = 0; p < total; ++p) {
    long long off;
    uint32_t len;
    const bool real = piece_at(p, &off, &len);
    const int b = (int)(p % nbuf);
    if (real) {
      mbar_wait(&bars[b], (phase >> b) & 1);
      phase ^= 1u << b;
      bulk_s2g(a.dst + off, smem + (size_t)b * piece, len);
    }
    bulk_commit();
    if (p + nbuf - 1 < total) {
      bulk_wait_read<1>();            // the buffer of piece p + nbuf - 1 (last used by p - 1) was read
      issue(p + nbuf - 1);
    }
  }
  bulk_wait<0>();
}

int preload_mech() {
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, probe_reg_kernel<false>));
  PK_CUDA(cudaFuncGetAttributes(&fa, probe_reg_kernel<true>));
  PK_CUDA(cudaFuncGetAttributes(&fa, probe_tma_kernel));
  return PK_OK;
}

int mech_probe(Comm* c, Pgl* src, Pgl* dst, int peer, size_t bytes, size_t msg, int mech, int pull, int num_sms,
               cudaStream_t st) {
  if (!src || !dst) return fail(PK_ERR_INVALID, "mech_probe: null pgl");
  if (peer < 0 || peer >= c->world) return fail(PK_ERR_INVALID, "mech_probe: peer %d outside the world of %d", peer, c->world);
  if (bytes == 0) return PK_OK;
  if (bytes > src->bytes || bytes > dst->bytes) return fail(PK_ERR_INVALID, "mech_probe: %zu bytes exceed the PGLs", bytes);
  if (msg == 0 || msg % 16 || bytes % 16) return fail(PK_ERR_INVALID, "mech_probe: bytes and message size must be 16 B multiples");
  const uint8_t* s = static_cast<const uint8_t*>(pull ? src->peers[peer] : src->local);
  uint8_t* d = static_cast<uint8_t*>(pull ? dst->local : dst->peers[peer]);
  int sms = c->num_sms;
  if (num_sms > 0) sms = std::min(sms, num_sms);
  ProbeArgs a{s, d, (long long)bytes, (long long)msg};
  switch (mech) {
    case PK_MECH_CE: {
      for (size_t off = 0; off < bytes; off += msg)
        PK_CUDA(cudaMemcpyAsync(d + off, s + off, std::min(msg, bytes - off), cudaMemcpyDeviceToDevice, st));
      return PK_OK;
    }
    case PK_MECH_REG:
    case PK_MECH_MULTIMEM: {
      if (mech == PK_MECH_MULTIMEM) {
        if (!dst->mc) return fail(PK_ERR_CAPABILITY, "mech_probe: multimem needs a multicast PGL (NVLS)");
        a.src = static_cast<const uint8_t*>(src->local);
        a.dst = static_cast<uint8_t*>(dst->mc);
      }
      const long long nmsg = (long long)((bytes + msg - 1) / msg);
      long long perm = 1;                               // scatter stride: coprime to nmsg, near nmsg / phi
      if (nmsg > 2) {
        perm = (long long)(0.618 * (double)nmsg) | 1;
        auto gcd = [](long long x, long long y) { while (y) { long long t = x % y; x = y; y = t; } return x; };
        while (gcd(perm, nmsg) != 1) perm += 2;
      }
      const long long nvec = (long long)(bytes / 16);
      const int blocks = (int)std::max<long long>(1, std::min<long long>(sms, (nvec + kProbeThreads * 8 - 1) / (kProbeThreads * 8)));
      if (mech == PK_MECH_MULTIMEM) probe_reg_kernel<true><<<blocks, kProbeThreads, 0, st>>>(a, perm);
      else probe_reg_kernel<false><<<blocks, kProbeThreads, 0, st>>>(a, perm);
      PK_CUDA(cudaGetLastError());
      return PK_OK;
    }
    case PK_MECH_TMA: {
      const int piece = (int)std::min<size_t>(msg, kProbeMaxPiece);
      const int nbuf = std::max(2, std::min(32, kProbeTmaSmem / piece));
      const long long nmsg = (long long)((bytes + msg - 1) / msg);
      const int blocks = (int)std::max<long long>(1, std::min<long long>(sms, nmsg));
      const int smem = nbuf * piece;
      PK_TRY(ensure_smem_attr((const void*)probe_tma_kernel, kProbeTmaSmem));
      probe_tma_kernel<<<blocks, 32, smem, st>>>(a, piece, nbuf);
      PK_CUDA(cudaGetLastError());
      return PK_OK;
    }
  }
  return fail(PK_ERR_INVALID, "mech_probe: unknown mechanism %d", mech);
}

}  // namespace pk

extern "C" PK_API int pk_mech_probe(pk_comm* comm, pk_pgl* src, pk_pgl* dst, int peer, size_t bytes,
                                    size_t msg_bytes, int mechanism, int pull, int num_sms, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::mech_probe(comm, src, dst, peer, bytes, msg_bytes, mechanism, pull, num_sms, (cudaStream_t)stream);
}
