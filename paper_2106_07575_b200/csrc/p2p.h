// Peer-memory transport (kernels_p2p.cu): exchange-window layout shared by the host runtime and the
// kernels.  Every rank's window is one cudaMalloc allocation exported with CUDA IPC:
//   [flags u64 [P2P_MAX_RANKS][P2P_CHANNELS] | mailbox f64 [2][P2P_MAX_RANKS][P2P_MBW] |
//    full object c64 [2][H*W] | recv0 c64 [band rows from the left neighbour * W] | recv1 (right)]
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace pty {

constexpr int P2P_MAX_RANKS = 8;
constexpr int P2P_CHANNELS = 4;
constexpr int P2P_CH_BAND = 0, P2P_CH_SCALAR = 1, P2P_CH_GATHER = 2;
constexpr int P2P_MBW = 32;   // doubles per mailbox slot (>= LSW)
static_assert(P2P_MBW >= LSW, "mailbox slot too small");

struct P2PView {
    unsigned char* win[P2P_MAX_RANKS];   // every rank's window mapped into this process (own included)
    int world, rank;
    int64_t off_flags, off_mail, off_full, full_elems;
    int64_t off_recv0[P2P_MAX_RANKS], off_recv1[P2P_MAX_RANKS];
};

int launch_p2p_band(const float2* gcur, int64_t lo0, int64_t rows0, int64_t lo1, int64_t rows1, int64_t W,
                    const P2PView& v, DevState* st, int grid, cudaStream_t s);
int launch_p2p_allreduce(double* buf, int count, const P2PView& v, DevState* st, cudaStream_t s);
// gathers owned rows [lo, hi) (global) of src into every window's full buffer of the current epoch
// parity; returns that parity through *par_out (host-known: the gather epoch counter is mirrored)
int launch_p2p_gather(const float2* src, int64_t st_lo, int64_t lo, int64_t hi, int64_t W, const P2PView& v,
                      DevState* st, int grid, cudaStream_t s);

}  // namespace pty
