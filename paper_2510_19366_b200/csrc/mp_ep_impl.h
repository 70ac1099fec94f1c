// mp_ep_impl.h -- internal state of an expert-parallel handle (mp_ep_t),
// shared by ep.cu (plan / pack / combine / peer-memory exchange) and
// ep_nccl.cu (the NCCL-transport layer forward, mp_ep_forward).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "mp_kernels.h"

struct mp_ep_nccl_s;  // ep_nccl.cu

struct mp_ep_s {
    uint32_t world, rank, per_rank, S, d, k_max, max_tokens, dtype;
    int device;
    uint32_t* dest = nullptr;
    mp::BucketWs ws{};
    uint32_t last_T = 0;
    // peer-memory exchange (mp_ep_p2p_*): own receive / return buffers, the
    // peers' (CUDA IPC) and device tables of [world] pointers
    uint32_t max_recv = 0;
    void* recv_x = nullptr;
    uint32_t* recv_sel = nullptr;
    float* recv_w = nullptr;
    void* back = nullptr;
    std::vector<void*> opened;  // IPC mappings to close
    void** d_px = nullptr;      // device [4][world]: x, sel, w, back
    uint32_t* d_meta = nullptr; // device [4][world + 1]: base, roff, dbase, ones
    bool p2p = false;
    mp_ep_nccl_s* nccl = nullptr;  // NCCL transport (mp_ep_nccl_init), owned
};

// ep_nccl.cu: releases the NCCL transport of a handle (communicator, buffers)
void mp_ep_nccl_free(mp_ep_s* E);

