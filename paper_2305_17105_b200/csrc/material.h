// material.h -- the device-resident material behind the opaque ntc_material handle.
#pragma once
#include "common.cuh"

struct ntc_material {
    ntc_desc d;
    int pid, M, L;
    uint8_t* grids = nullptr;  // bit-packed latent cells, per level G0 then G1
    uint4* wimg = nullptr;     // UMMA-swizzled fp16 weight image (decode SMEM layout)
    uint32_t wimg_bytes = 0;
    ntc::LevelGeom lv[ntc::MAX_LEVELS];
    float b3[16];              // output bias (kernel parameter)
    int num_sms = 148;
};
