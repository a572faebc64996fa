// lstm_rec_args.h -- launch arguments of the persistent LSTM recurrence (lstm_rec.cuh).
#pragma once
#include <cstdint>

namespace axq {

struct LstmRecArgs {
    int T, B, H;
    const float* gih;        // [T][B][4H]: fl(ih_deq + b_ih)
    const int8_t* qw;        // [4H][H] W_hh codes
    const float* sw;         // device scalar: W_hh scale
    const float* b_hh;       // [4H]
    const float* sh;         // device scalar: static scale of h
    int bits;
    const int8_t* table;     // delta8 [uw8][ua8] (64 KiB)
    float* hs;               // [T][B][H]
    float* c_out;            // [B][H]: c_T
    int8_t* hq;              // [2][B][H] exchange buffer of h codes
    unsigned int* bar;       // grid barrier counter (zero at launch)
};

}  // namespace axq
