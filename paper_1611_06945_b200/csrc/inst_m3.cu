// k_tconv instances of MODE 3 (one translation unit per MODE, compiled in parallel; see tconv_inst.cuh)
#define B2C_INST_TU 1
#include "tconv_inst.cuh"

namespace b2c {
B2C_DEFINE_PICK(3)
}  // namespace b2c
