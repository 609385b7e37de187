// fmoe/param_tag.hpp -- which ranks share a parameter's gradient (reference:
// proj/include/fmoe/param_tag.hpp).  World: all ranks (the gate);
// DataParallel: ranks with equal rank % model_parallel_size; NoSync: local
// (experts).
#pragma once

namespace fmoe {

enum class ParamTag { World, DataParallel, NoSync };

const char* to_string(ParamTag tag);

}  // namespace fmoe
