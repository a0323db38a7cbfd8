// sweep_L9.cu -- kernel instantiations for n = 2^9 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(9)
}
