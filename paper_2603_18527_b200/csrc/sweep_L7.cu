// sweep_L7.cu -- kernel instantiations for n = 2^7 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(7)
}
