// sweep_L4.cu -- kernel instantiations for n = 2^4 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(4)
}
