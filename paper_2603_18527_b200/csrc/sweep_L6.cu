// sweep_L6.cu -- kernel instantiations for n = 2^6 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(6)
}
