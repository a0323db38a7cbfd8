// sweep_L5.cu -- kernel instantiations for n = 2^5 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(5)
}
