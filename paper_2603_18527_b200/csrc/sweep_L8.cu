// sweep_L8.cu -- kernel instantiations for n = 2^8 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(8)
}
