// sweep_L12.cu -- kernel instantiations for n = 2^12 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(12)
}
