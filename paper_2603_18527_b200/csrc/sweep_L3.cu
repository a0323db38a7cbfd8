// sweep_L3.cu -- kernel instantiations for n = 2^3 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(3)
}
