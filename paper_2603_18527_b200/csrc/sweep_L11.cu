// sweep_L11.cu -- kernel instantiations for n = 2^11 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(11)
}
