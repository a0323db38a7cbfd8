// sweep_L10.cu -- kernel instantiations for n = 2^10 (see sweep_launch.cuh)
#include "sweep_launch.cuh"
namespace bs {
BS_DEFINE_SIZE(10)
}
