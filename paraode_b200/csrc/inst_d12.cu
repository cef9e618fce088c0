// Engine instantiation for state dimension D = 12.
#define PODE_D 12
#include "inst.cuh"
