// Engine instantiation for state dimension D = 6.
#define PODE_D 6
#include "inst.cuh"
