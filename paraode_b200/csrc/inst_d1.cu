// Engine instantiation for state dimension D = 1.
#define PODE_D 1
#include "inst.cuh"
