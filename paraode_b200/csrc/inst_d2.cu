// Engine instantiation for state dimension D = 2.
#define PODE_D 2
#include "inst.cuh"
