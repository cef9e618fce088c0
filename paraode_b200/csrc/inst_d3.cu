// Engine instantiation for state dimension D = 3.
#define PODE_D 3
#include "inst.cuh"
