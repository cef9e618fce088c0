// Engine instantiation for state dimension D = 15.
#define PODE_D 15
#include "inst.cuh"
