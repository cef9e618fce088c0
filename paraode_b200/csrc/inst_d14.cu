// Engine instantiation for state dimension D = 14.
#define PODE_D 14
#include "inst.cuh"
