// Engine instantiation for state dimension D = 4.
#define PODE_D 4
#include "inst.cuh"
