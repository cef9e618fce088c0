// Engine instantiation for state dimension D = 9.
#define PODE_D 9
#include "inst.cuh"
