#ifndef SELECT_F32_NN_H
#define SELECT_F32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nn_config;

static inline select_f32_nn_config select_f32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(448)) {
        if (m < INT64_C(12)) {
            select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
            return out;
        } else {
            if (n < INT64_C(144)) {
                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                return out;
            } else {
                if (n < INT64_C(544)) {
                    if (m < INT64_C(139)) {
                        if (n < INT64_C(227)) {
                            select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(3072)) {
                                if (k < INT64_C(992)) {
                                    if (m < INT64_C(70)) {
                                        select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(287)) {
                            if (k < INT64_C(1536)) {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(70)) {
                        if (n < INT64_C(1132)) {
                            if (m < INT64_C(29)) {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(405)) {
                                if (m < INT64_C(139)) {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(124)) {
                                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(405)) {
                                if (k < INT64_C(124)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(287)) {
                                        select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(4435)) {
            if (n < INT64_C(363)) {
                if (m < INT64_C(2218)) {
                    if (n < INT64_C(144)) {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(236)) {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(46)) {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(363)) {
                                    if (k < INT64_C(222)) {
                                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(128)) {
                            if (m < INT64_C(1109)) {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                if (m < INT64_C(1109)) {
                                    select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(46)) {
                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(111)) {
                            if (k < INT64_C(314)) {
                                if (k < INT64_C(222)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(222)) {
                                if (k < INT64_C(28)) {
                                    select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(725)) {
                                    select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1087)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(1792)) {
                    if (n < INT64_C(544)) {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(725)) {
                                if (m < INT64_C(634)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(182)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(896)) {
                            if (k < INT64_C(124)) {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(287)) {
                                    select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(405)) {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(768)) {
                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(2535)) {
                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(28)) {
                if (m < INT64_C(8870)) {
                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(118)) {
                        select_f32_nn_config out = {4u, 2u, 8u, 128u, 1u};
                        return out;
                    } else {
                        if (m < INT64_C(35480)) {
                            select_f32_nn_config out = {4u, 2u, 8u, 128u, 1u};
                            return out;
                        } else {
                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(70960)) {
                    if (k < INT64_C(815)) {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(167)) {
                                if (k < INT64_C(363)) {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(167)) {
                                            if (k < INT64_C(59)) {
                                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(96)) {
                                            if (k < INT64_C(20)) {
                                                select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(46)) {
                                                    select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(168)) {
                                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(222)) {
                                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(544)) {
                                            select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(182)) {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(26)) {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(42)) {
                                    if (n < INT64_C(46)) {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(97)) {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(35480)) {
                                            if (n < INT64_C(91)) {
                                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(291)) {
                                                select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(182)) {
                            if (m < INT64_C(8870)) {
                                select_f32_nn_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(35480)) {
                                        select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(25088)) {
                                if (k < INT64_C(6144)) {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(21)) {
                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(46)) {
                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(141920)) {
                                if (k < INT64_C(291)) {
                                    select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(91)) {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        }
    }
}

#endif /* SELECT_F32_NN_H */
